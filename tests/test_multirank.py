"""World-size-2 tests of the multi-GPU host logic on CPU (gloo backend).

They check the exchange protocol the library implements over NCCL
with the oracle standing in for each rank's kernels:
  * the NCCL unique id bootstrap delivers identical bytes to every rank;
  * S5: merging the per-rank top-k lists (all-gather) gives exactly the unsharded top-k;
  * S7: every rank reduces only the winners it OWNS into a partial prediction P_g; the
    partials are exchanged (all-gather, or all-to-all by query slice + broadcast of the
    finished slices -- the two layouts runtime.cu picks by size) and summed in rank order,
    so every rank holds the same prediction, equal to the unsharded one.
The library's own implementation of this protocol (runtime.cu stage functions) runs on
one GPU through a loopback group: tests/test_gpu_loopback.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return out


def _bootstrap(rank, world):
    from paper_2512_18674_b200.dist import broadcast_unique_id
    return broadcast_unique_id()


def test_unique_id_bootstrap_over_gloo():
    out = run_ranks(_bootstrap)
    assert isinstance(out[0], bytes) and len(out[0]) == 128
    assert out[0] == out[1]


def _exchange(rank, world):
    import gen
    import oracle
    from paper_2512_18674_b200.dist import shard_range
    c = gen.CONFIGS["c2"]
    n_total, k, B = 6001, 10, 8
    off, n = shard_range(n_total, world, rank)
    x = gen.store_emb(c.store_seed, n_total, c.dim, off, n)
    a = gen.store_act(c.store_seed, n_total, c.layers, c.experts, c.moe_topk, off, n)
    q = gen.queries(c.store_seed, c.query_seed, n_total, c.dim, B, mode=1)
    ids, sc, _ = oracle.sps(q, x, a, min(k, n), id_offset=off, want_pred=False)
    # S5: all-gather (score, id) candidates, identical deterministic merge on every rank
    cand = torch.from_numpy(np.stack([sc, ids.astype(np.float64)], -1))   # [B, k, 2]
    allc = [torch.zeros_like(cand) for _ in range(world)]
    dist.all_gather(allc, cand)
    merged = torch.cat(allc, 1).numpy()                                  # [B, G*k, 2]
    top_ids = np.empty((B, k), np.int64)
    top_sc = np.empty((B, k))
    for i in range(B):
        order = sorted(range(merged.shape[1]), key=lambda r: (-merged[i, r, 0], merged[i, r, 1]))[:k]
        top_ids[i] = merged[i, order, 1].astype(np.int64)
        top_sc[i] = merged[i, order, 0]
    # S6 + partial S7: weights from the (identical) merged scores; P_g over owned winners
    L, E = c.layers, c.experts
    part = np.zeros((B, L, E))
    for i in range(B):
        w = oracle.softmax(top_sc[i])
        for r in range(k):
            j = top_ids[i, r] - off
            if 0 <= j < n:
                part[i] += w[r] * a[j].astype(np.float64)
    # exchange 2, layout 1: all-gather of whole partials, rank-order sum
    allp = [torch.zeros(B, L, E, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allp, torch.from_numpy(part))
    pred_ag = sum(p.numpy() for p in allp)  # g ascending
    # layout 2: rank g owns query slice [B g / G, B (g+1) / G): it receives every rank's
    # partial of its slice (all_gather stands in for the all-to-all), sums in rank order,
    # then the finished slices are broadcast from their owners
    lo = [B * g // world for g in range(world + 1)]
    mine = [torch.zeros(lo[rank + 1] - lo[rank], L, E, dtype=torch.float64) for _ in range(world)]
    for g in range(world):
        src = torch.from_numpy(part[lo[g]:lo[g + 1]].copy())
        got = [torch.zeros_like(src) for _ in range(world)]
        dist.all_gather(got, src)
        if g == rank:
            mine = got
    pred_a2a = np.zeros((B, L, E))
    pred_a2a[lo[rank]:lo[rank + 1]] = sum(t.numpy() for t in mine)
    for g in range(world):
        sl = torch.from_numpy(pred_a2a[lo[g]:lo[g + 1]].copy())
        dist.broadcast(sl, g)
        pred_a2a[lo[g]:lo[g + 1]] = sl.numpy()
    return top_ids, top_sc, pred_ag, pred_a2a


def test_sharded_exchange_equals_unsharded_oracle():
    import sys
    sys.path.insert(0, ROOT)
    import gen
    import oracle
    out = run_ranks(_exchange)
    assert not isinstance(out[0], str), out[0]
    c = gen.CONFIGS["c2"]
    n_total, k, B = 6001, 10, 8
    x = gen.store_emb(c.store_seed, n_total, c.dim)
    a = gen.store_act(c.store_seed, n_total, c.layers, c.experts, c.moe_topk)
    q = gen.queries(c.store_seed, c.query_seed, n_total, c.dim, B, mode=1)
    ids, sc, pred = oracle.sps(q, x, a, k)
    for r in (0, 1):
        top_ids, top_sc, pred_ag, pred_a2a = out[r]
        np.testing.assert_array_equal(top_ids, ids)          # exact global top-k
        np.testing.assert_array_equal(top_sc, sc)
        np.testing.assert_allclose(pred_ag, pred, rtol=0, atol=1e-14)   # owner partials, summed
        np.testing.assert_array_equal(pred_a2a, pred_ag)     # both layouts: the same rank-order sum
    for u, v in zip(out[0], out[1]):
        np.testing.assert_array_equal(u, v)                   # identical on every rank


def test_shard_range_matches_generator():
    import sys
    sys.path.insert(0, ROOT)
    import gen
    from paper_2512_18674_b200.dist import shard_range
    for n in (1, 5, 9, 1000, 10_000_000):
        for w in (1, 2, 3, 4, 8):
            parts = [shard_range(n, w, r) for r in range(w)]
            for r in range(w):
                assert parts[r] == gen.shard_range(n, w, r)
            assert parts[0][0] == 0 and sum(p[1] for p in parts) == n   # tiles [0, n)
            for r in range(1, w):
                assert parts[r][0] == parts[r - 1][0] + parts[r - 1][1]
            if n >= w:
                assert min(p[1] for p in parts) >= 1                    # balanced: none empty
                assert max(p[1] for p in parts) - min(p[1] for p in parts) <= 1
