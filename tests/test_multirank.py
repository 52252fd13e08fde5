"""World-size-2 tests of the multi-GPU host logic on CPU (gloo backend).

They check the exchange protocol the library implements over NCCL
with the oracle standing in for each rank's kernels:
  * the NCCL unique id bootstrap delivers identical bytes to every rank;
  * S5: merging the per-rank top-k lists (all-gather) gives exactly the unsharded top-k;
  * S7: the all-reduce of owned winner rows (zeros elsewhere) reproduces every winner
    row bit-exactly on every rank, so the prediction equals the one-GPU prediction.
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
    # S7: owned winner rows, zeros elsewhere, summed across ranks
    L, E = c.layers, c.experts
    rows = np.zeros((B, k, L, E), np.float32)
    for i in range(B):
        for r in range(k):
            j = top_ids[i, r] - off
            if 0 <= j < n:
                rows[i, r] = a[j]
    t = torch.from_numpy(rows)
    dist.all_reduce(t)
    return top_ids, top_sc, t.numpy()


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
        top_ids, top_sc, rows = out[r]
        np.testing.assert_array_equal(top_ids, ids)          # exact global top-k
        np.testing.assert_array_equal(top_sc, sc)
        np.testing.assert_array_equal(rows, a[ids])          # exact winner rows on every rank
        # the prediction from the gathered rows equals the one-GPU prediction
        w = np.stack([oracle.softmax(top_sc[i]) for i in range(B)])
        p = np.einsum("br,brle->ble", w, rows.astype(np.float64))
        np.testing.assert_allclose(p, pred, rtol=0, atol=1e-15)
    for u, v in zip(out[0], out[1]):
        np.testing.assert_array_equal(u, v)                   # identical on every rank


def test_shard_range_matches_generator():
    import sys
    sys.path.insert(0, ROOT)
    import gen
    from paper_2512_18674_b200.dist import shard_range
    for n in (1, 5, 1000, 10_000_000):
        for w in (1, 2, 4, 8):
            for r in range(w):
                assert shard_range(n, w, r) == gen.shard_range(n, w, r)
