"""Multi-GPU SPS through NCCL (needs >= 2 GPUs; skipped otherwise), plus the one-GPU
shard check: handles built on row shards (global_offset) return global ids whose
host-side merge equals the unsharded result."""
import os
import socket

import numpy as np
import pytest

import gen
import oracle
from parity import compare

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("remoe_lib_built")]
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_18674_b200 as remoe  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_offsets_on_one_gpu():
    c = gen.CONFIGS["c2"]
    n, B, k = 30_000, 12, 10
    x = gen.store_emb(c.store_seed, n, c.dim)
    a = gen.store_act(c.store_seed, n, c.layers, c.experts, c.moe_topk)
    qb = gen.queries(c.store_seed, c.query_seed, n, c.dim, B, mode=1)
    q = torch.from_numpy(qb.view(np.int16)).cuda()
    parts = []
    for g in range(3):
        off, nl = gen.shard_range(n, 3, g)
        s = remoe.Sps(x[off:off + nl].copy(), a[off:off + nl].copy(), global_offset=off, max_k=16)
        ids, sc, _ = s.query(q, k, want_pred=False)
        parts.append((ids.cpu().numpy(), sc.cpu().numpy()))
        s.close()
    full = remoe.Sps(x, a, max_k=16)
    ids_f, sc_f, pred_f = full.query(q, k)
    ids_f, sc_f = ids_f.cpu().numpy(), sc_f.cpu().numpy()
    for i in range(B):
        cand = [(s_, id_) for ids_, sc_ in parts for id_, s_ in zip(ids_[i], sc_[i])]
        cand.sort(key=lambda t: (-t[0], t[1]))
        assert [t[1] for t in cand[:k]] == list(ids_f[i])
        assert [t[0] for t in cand[:k]] == list(sc_f[i])
    assert compare(qb, x, a, k, ids_f, sc_f, pred_f.cpu().numpy()).ok()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_worker(rank, world, port, q, fused):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), REMOE_FUSED_COMM=str(fused))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_2512_18674_b200.dist import build_sharded, shard_range
        c = gen.CONFIGS["c2"]
        n, B, k = 50_001, 16, 10
        off, nl = shard_range(n, world, rank)
        x = gen.store_emb(c.store_seed, n, c.dim, off, nl)
        a = gen.store_act(c.store_seed, n, c.layers, c.experts, c.moe_topk, off, nl)
        s = build_sharded(x, a, n, device=rank, max_k=16, max_batch=5)
        assert s.info().fused_exchange == fused, "every rank agreed on the exchange path"
        qb = gen.queries(c.store_seed, c.query_seed, n, c.dim, B, mode=1)
        for _ in range(2):  # chunks of 5 and a repeat: both parity buffers, advancing flags
            ids, sc, pred = s.query(torch.from_numpy(qb.view(np.int16)).cuda(rank), k)
        torch.cuda.synchronize()
        q.put((rank, (ids.cpu().numpy(), sc.cpu().numpy(), pred.cpu().numpy())))
        s.close()
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("fused", [0, 1])
def test_nccl_sharded_query_matches_oracle_and_single_gpu(fused):
    """Real NCCL ranks, one per GPU: the collective exchanges (fused = 0) or the fused
    peer-memory exchange over CUDA IPC / NVLink (fused = 1)."""
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 8)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_nccl_worker, args=(r, world, port, q, fused)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(out[r], str), out[r]
    c = gen.CONFIGS["c2"]
    n, B, k = 50_001, 16, 10
    x = gen.store_emb(c.store_seed, n, c.dim)
    a = gen.store_act(c.store_seed, n, c.layers, c.experts, c.moe_topk)
    qb = gen.queries(c.store_seed, c.query_seed, n, c.dim, B, mode=1)
    ids, sc, pred = out[0]
    assert compare(qb, x, a, k, ids, sc, pred).ok()
    for r in range(1, world):
        for u, v in zip(out[0], out[r]):
            assert np.array_equal(u, v), "every rank must return identical outputs"
    single = remoe.Sps(x, a, max_k=16)
    i1, s1, p1 = single.query(torch.from_numpy(qb.view(np.int16)).cuda(), k)
    assert np.array_equal(i1.cpu().numpy(), ids) and np.array_equal(s1.cpu().numpy(), sc)
    # P = sum of the owners' partials in rank order: a re-association of the world-1 sum
    assert np.abs(p1.cpu().numpy() - pred).max() <= 1e-6
