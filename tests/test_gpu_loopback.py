"""The multi-rank path of runtime.cu on ONE GPU: a loopback group of G handles (one per
row shard) runs exactly the stage functions an NCCL rank runs -- S1-S4 per shard, the
all-gather of the local top-k keys, the cross-rank merge (S5), the owner-side partial
prediction (S6 + partial S7) and its exchange (all-gather of partials, or the all-to-all
of query slices + broadcast) and the fixed rank-order sum -- with device copies standing
in for the NCCL collectives (include/remoe.h "Loopback groups").

Checked against the oracle (tests/parity.py protocol), against the single-handle
world == 1 result (ids/scores bit-identical, pred within fp32 re-association), and
across ranks (every rank's outputs bit-identical).
"""
import numpy as np
import pytest

import gen
from parity import compare, log_report, oracle_run, take

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("remoe_lib_built")]
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_18674_b200 as remoe  # noqa: E402
from paper_2512_18674_b200.dist import shard_range  # noqa: E402

_STORE = {}


def store(n, name="c2"):
    key = (name, n)
    if key not in _STORE:
        c = gen.CONFIGS[name]
        _STORE[key] = (c, gen.store_emb(c.store_seed, n, c.dim), gen.store_act(c.store_seed, n, c.layers,
                                                                                c.experts, c.moe_topk))
    return _STORE[key]


def group(x, a, G, **kw):
    n = x.shape[0]
    shards, acts = [], []
    for r in range(G):
        off, nl = shard_range(n, G, r)
        shards.append(np.ascontiguousarray(x[off:off + nl]))
        acts.append(np.ascontiguousarray(a[off:off + nl]))
    return remoe.LoopbackGroup(shards, acts, n, **kw)


def run_group(g, qb, k, want_pred=True):
    q = torch.from_numpy(qb.view(np.int16)).cuda()
    ids, sc, pred = g.query(q, k, want_pred)
    torch.cuda.synchronize()
    return ([t.cpu().numpy() for t in ids], [t.cpu().numpy() for t in sc],
            [t.cpu().numpy() for t in pred] if want_pred else None)


def run_single(x, a, qb, k, **kw):
    s = remoe.Sps(x, a, **kw)
    q = torch.from_numpy(qb.view(np.int16)).cuda()
    ids, sc, pred = s.query(q, k)
    torch.cuda.synchronize()
    out = ids.cpu().numpy(), sc.cpu().numpy(), pred.cpu().numpy()
    s.close()
    return out


def check_ranks_identical(ids, sc, pred):
    for r in range(1, len(ids)):
        assert np.array_equal(ids[r], ids[0]) and np.array_equal(sc[r], sc[0]), f"rank {r} ids/scores differ"
        if pred is not None:
            assert np.array_equal(pred[r], pred[0]), f"rank {r} prediction differs"


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("xchg", ["allgather", "alltoall"])
def test_loopback_matches_oracle_and_world1(G, xchg, monkeypatch):
    """c2-shaped store (50,001 rows, uneven shards), mixed queries, k = 10: the G-rank
    result equals the oracle, is identical on every rank, and equals world == 1 (ids and
    scores bit-exact, pred within 1e-6).  `alltoall` forces the large-batch exchange
    (REMOE_XCHG_AG_MAX=0 at build): slices of 13 queries over G ranks, uneven."""
    if xchg == "alltoall":
        monkeypatch.setenv("REMOE_XCHG_AG_MAX", "0")
    c, x, a = store(50_001)
    B, k = 13, 10
    qb = gen.queries(c.store_seed, c.query_seed, 50_001, c.dim, B, mode=1)
    g = group(x, a, G, max_k=16)
    ids, sc, pred = run_group(g, qb, k)
    g.close()
    check_ranks_identical(ids, sc, pred)
    rep = compare(qb, x, a, k, ids[0], sc[0], pred[0])
    log_report(f"loopback G={G} {xchg} c2[50k] B={B} k={k}", rep)
    assert rep.ok(), "\n".join(rep.failures[:20])
    i1, s1, p1 = run_single(x, a, qb, k, max_k=16)
    assert np.array_equal(ids[0], i1) and np.array_equal(sc[0], s1), "world > 1 ids/scores == world 1"
    assert np.abs(pred[0] - p1).max() <= 1e-6


def test_loopback_batch_smaller_than_world_and_chunks(monkeypatch):
    """All-to-all layout with B < G (empty slices) and internal chunking (max_batch 5)."""
    monkeypatch.setenv("REMOE_XCHG_AG_MAX", "0")
    c, x, a = store(20_000)
    qb = gen.queries(c.store_seed, c.query_seed, 20_000, c.dim, 12, mode=1)
    g = group(x, a, 8, max_k=16, max_batch=5)
    for B in (2, 12):
        ids, sc, pred = run_group(g, qb[:B], 7)
        check_ranks_identical(ids, sc, pred)
        rep = compare(qb[:B], x, a, 7, ids[0], sc[0], pred[0])
        log_report(f"loopback G=8 alltoall B={B} max_batch=5", rep)
        assert rep.ok(), "\n".join(rep.failures[:20])
    g.close()


def test_loopback_shards_smaller_than_k():
    """k larger than every shard (7 rows per rank at G = 8): each rank contributes its
    rows plus sentinels; the merged top-k is the exact global one (k = N: every row)."""
    c, x, a = store(1_000, "tiny")
    x, a = x[:57].copy(), a[:57].copy()
    qb = gen.queries(c.store_seed, c.query_seed, 1_000, c.dim, 5, mode=0)
    g = group(x, a, 8, max_k=64)
    for k in (10, 57):
        ids, sc, pred = run_group(g, qb, k)
        check_ranks_identical(ids, sc, pred)
        rep = compare(qb, x, a, k, ids[0], sc[0], pred[0])
        assert rep.ok(), "\n".join(rep.failures[:20])
    g.close()


@pytest.mark.parametrize("k", [16, 64])
def test_loopback_c3_shards_bench_batch(k):
    """BASELINE c3 (1M x 1024, 24 x 60) over 8 loopback ranks at the bench batch B = 64:
    the per-shard scans use the seeded tensor-core path (125k-row shards); 16 queries
    checked against the oracle, every rank identical, ids/scores == world 1."""
    c, x, a = store(1_000_000, "c3")
    qb = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, 64, mode=0)
    g = group(x, a, 8, max_k=64, max_batch=64)
    ids, sc, pred = run_group(g, qb, k)
    g.close()
    check_ranks_identical(ids, sc, pred)
    pick = list(range(0, 64, 4))
    o = oracle_run(qb[pick], x, a, k)
    rep = compare(qb[pick], x, a, k, ids[0][pick], sc[0][pick], pred[0][pick], oracle_out=o)
    log_report(f"loopback G=8 c3 B=64 k={k} (16 sampled)", rep)
    assert rep.ok(), "\n".join(rep.failures[:20])
    i1, s1, p1 = run_single(x, a, qb, k, max_k=64, max_batch=64)
    assert np.array_equal(ids[0], i1) and np.array_equal(sc[0], s1)
    assert np.abs(pred[0] - p1).max() <= 1e-6


def test_loopback_pair_scan_and_no_pred():
    """B = 300 crosses the CTA-pair threshold on every shard; pred = NULL skips S6-S7."""
    c, x, a = store(100_000)
    qb = gen.queries(c.store_seed, c.query_seed, 100_000, c.dim, 300, mode=1)
    g = group(x, a, 4, max_k=16, max_batch=512)
    ids, sc, _ = run_group(g, qb, 10, want_pred=False)
    check_ranks_identical(ids, sc, None)
    assert g.ranks[0].info().last_scan_kernel == remoe.KERNEL_PAIR
    pick = list(range(0, 300, 20))
    o = oracle_run(qb[pick], x, a, 10, want_pred=False)
    rep = compare(qb[pick], x, a, 10, ids[0][pick], sc[0][pick], None, oracle_out=o)
    assert rep.ok(), "\n".join(rep.failures[:20])
    g.close()


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("xchg", ["allgather", "alltoall"])
def test_loopback_fused_exchange(G, xchg, monkeypatch):
    """REMOE_FUSED_COMM=1: the exchanges run as peer stores inside the merge kernels (the
    S4 merge writes every rank's gathered[parity][rank], the S5 merge every rank's partial
    slot, each last CTA raises its flag; the consumers wait on the flags) -- no copies.
    Several chunks (max_batch 5 over B = 13) exercise both parity buffers and the flag
    sequence; results equal the collective path bit for bit, the oracle, and world 1."""
    if xchg == "alltoall":
        monkeypatch.setenv("REMOE_XCHG_AG_MAX", "0")
    c, x, a = store(50_001)
    B, k = 13, 10
    qb = gen.queries(c.store_seed, c.query_seed, 50_001, c.dim, B, mode=1)
    g0 = group(x, a, G, max_k=16, max_batch=5)
    ref = run_group(g0, qb, k)
    assert g0.ranks[0].info().fused_exchange == 0
    g0.close()
    monkeypatch.setenv("REMOE_FUSED_COMM", "1")
    g = group(x, a, G, max_k=16, max_batch=5)
    for rep_i in range(3):  # repeated queries: the flag sequence keeps advancing
        ids, sc, pred = run_group(g, qb, k)
        assert g.ranks[0].info().fused_exchange == 1
        check_ranks_identical(ids, sc, pred)
        for r in range(G):
            assert np.array_equal(ids[r], ref[0][r]) and np.array_equal(sc[r], ref[1][r])
            assert np.array_equal(pred[r], ref[2][r]), "fused exchange == collective exchange, bit for bit"
    ids2, sc2, _ = run_group(g, qb, k, want_pred=False)  # no prediction: exchange 1 only
    assert np.array_equal(ids2[0], ids[0]) and np.array_equal(sc2[0], sc[0])
    g.close()
    rep = compare(qb, x, a, k, ids[0], sc[0], pred[0])
    log_report(f"loopback fused G={G} {xchg} c2[50k] B={B} k={k}", rep)
    assert rep.ok(), "\n".join(rep.failures[:20])
    i1, s1, p1 = run_single(x, a, qb, k, max_k=16)
    assert np.array_equal(ids[0], i1) and np.array_equal(sc[0], s1)
    assert np.abs(pred[0] - p1).max() <= 1e-6


@pytest.mark.parametrize("G", [2, 8])
def test_loopback_fused_graph_replays(G, monkeypatch):
    """Fused exchange with B <= max_batch: the whole G-rank query is captured once as a CUDA
    graph and replayed; the chunk sequence numbers live on the device (k_seq_bump), so
    replays alternate the double-buffer parity and keep advancing the flags.  Five replays
    with the same buffers and one capture with new buffers all equal the collective path
    bit for bit (ids, scores, pred); without pred the graph is the exchange-1 half."""
    c, x, a = store(50_001)
    B, k = 13, 10
    qb = gen.queries(c.store_seed, c.query_seed, 50_001, c.dim, B, mode=1)
    g0 = group(x, a, G, max_k=16, max_batch=16)
    ref = run_group(g0, qb, k)
    g0.close()
    monkeypatch.setenv("REMOE_FUSED_COMM", "1")
    g = group(x, a, G, max_k=16, max_batch=16)
    q = torch.from_numpy(qb.view(np.int16)).cuda()
    dev_ids = [torch.empty((B, k), dtype=torch.int64, device="cuda") for _ in range(G)]
    dev_sc = [torch.empty((B, k), dtype=torch.float32, device="cuda") for _ in range(G)]
    dev_pred = [torch.empty((B, c.layers, c.experts), dtype=torch.float32, device="cuda") for _ in range(G)]
    for rep in range(6):  # the first call captures, the next five replay (same buffers)
        for t in dev_ids + dev_sc + dev_pred:
            t.zero_()
        remoe.remoe_sps_query_group(g.group, q, B, k, dev_ids, dev_sc, dev_pred)
        torch.cuda.synchronize()
        ids = [t.cpu().numpy() for t in dev_ids]
        sc = [t.cpu().numpy() for t in dev_sc]
        pred = [t.cpu().numpy() for t in dev_pred]
        for r in range(G):
            assert np.array_equal(ids[r], ref[0][r]) and np.array_equal(sc[r], ref[1][r]), f"replay {rep} rank {r}"
            assert np.array_equal(pred[r], ref[2][r]), f"replay {rep} rank {r}: pred"
    ids2, sc2, _ = run_group(g, qb, k, want_pred=False)
    for r in range(G):
        assert np.array_equal(ids2[r], ref[0][r]) and np.array_equal(sc2[r], ref[1][r])
    assert g.ranks[0].info().fused_exchange == 1
    g.close()


def test_loopback_errors():
    c, x, a = store(1_000, "tiny")
    gid = remoe.remoe_loopback_group_create(2)
    off, n = shard_range(1_000, 2, 0)
    s0 = remoe.Sps(x[off:off + n].copy(), a[off:off + n].copy(), rank=0, world=2, global_offset=off,
                   loopback_group=gid, max_k=8)
    q = torch.zeros((1, c.dim), dtype=torch.int16, device="cuda")
    ids = [torch.empty((1, 3), dtype=torch.int64, device="cuda") for _ in range(2)]
    sc = [torch.empty((1, 3), dtype=torch.float32, device="cuda") for _ in range(2)]
    with pytest.raises(remoe.RemoeError, match="STATE"):
        remoe.remoe_sps_query_group(gid, q, 1, 3, ids, sc)       # rank 1 missing
    with pytest.raises(remoe.RemoeError, match="STATE"):
        s0.query(q, 3)                                           # members query as a group
    with pytest.raises(remoe.RemoeError, match="STATE"):
        remoe.Sps(x[:10].copy(), a[:10].copy(), rank=0, world=2, loopback_group=gid)  # rank taken
    with pytest.raises(remoe.RemoeError, match="STATE"):
        remoe.remoe_loopback_group_destroy(gid)                  # members still built
    s0.close()
    remoe.remoe_loopback_group_destroy(gid)


@pytest.mark.parametrize("case", range(12))
def test_loopback_random(case, monkeypatch):
    """Seeded random multi-rank cases: G 2-8 uneven shards (some smaller than k), D, B, k,
    chunking, the fused or the collective exchange (half each), both exchange layouts;
    against the oracle and across ranks."""
    rng = np.random.default_rng(500 + case)
    G = int(rng.integers(2, 9))
    n = int(rng.choice([G * 3, 500, 4000, 20000]))
    D = int(rng.choice([64, 256, 768]))
    B = int(rng.choice([1, 7, 40, 130]))
    k = int(min(n, rng.choice([1, 5, 16, 40])))
    mb = int(B if case % 3 else max(1, B // 3))
    if case % 2:
        monkeypatch.setenv("REMOE_FUSED_COMM", "1")
    if case % 5 == 0:
        monkeypatch.setenv("REMOE_XCHG_AG_MAX", "0")
    x = gen.f32_to_bf16_bits(rng.standard_normal((n, D)).astype(np.float32))
    a = rng.random((n, 3, 8)).astype(np.float32) + 1e-3
    a /= a.sum(-1, keepdims=True)
    qb = gen.f32_to_bf16_bits(rng.standard_normal((B, D)).astype(np.float32))
    g = group(x, a, G, max_k=max(k, 1), max_batch=mb)
    for _ in range(2):  # a second query: replays / advancing sequence numbers
        ids, sc, pred = run_group(g, qb, k)
    assert g.ranks[0].info().fused_exchange == (case % 2)
    g.close()
    check_ranks_identical(ids, sc, pred)
    rep = compare(qb, x, a, k, ids[0], sc[0], pred[0])
    log_report(f"loopback random {case}: G={G} n={n} D={D} B={B} mb={mb} k={k} fused={case % 2}", rep)
    assert rep.ok(), "\n".join(rep.failures[:20])
