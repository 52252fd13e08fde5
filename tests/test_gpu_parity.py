"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Sizes the oracle finishes in seconds that still span several tiles / CTAs and a
ragged tail, plus sampled queries at BASELINE's full c3 size in the launch
configuration bench.py times.  Protocol: tests/parity.py.
"""
import numpy as np
import pytest

import gen
import oracle
from parity import compare, log_report, oracle_run, plan_compare, take

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("remoe_lib_built")]

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_18674_b200 as remoe  # noqa: E402

KERNELS = {"stream": remoe.KERNEL_STREAM, "tc": remoe.KERNEL_TC, "pair": remoe.KERNEL_PAIR}


def _store(name, n=None):
    c = gen.CONFIGS[name]
    n = n or c.n
    x = gen.store_emb(c.store_seed, n, c.dim)
    a = gen.store_act(c.store_seed, n, c.layers, c.experts, c.moe_topk)
    return c, x, a


_CACHE = {}


def store(name, n=None):
    key = (name, n)
    if key not in _CACHE:
        _CACHE[key] = _store(name, n)
    return _CACHE[key]


def run(sps, q_bits, k, want_pred=True):
    q = torch.from_numpy(q_bits.view(np.int16)).cuda()
    ids, sc, pred = sps.query(q, k, want_pred)
    torch.cuda.synchronize()
    return (ids.cpu().numpy(), sc.cpu().numpy(), pred.cpu().numpy() if want_pred else None)


def make(x, a, **kw):
    return remoe.Sps(x, a, **kw)


def kernel_available(sps, which):
    try:
        sps.set_kernel(KERNELS[which])
        return True
    except remoe.RemoeError:
        return False


def assert_parity(rep, name=None):
    if name:
        log_report(name, rep)
    assert rep.ok(), "\n".join(rep.failures[:20])


# ------------------------------------------------------------------ tiny: everything, full

@pytest.mark.parametrize("kern", ["stream", "tc", "pair"])
def test_tiny_full(kern):
    c, x, a = store("tiny")
    q = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, c.batch, mode=1)
    s = make(x, a, max_k=32)
    if not kernel_available(s, kern):
        pytest.skip(f"{kern} kernel unavailable")
    ids, sc, pred = run(s, q, c.k)
    rep = compare(q, x, a, c.k, ids, sc, pred, exact_ids=True)
    assert_parity(rep)
    assert s.info().last_scan_kernel == KERNELS[kern]
    # exact copies retrieve their source row first; duplicates are bit-identical
    for i in range(c.batch):
        if i % 8 in (4, 5):
            assert ids[i, 0] == gen.query_source_row(c.query_seed, c.n, i)
        if i % 8 == 7:
            assert np.array_equal(ids[i], ids[i - 1]) and np.array_equal(pred[i], pred[i - 1])
            assert np.array_equal(sc[i], sc[i - 1])


# ------------------------------------------------------------------ c2: batch sweep

_C2Q = {}


def c2_oracle(B, k):
    c, x, a = store("c2")
    key = (B, k)
    if key not in _C2Q:
        q = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, B, mode=1)
        _C2Q[key] = (q, oracle_run(q, x, a, k))
    return _C2Q[key]


@pytest.mark.parametrize("kern", ["stream", "tc", "pair"])
@pytest.mark.parametrize("B", [1, 2, 3, 4, 8, 16, 64, 256])
def test_c2_batch_sweep(kern, B):
    c, x, a = store("c2")
    q_all, o_all = c2_oracle(256, c.k)
    q = q_all[:B]
    o = take(o_all, slice(0, B))
    s = make(x, a, max_k=64)
    if not kernel_available(s, kern):
        pytest.skip(f"{kern} kernel unavailable")
    if kern == "stream" and B > 16:
        pytest.skip("streaming kernel is only used for small batches")
    ids, sc, pred = run(s, q, c.k)
    rep = compare(q, x, a, c.k, ids, sc, pred, oracle_out=o)
    assert_parity(rep, f"c2 B={B} {kern}")
    assert rep.substitutions == 0, "c2 is well separated at k=10: ids must match exactly"


@pytest.mark.parametrize("kern", ["stream", "tc", "pair"])
@pytest.mark.parametrize("k", [1, 2, 5, 16, 32, 64, 128, 256])
def test_c2_k_sweep(kern, k):
    c, x, a = store("c2", 20_000)
    q = gen.queries(c.store_seed, c.query_seed, 20_000, c.dim, 8, mode=1)
    s = make(x, a, max_k=256)
    if not kernel_available(s, kern):
        pytest.skip(f"{kern} kernel unavailable")
    ids, sc, pred = run(s, q, k)
    rep = compare(q, x, a, k, ids, sc, pred)
    assert_parity(rep, f"c2[20k] k={k} {kern}")


# ------------------------------------------------------------------ invariants

@pytest.mark.parametrize("kern", ["stream", "tc", "pair"])
def test_invariants_rerun_batch_order_k1(kern):
    c, x, a = store("c2", 30_000)
    q = gen.queries(c.store_seed, c.query_seed, 30_000, c.dim, 24, mode=1)
    s = make(x, a, max_k=32)
    if not kernel_available(s, kern):
        pytest.skip(f"{kern} kernel unavailable")
    r1 = run(s, q, 10)
    r2 = run(s, q, 10)
    for u, v in zip(r1, r2):
        assert np.array_equal(u, v), "reruns must be bit-identical"
    perm = np.random.default_rng(0).permutation(24)
    rp = run(s, q[perm], 10)
    for u, v in zip(r1, rp):
        assert np.array_equal(u[perm], v), "outputs must be invariant to batch order"
    # k = 1: exact copies return their source with w = 1 -> pred == table row bit-exact
    ids, sc, pred = run(s, q, 1)
    for i in range(24):
        if i % 8 in (4, 5):
            src = gen.query_source_row(c.query_seed, 30_000, i)
            assert ids[i, 0] == src
            assert np.array_equal(pred[i], a[src])
    # convex hull (+-1e-5) and per-layer row sums of the prediction
    ids, sc, pred = r1
    for i in range(24):
        nb = a[ids[i]]
        assert np.all(pred[i] >= nb.min(0) - 1e-5) and np.all(pred[i] <= nb.max(0) + 1e-5)
        np.testing.assert_allclose(pred[i].sum(-1), 1.0, atol=2e-5)


# ------------------------------------------------------------------ edge cases

@pytest.mark.parametrize("kern", ["stream", "tc", "pair"])
@pytest.mark.parametrize("n", [1, 2, 7, 64, 149, 300])
def test_small_stores_k_equals_n(kern, n):
    """Fewer rows than CTAs, k = N returns every row in key order."""
    c, x, a = store("tiny")
    x, a = x[:n].copy(), a[:n].copy()
    q = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, 5, mode=0)
    s = make(x, a, max_k=256)
    if not kernel_available(s, kern):
        pytest.skip(f"{kern} kernel unavailable")
    k = min(n, 256)
    ids, sc, pred = run(s, q, k)
    assert_parity(compare(q, x, a, k, ids, sc, pred))
    for i in range(5):
        assert sorted(ids[i].tolist()) == sorted(set(ids[i].tolist()))


@pytest.mark.parametrize("kern", ["stream", "tc", "pair"])
def test_degenerate_rows(kern):
    """Zero rows score 0; exact duplicate rows tie and the lower id comes first;
    a zero query scores 0 everywhere (sigma keeps it finite)."""
    c, x, a = store("tiny")
    x = x[:500].copy()
    a = a[:500].copy()
    x[3] = 0
    x[100] = x[50]
    x[400] = x[50]
    q = np.stack([x[50], np.zeros_like(x[0]), x[7]])
    s = make(x, a, max_k=16)
    if not kernel_available(s, kern):
        pytest.skip(f"{kern} kernel unavailable")
    ids, sc, pred = run(s, q, 5)
    assert list(ids[0, :3]) == [50, 100, 400] and sc[0, 0] == sc[0, 1] == sc[0, 2]
    assert np.all(sc[1] == 0.0) and list(ids[1]) == [0, 1, 2, 3, 4]
    assert_parity(compare(q, x, a, 5, ids, sc, pred))


@pytest.mark.parametrize("B", [6, 9])
def test_dims_and_table_shapes(B):
    """D at the minimum (8), odd chunk counts (D=40, 776: streaming kernel only), D=4096
    (the streaming kernel's B = 9 takes its 8-query slab, which must be sized to fit shared
    memory; the tensor-core scan a reduced slab), E=1 and E=256."""
    rng = np.random.default_rng(4)
    for D, L, E, n in [(8, 3, 1, 777), (40, 2, 256, 3000), (776, 27, 64, 5000), (4096, 4, 8, 2000)]:
        x = gen.f32_to_bf16_bits(rng.standard_normal((n, D)).astype(np.float32))
        a = rng.random((n, L, E)).astype(np.float32) + 1e-3
        a /= a.sum(-1, keepdims=True)
        q = gen.f32_to_bf16_bits(rng.standard_normal((B, D)).astype(np.float32))
        s = make(x, a, max_k=32)
        for kern in ("stream", "tc", "pair"):
            if not kernel_available(s, kern):
                continue
            ids, sc, pred = run(s, q, 9)
            assert_parity(compare(q, x, a, 9, ids, sc, pred), f"D={D} E={E} B={B} {kern}")
        s.close()


@pytest.mark.parametrize("D", [2048, 3072, 4096])
def test_large_dim_reduced_slabs(D):
    """D > 1536: the tensor-core scan keeps fewer query rows resident (40 at D = 2048, 16 at
    4096) and takes several slabs above that; every kernel and the automatic
    choice match the oracle, with a ragged tail, for batches around the slab size and k on
    both sides of the register top-k (9, 40)."""
    rng = np.random.default_rng(D)
    n = 2000 + 77
    x = gen.f32_to_bf16_bits(rng.standard_normal((n, D)).astype(np.float32))
    a = rng.random((n, 4, 8)).astype(np.float32) + 1e-3
    a /= a.sum(-1, keepdims=True)
    q_all = gen.f32_to_bf16_bits(rng.standard_normal((100, D)).astype(np.float32))
    q_all[5] = x[1234]  # an exact copy
    s = make(x, a, max_k=64)
    for B in (1, 9, 17, 41, 100):
        q = q_all[:B]
        for k in (9, 40):
            s.set_kernel(0)
            ids, sc, pred = run(s, q, k)
            assert s.info().last_scan_kernel == (KERNELS["tc"] if B < 128 else KERNELS["pair"])
            assert_parity(compare(q, x, a, k, ids, sc, pred), f"D={D} B={B} k={k} auto")
            if B > 5:
                assert ids[5, 0] == 1234
            for kern in ("stream", "pair"):
                if not kernel_available(s, kern):
                    continue
                ids, sc, pred = run(s, q, k)
                assert_parity(compare(q, x, a, k, ids, sc, pred), f"D={D} B={B} k={k} {kern}")
    s.close()


def test_pair_lockstep_same_results(monkeypatch):
    """REMOE_PAIR_LOCKSTEP=1 (the CTA-pair scan's query groups wait for each other, DESIGN.md
    §7): only the timing changes -- ids, scores and pred equal the free-running scan bit for
    bit at B = 600 (3 query groups in one launch), repeated (the counters self-reset)."""
    c, x, a = store("c2")
    q = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, 600, mode=1)
    s_free = make(x, a, max_k=16, max_batch=600)
    monkeypatch.setenv("REMOE_PAIR_LOCKSTEP", "1")
    s_lock = make(x, a, max_k=16, max_batch=600)
    r_free = run(s_free, q, 10)
    assert s_free.info().last_scan_kernel == KERNELS["pair"]
    for _ in range(3):
        r_lock = run(s_lock, q, 10)
        for u, v in zip(r_free, r_lock):
            assert np.array_equal(u, v)
    pick = list(range(0, 600, 40))
    assert_parity(compare(q[pick], x, a, 10, r_lock[0][pick], r_lock[1][pick], r_lock[2][pick]),
                  "c2 B=600 pair lockstep (15 sampled)")
    s_free.close()
    s_lock.close()


@pytest.mark.parametrize("D", [8, 40, 776, 1000])
def test_dim_not_multiple_of_64_on_tensor_cores(D):
    """D % 64 != 0 runs on the tensor cores with a zero-padded last K-block (tiled copy and
    query slab padded; TMA zero fill for the CTA-pair scan): the automatic choice is the
    tensor-core scan, and every kernel (the streaming one included) matches the oracle."""
    rng = np.random.default_rng(D)
    n = 1500
    x = gen.f32_to_bf16_bits(rng.standard_normal((n, D)).astype(np.float32))
    a = rng.random((n, 3, 8)).astype(np.float32) + 1e-3
    a /= a.sum(-1, keepdims=True)
    for B in (3, 130):
        q = gen.f32_to_bf16_bits(rng.standard_normal((B, D)).astype(np.float32))
        q[0] = x[7]
        s = make(x, a, max_k=32, max_batch=B)
        ids, sc, pred = run(s, q, 12)
        assert s.info().last_scan_kernel == (KERNELS["tc"] if B < 128 else KERNELS["pair"])
        assert ids[0, 0] == 7
        assert_parity(compare(q, x, a, 12, ids, sc, pred), f"D={D} B={B} auto")
        for kern in ("stream", "tc", "pair"):
            if kernel_available(s, kern):
                r = run(s, q, 12)
                assert_parity(compare(q, x, a, 12, *r), f"D={D} B={B} {kern}")
        s.close()


def test_dim_not_multiple_of_64_seeded():
    """D = 776 on a 40,000-row store: the seeded paths (the padded tiled sample inside the
    resident-slab scan at B = 40; the strided-tensor-map seed scan of the CTA-pair scan at
    B = 200) against the oracle on sampled queries."""
    rng = np.random.default_rng(776)
    n, D = 40_000, 776
    x = gen.f32_to_bf16_bits(rng.standard_normal((n, D)).astype(np.float32))
    a = rng.random((n, 2, 4)).astype(np.float32) + 1e-3
    a /= a.sum(-1, keepdims=True)
    q = gen.f32_to_bf16_bits(rng.standard_normal((200, D)).astype(np.float32))
    q[3] = x[12345]
    s = make(x, a, max_k=32, max_batch=200)
    for B, kern in ((40, "tc"), (200, "pair")):
        ids, sc, pred = run(s, q[:B], 16)
        assert s.info().last_scan_kernel == KERNELS[kern]
        assert ids[3, 0] == 12345
        pick = list(range(0, B, max(1, B // 12)))
        assert_parity(compare(q[pick], x, a, 16, ids[pick], sc[pick], pred[pick]), f"D=776 n=40k B={B} seeded")
    s.close()


def test_chunking_above_max_batch():
    c, x, a = store("c2", 20_000)
    q = gen.queries(c.store_seed, c.query_seed, 20_000, c.dim, 37, mode=1)
    s = make(x, a, max_batch=5, max_k=16)
    ids, sc, pred = run(s, q, 10)
    assert_parity(compare(q, x, a, 10, ids, sc, pred))


def test_errors():
    c, x, a = store("tiny")
    s = make(x, a, max_k=8)
    q = torch.zeros((2, c.dim), dtype=torch.int16, device="cuda")
    with pytest.raises(remoe.RemoeError, match="INVALID_ARG"):
        s.query(q, 9)          # k > max_k
    with pytest.raises(remoe.RemoeError, match="INVALID_ARG"):
        s.query(q, 0)
    s2 = make(x[:4].copy(), a[:4].copy(), max_k=8)
    with pytest.raises(remoe.RemoeError, match="INVALID_ARG"):
        s2.query(q, 5)         # k > N
    ids, sc, pred = s.query(q[:0], 3)  # B == 0: no-op
    assert ids.shape == (0, 3)
    # a query view 2 bytes off a 16-byte boundary: rejected synchronously, not a fault
    qm = torch.zeros(2 * c.dim + 8, dtype=torch.int16, device="cuda")[1:1 + 2 * c.dim].view(2, c.dim)
    with pytest.raises(remoe.RemoeError, match="misaligned"):
        s.query(qm, 3)
    s.sync()
    bad = x.copy()
    bad[5, 3] = 0x7FC0       # NaN
    with pytest.raises(remoe.RemoeError, match="INVALID_ARG"):
        make(bad, a)
    bada = a.copy()
    bada[9, 1, 0] += 0.5     # row no longer sums to 1
    with pytest.raises(remoe.RemoeError, match="INVALID_ARG"):
        make(x, bada)
    with pytest.raises(remoe.RemoeError, match="UNSUPPORTED"):
        make(x, a, max_k=300)


def test_host_path_matches_device_path():
    c, x, a = store("c2", 20_000)
    q = gen.queries(c.store_seed, c.query_seed, 20_000, c.dim, 12, mode=1)
    s = make(x, a, max_batch=8, max_k=16)
    d = run(s, q, 10)
    h = s.query_host(q, 10)
    for u, v in zip(d, h):
        assert np.array_equal(u, v)


def test_host_graph_path_matches_device_path():
    """Pinned host buffers take the cached CUDA-graph replay of remoe_sps_query_host: every
    call re-points the graph's copies at the caller's buffers (two buffer sets, a new
    batch shape, pred on/off, a kernel switch), results bit-identical to the device path."""
    c, x, a = store("c2", 20_000)
    s = make(x, a, max_batch=16, max_k=16)
    L, E = c.layers, c.experts
    for B, k, want_pred, kern in ((12, 10, True, 0), (12, 10, True, 0), (5, 3, True, 0), (5, 3, False, 0),
                                  (12, 10, True, 2), (12, 10, True, 0)):
        q = gen.queries(c.store_seed, c.query_seed + B + k, 20_000, c.dim, B, mode=1)
        s.set_kernel(kern)
        d = run(s, q, k)
        qh = torch.from_numpy(q.view(np.int16)).pin_memory()
        ids = torch.full((B, k), -7, dtype=torch.int64).pin_memory()
        sc = torch.full((B, k), -7.0, dtype=torch.float32).pin_memory()
        pr = torch.full((B, L, E), -7.0, dtype=torch.float32).pin_memory() if want_pred else None
        remoe.remoe_sps_query_host(s.handle, qh, B, k, ids, sc, pr)
        assert np.array_equal(ids.numpy(), d[0]) and np.array_equal(sc.numpy(), d[1])
        if want_pred:
            assert np.array_equal(pr.numpy(), d[2])
    s.set_kernel(0)


# ------------------------------------------------------------------ S8 expert plan

def test_expert_plan_vs_oracle():
    c, x, a = store("c2", 20_000)
    q = gen.queries(c.store_seed, c.query_seed, 20_000, c.dim, 16, mode=1)
    s = make(x, a, max_k=16)
    ids, sc, pred = run(s, q, 10)
    pt = torch.from_numpy(pred).cuda()
    for n_cold in (0, 1, 13, 32, 63, 64):
        m = s.plan(pt, n_cold).cpu().numpy()
        assert not plan_compare(pred.astype(np.float64), m, n_cold)
        assert np.all(m.sum(-1) == n_cold)
    # SPEC S:434 worked example, and ties -> lower index goes cold first
    p = torch.tensor([[[0.4, 0.3, 0.2, 0.1]], [[0.25, 0.25, 0.25, 0.25]]], device="cuda")
    m = s.plan(p, 2).cpu().numpy()
    assert list(m[0, 0]) == [0, 0, 1, 1] and list(m[1, 0]) == [1, 1, 0, 0]


# ------------------------------------------------------------------ full-size sampled parity

_C3O = {}


def c3_oracle(B, k):
    """The oracle on the c3 bench batch (fresh cluster members, mode 0 as bench.py times it)
    and on the correctness mix (mode 1)."""
    c, x, a = store("c3")
    key = (B, k)
    if key not in _C3O:
        q = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, B, mode=0)
        _C3O[key] = (q, oracle_run(q, x, a, k))
    return _C3O[key]


@pytest.mark.parametrize("kern", ["tc", "stream", "pair"])
def test_c3_full_size_bench_batch(kern):
    """BASELINE c3 (1M x 1024, 24x60, k = 16) at bench.py's batch (B = 64 fresh cluster
    members, the launch configuration bench.py times): ALL 64 queries against the oracle
    (tensor-core and CTA-pair scans; the streaming kernel on 8 of them)."""
    c, x, a = store("c3")
    q, o = c3_oracle(64, c.k)
    B = 64 if kern != "stream" else 8
    s = make(x, a, max_k=c.k, max_batch=256)
    if not kernel_available(s, kern):
        pytest.skip(f"{kern} kernel unavailable")
    ids, sc, pred = run(s, q[:B], c.k)
    rep = compare(q[:B], x, a, c.k, ids, sc, pred, oracle_out=take(o, slice(0, B)))
    assert_parity(rep, f"c3 B={B} {kern} (bench batch, all queries)")
    s.close()


def test_c3_full_size_mixed_queries():
    """c3 with the correctness query mix (fresh, exact copies, perturbed copies,
    duplicates) at B = 64: 16 sampled queries; copies retrieve their source."""
    c, x, a = store("c3")
    B = 64
    q = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, B, mode=1)
    s = make(x, a, max_k=c.k, max_batch=256)
    ids, sc, pred = run(s, q, c.k)
    pick = list(range(0, 64, 4))
    rep = compare(q[pick], x, a, c.k, ids[pick], sc[pick], pred[pick])
    assert_parity(rep, "c3 B=64 tc (mixed queries, 16 sampled)")
    for i in range(B):
        if i % 8 in (4, 5):
            assert ids[i, 0] == gen.query_source_row(c.query_seed, c.n, i)
        if i % 8 == 7:
            assert np.array_equal(ids[i], ids[i - 1]) and np.array_equal(pred[i], pred[i - 1])
    s.close()


def test_c3_past_one_slab_auto_pair():
    """c3 (a shard of >= 16 x 256 rows per SM): a batch past one resident slab (B = 96) goes
    to the CTA-pair scan automatically (kPairLargeUnits); the pair scan and
    the two-slab resident scan (forced) both match the oracle on 12 sampled queries."""
    c, x, a = store("c3")
    B = 96
    q = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, B, mode=1)
    s = make(x, a, max_k=c.k, max_batch=256)
    ids, sc, pred = run(s, q, c.k)
    assert s.info().last_scan_kernel == KERNELS["pair"]
    pick = list(range(0, B, 8))
    o = oracle_run(q[pick], x, a, c.k)
    assert_parity(compare(q[pick], x, a, c.k, ids[pick], sc[pick], pred[pick], oracle_out=o),
                  "c3 B=96 auto (pair, 12 sampled)")
    s.set_kernel(KERNELS["tc"])
    ids2, sc2, pred2 = run(s, q, c.k)
    assert s.info().last_scan_kernel == KERNELS["tc"]
    assert_parity(compare(q[pick], x, a, c.k, ids2[pick], sc2[pick], pred2[pick], oracle_out=o),
                  "c3 B=96 tc two slabs (12 sampled)")
    s.close()


# ------------------------------------------------------------------ BASELINE c4 and c5 (sampled)

def test_c4_full_size_sampled():
    """BASELINE c4: 10M x 1024, Mixtral 32x8 table, k = 32, at B = 1 (single-query latency)
    and B = 1024 (throughput), on one GPU; 1 + 4 sampled queries checked against the oracle."""
    c = gen.CONFIGS["c4"]
    x = gen.store_emb(c.store_seed, c.n, c.dim)
    a = gen.store_act(c.store_seed, c.n, c.layers, c.experts, c.moe_topk)
    q = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, 1024, mode=1)
    s = make(x, a, max_k=32, max_batch=1024)
    for B, pick in ((1, [0]), (1024, [4, 517, 770, 1023])):
        ids, sc, pred = run(s, q[:B], 32)
        rep = compare(q[pick], x, a, 32, ids[pick], sc[pick], pred[pick])
        assert_parity(rep, f"c4 B={B} ({len(pick)} sampled)")
    s.close()


@pytest.mark.parametrize("k", [1, 64, 128])
def test_c5_sweep_corners_sampled(k):
    """BASELINE c5 corners on the c3 store: B = 4096 (internal chunks of max_batch) and
    k in {1, 64, 128}; 16 sampled queries per corner (spread over the 4 chunks) vs the oracle."""
    c, x, a = store("c3")
    q = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, 4096, mode=1)
    s = make(x, a, max_k=128, max_batch=1024)
    ids, sc, pred = run(s, q, k)
    pick = [0, 5, 255, 256, 511, 1023, 1024, 1500, 2047, 2048, 2600, 3071, 3072, 3500, 4094, 4095]
    assert_parity(compare(q[pick], x, a, k, ids[pick], sc[pick], pred[pick]),
                  f"c5 B=4096 k={k} (16 sampled)")
    # identical queries (i % 8 == 7 duplicates i - 1) across chunk boundaries
    for i in (7, 1031, 4095):
        assert np.array_equal(ids[i], ids[i - 1]) and np.array_equal(pred[i], pred[i - 1])
    s.close()


@pytest.mark.parametrize("kern", ["tc", "pair"])
@pytest.mark.parametrize("k", [33, 64, 128, 256])
def test_seeded_large_k(kern, k):
    """k > 32 seeds the shared thresholds from a strided sample (every 16th row, scanned
    with the register top-32 per state): results must
    still equal the oracle's exactly, including when the sample holds the winners."""
    c, x, a = store("c2", 200_000)
    q = gen.queries(c.store_seed, c.query_seed, 200_000, c.dim, 40, mode=1)
    q[3] = x[16 * 7]          # an exact copy of a sampled row
    q[4] = x[16 * 7 + 1]      # ... and of an unsampled neighbour
    s = make(x, a, max_k=256)
    if not kernel_available(s, kern):
        pytest.skip(f"{kern} kernel unavailable")
    ids, sc, pred = run(s, q, k)
    assert_parity(compare(q, x, a, k, ids, sc, pred), f"c2[200k] seeded k={k} {kern}")
    assert ids[3, 0] == 16 * 7 and ids[4, 0] == 16 * 7 + 1


# ------------------------------------------------------------------ randomized shapes

@pytest.mark.parametrize("case", range(48))
def test_random_shapes_vs_oracle(case):
    """Seeded random shapes (store size, D incl. non-multiples of 64 and > 1536, batch across
    the slab / CTA-pair thresholds, k across the register / buffer top-k boundary, table
    shape), automatic kernel choice plus one forced kernel each, against the oracle."""
    rng = np.random.default_rng(1000 + case)
    n = int(rng.choice([1, 3, 127, 129, 700, 2500, 6000]))
    D = int(rng.choice([8, 40, 64, 192, 768, 1024, 2048]))
    B = int(rng.choice([1, 5, 16, 63, 64, 65, 130, 257]))
    k = int(min(n, rng.choice([1, 2, 7, 16, 31, 33, 64, 100])))
    L, E = int(rng.integers(1, 6)), int(rng.choice([1, 3, 8, 60]))
    x = gen.f32_to_bf16_bits(rng.standard_normal((n, D)).astype(np.float32))
    if n > 3:
        x[n // 2] = x[n // 3]  # an exact duplicate (tie: lower id first)
    a = rng.random((n, L, E)).astype(np.float32) + 1e-3
    a /= a.sum(-1, keepdims=True)
    q = gen.f32_to_bf16_bits(rng.standard_normal((B, D)).astype(np.float32))
    q[0] = x[n - 1]  # an exact copy
    mb = int(max(1, B if case % 4 else rng.integers(1, B + 1)))  # every 4th case: internal chunks
    s = make(x, a, max_k=max(k, 1), max_batch=mb)
    ids, sc, pred = run(s, q, k)
    assert_parity(compare(q, x, a, k, ids, sc, pred),
                  f"random case {case}: n={n} D={D} B={B} (max_batch {mb}) k={k} L={L} E={E} auto")
    forced = ["stream", "tc", "pair"][case % 3]
    if kernel_available(s, forced):
        ids2, sc2, pred2 = run(s, q, k)
        assert_parity(compare(q, x, a, k, ids2, sc2, pred2), f"random case {case}: {forced}")
    s.close()
