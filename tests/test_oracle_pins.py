"""Pins for the oracle (CPU only).  Each test ties an oracle function to something
other than itself: the paper's literal Eq. 11, hand-worked closed forms, textbook
or library routines (scipy, Python's sort), and invariants.  A plausible mistake
in any oracle step (dropped term, wrong sign, wrong sigma placement, transposed
operand, wrong tie rule) fails at least one of these.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy.spatial.distance import cosine as scipy_cosine
from scipy.special import softmax as scipy_softmax

import gen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SIGMA = oracle.SIGMA


def _h1():
    with open(os.path.join(GOLD, "h1.json")) as f:
        return json.load(f)


# ---------------------------------------------------------------- Eq. 11 (step 3)

def test_eq11_literal_gram_equals_reduced_form():
    """O0 (literal Eq. 11 Gram/ownership-vector route) equals the
    oracle's reduced score on summed normalised token rows to 1e-12."""
    rng = np.random.default_rng(11)
    for _ in range(40):
        n1, n2, d = rng.integers(1, 8), rng.integers(1, 8), int(rng.choice([4, 16, 33]))
        t1 = rng.standard_normal((n1, d))
        t2 = rng.standard_normal((n2, d))
        lit = oracle.scs_gram(t1, t2, SIGMA)
        a = oracle.prompt_vector(t1)[None]
        b = oracle.prompt_vector(t2)[None]
        act = np.full((1, 1, 1), 1.0, np.float32)
        _, sc, _ = oracle.sps_f64(a, b, act, 1)
        assert abs(sc[0, 0] - lit) <= 1e-12
        # symmetry of Eq. 11
        assert abs(oracle.scs_gram(t2, t1, SIGMA) - lit) <= 1e-12


def test_eq11_literal_special_cases():
    """SCS(p, p) = 1 within 1e-5; orthogonal single tokens -> 0."""
    rng = np.random.default_rng(3)
    p = rng.standard_normal((5, 8))
    assert abs(oracle.scs_gram(p, p) - 1.0) <= 1e-5
    e1 = np.array([[1.0, 0, 0]])
    e2 = np.array([[0, 1.0, 0]])
    assert abs(oracle.scs_gram(e1, e2)) <= 1e-12


def test_scores_closed_forms():
    """self -> |x|^2/(|x|^2+s); antiparallel -> negative of that; orthogonal -> 0;
    zero vector -> 0 (sigma keeps the denominator positive)."""
    x = np.array([[3.0, 4.0, 0, 0], [-3.0, -4.0, 0, 0], [0, 0, 2.0, 0], [0, 0, 0, 0]])
    q = np.array([[3.0, 4.0, 0, 0]])
    s = oracle.scores(gen.f32_to_bf16_bits(q), gen.f32_to_bf16_bits(x))[0]
    assert s[0] == 25.0 / (25.0 + SIGMA)
    assert s[1] == -25.0 / (25.0 + SIGMA)
    assert s[2] == 0.0
    assert s[3] == 0.0


def test_scores_vs_scipy_cosine():
    """Library routine: with sigma -> 0 the score is the textbook cosine; the
    sigma term moves it by at most sigma/(|q||x|)."""
    c = gen.CONFIGS["tiny"]
    x = gen.store_emb(c.store_seed, c.n, c.dim)[:200]
    q = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, 4, mode=1)
    s = oracle.scores(q, x)
    xf = gen.bf16_bits_to_f32(x).astype(np.float64)
    qf = gen.bf16_bits_to_f32(q).astype(np.float64)
    for i in range(q.shape[0]):
        for j in range(0, 200, 7):
            cos = 1.0 - scipy_cosine(qf[i], xf[j])
            bound = SIGMA / (np.linalg.norm(qf[i]) * np.linalg.norm(xf[j])) + 1e-13
            assert abs(s[i, j] - cos) <= bound


# ---------------------------------------------------------------- H1 hand example

@pytest.mark.parametrize("path", ["f64", "bf16"])
def test_h1_hand_example(path):
    h = _h1()
    x = np.array(h["store"], np.float64)
    q = np.array([h["query"]], np.float64)
    act = np.array(h["act"], np.float32)
    # closed forms (exact up to one rounding each)
    s = h["sigma"]
    closed = [1 / (1 + s), 0.0, 1 / (math.sqrt(2) + s), -1 / (1 + s), 2 / (2 + s), 0.5 / (1 + s)]
    full = oracle.scores(gen.f32_to_bf16_bits(q), gen.f32_to_bf16_bits(x))[0]
    np.testing.assert_allclose(full, closed, rtol=0, atol=1e-15)
    np.testing.assert_allclose(full, h["scores"], rtol=0, atol=5e-9)
    for k in (1, 2, 3, 6):
        if path == "f64":
            ids, sc, pred = oracle.sps_f64(q, x, act, k)
        else:
            ids, sc, pred = oracle.sps(gen.f32_to_bf16_bits(q), gen.f32_to_bf16_bits(x), act, k)
        assert list(ids[0]) == h["order"][:k]
        key = f"k{k}"
        if key in h:
            w = oracle.softmax(sc[0])
            np.testing.assert_allclose(w, h[key]["weights"], rtol=0, atol=5e-9)
            np.testing.assert_allclose(pred[0], h[key]["pred"], rtol=0, atol=5e-9)
    # sigma -> 0 limit: x0 and x4 tie at 1 and the lower id wins (reading R5)
    ids, _, _ = oracle.sps_f64(q, x, act, 6, sigma=1e-300)
    assert list(ids[0]) == h["order_sigma_to_zero"]


# ---------------------------------------------------------------- selection (step 4)

def test_select_matches_python_sort_with_ties():
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 33, 64):
        s = rng.integers(-3, 4, size=n).astype(np.float64) / 4.0   # many exact ties
        for k in {1, min(3, n), n}:
            ids, top = oracle.select(s, k, id_offset=100)
            ref = sorted(range(n), key=lambda j: (-s[j], j))[:k]
            assert list(ids) == [100 + j for j in ref]
            assert list(top) == [s[j] for j in ref]


def test_select_rejects_k_above_n():
    """alpha exceeding history size is an error."""
    with pytest.raises(ValueError):
        oracle.select(np.zeros(4), 5)


def test_sps_permutation_invariance_and_duplicates():
    """Permuting store rows permutes ids; an exact duplicate row ranks right after
    its lower-id twin (equal scores, reading R5)."""
    c = gen.CONFIGS["tiny"]
    x = gen.store_emb(c.store_seed, c.n, c.dim)[:64].copy()
    x[40] = x[10]
    act = gen.store_act(c.store_seed, c.n, 2, 4, 2)[:64]
    q = x[10:11].copy()
    ids, sc, _ = oracle.sps(q, x, act, 5)
    assert ids[0, 0] == 10 and ids[0, 1] == 40 and sc[0, 0] == sc[0, 1]
    perm = np.random.default_rng(1).permutation(64)
    ids2, sc2, _ = oracle.sps(q, x[perm], act[perm], 5)
    inv = np.argsort(perm)
    mapped = perm[ids2[0]]
    assert set(mapped[:2]) == {10, 40}
    np.testing.assert_array_equal(sc2, sc)
    assert inv[10] in ids2[0]


# ---------------------------------------------------------------- weights (step 5)

def test_softmax_vs_scipy_and_printed_example():
    rng = np.random.default_rng(2)
    for k in (1, 2, 5, 32, 128):
        s = rng.uniform(-1, 1, size=k)
        for T in (1.0, 0.5, 3.0):
            np.testing.assert_allclose(oracle.softmax(s, T), scipy_softmax(s / T), rtol=1e-13, atol=0)
    # SPEC S:240 three-neighbour example, re-derived: softmax{0.9,0.5,0.1}
    np.testing.assert_allclose(oracle.softmax([0.9, 0.5, 0.1]),
                               [0.471776, 0.316241, 0.211983], atol=5e-7)
    assert list(oracle.softmax([0.7])) == [1.0]


# ---------------------------------------------------------------- prediction (step 6)

def test_predict_singleton_mean_hull_rowsum():
    c = gen.CONFIGS["c2"]
    act = gen.store_act(c.store_seed, c.n, c.layers, c.experts, c.moe_topk, 0, 50)
    # k = 1: w = 1 exactly, prediction is the neighbour's matrix
    p = oracle.predict([7], oracle.softmax([0.3]), act)
    np.testing.assert_array_equal(p, act[7].astype(np.float64))
    # equal scores: element-wise mean
    ids = [3, 9, 21, 40]
    p = oracle.predict(ids, oracle.softmax([0.5] * 4), act)
    np.testing.assert_allclose(p, act[ids].astype(np.float64).mean(axis=0), rtol=0, atol=1e-15)
    # convex hull and row sums (rows of the table sum to 1 up to fp32 rounding)
    w = oracle.softmax([0.9, 0.8, 0.75, 0.6])
    p = oracle.predict(ids, w, act)
    lo = act[ids].min(axis=0)
    hi = act[ids].max(axis=0)
    assert np.all(p >= lo - 1e-15) and np.all(p <= hi + 1e-15)
    rows = act[ids].astype(np.float64).sum(axis=-1)  # [k, L]
    np.testing.assert_allclose(p.sum(axis=-1), (w[:, None] * rows).sum(axis=0), atol=1e-13)


# ---------------------------------------------------------------- plan (step 7)

def test_plan_spec_example_and_extremes():
    """K=4, s~ = [0.4, 0.3, 0.2, 0.1], n_cold = 2 -> experts {3, 2} remote."""
    m = oracle.plan(np.array([[[0.4, 0.3, 0.2, 0.1]]]), 2)
    assert list(m[0, 0]) == [0, 0, 1, 1]
    assert oracle.plan(np.array([[[0.4, 0.3, 0.2, 0.1]]]), 0).sum() == 0
    assert oracle.plan(np.array([[[0.4, 0.3, 0.2, 0.1]]]), 4).sum() == 4
    with pytest.raises(ValueError):
        oracle.plan(np.zeros((1, 1, 4)), 5)


def test_plan_minimises_utility_exhaustively():
    """R_l = argmin over |R_l| = bK_l of sum u.  Exhaustive check for
    E <= 9, ties resolved toward lower expert index (reading R12)."""
    rng = np.random.default_rng(8)
    for _ in range(60):
        E = int(rng.integers(1, 10))
        v = rng.integers(0, 4, size=E) / 8.0
        for n_cold in range(E + 1):
            m = oracle.plan(v[None, None], n_cold)[0, 0]
            chosen = [e for e in range(E) if m[e]]
            best = min(sum(v[list(c)]) for c in itertools.combinations(range(E), n_cold))
            assert len(chosen) == n_cold and abs(sum(v[chosen]) - best) <= 1e-15
            assert chosen == sorted(sorted(range(E), key=lambda e: (v[e], e))[:n_cold])


# ---------------------------------------------------------------- whole path vs library routines

def test_whole_path_vs_numpy_scipy_bruteforce():
    """Brute force built from library routines (numpy matmul/norm, lexsort, scipy
    softmax, einsum) on the tiny config, all 16 mixed queries."""
    c = gen.CONFIGS["tiny"]
    xb = gen.store_emb(c.store_seed, c.n, c.dim)
    act = gen.store_act(c.store_seed, c.n, c.layers, c.experts, c.moe_topk)
    qb = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, c.batch, mode=1)
    ids, sc, pred = oracle.sps(qb, xb, act, c.k)
    x = gen.bf16_bits_to_f32(xb).astype(np.float64)
    q = gen.bf16_bits_to_f32(qb).astype(np.float64)
    s = (q @ x.T) / (np.linalg.norm(q, axis=1)[:, None] * np.linalg.norm(x, axis=1)[None] + SIGMA)
    for i in range(c.batch):
        order = np.lexsort((np.arange(c.n), -s[i]))[: c.k]
        assert list(ids[i]) == list(order)
        np.testing.assert_allclose(sc[i], s[i, order], rtol=0, atol=1e-13)
        w = scipy_softmax(s[i, order])
        ref = np.einsum("r,rle->le", w, act[order].astype(np.float64))
        np.testing.assert_allclose(pred[i], ref, rtol=0, atol=1e-13)
    # copies of stored rows retrieve their source at rank 0 (SPEC S:229 self-retrieval)
    for i in range(c.batch):
        src = gen.query_source_row(c.query_seed, c.n, i, mode=1)
        if i % 8 in (4, 5):
            assert ids[i, 0] == src
    # identical queries (i % 8 == 7 duplicates i-1) give identical outputs
    for i in range(7, c.batch, 8):
        np.testing.assert_array_equal(ids[i], ids[i - 1])
        np.testing.assert_array_equal(pred[i], pred[i - 1])


@pytest.mark.parametrize("n,nthreads", [(5003, 1), (5003, 7), (12289, 8), (12289, 64), (20000, 256)])
def test_threaded_row_split_vs_numpy(n, nthreads):
    """The oracle's pthread row split (all_scores, N >= 1024) against numpy brute force:
    every score of the [B, N] matrix, and the whole path (select, softmax, predict) with
    exact duplicate rows planted across the per-thread range boundaries, so an off-by-one
    in a thread's [lo, hi) (a dropped, doubled or shifted row) or a tie broken by thread
    order instead of the lower id fails here."""
    c = gen.CONFIGS["c2"]
    xb = gen.store_emb(c.store_seed, n, c.dim).copy()
    act = gen.store_act(c.store_seed, n, c.layers, c.experts, c.moe_topk)
    qb = gen.queries(c.store_seed, c.query_seed, n, c.dim, 6, mode=1)
    per = -(-n // nthreads)
    for b in range(per, n, per):  # rows on both sides of each thread boundary
        xb[b] = xb[b - 1]
    qb[0] = xb[per - 1]            # a query whose best matches straddle a boundary
    x = gen.bf16_bits_to_f32(xb).astype(np.float64)
    q = gen.bf16_bits_to_f32(qb).astype(np.float64)
    ref = (q @ x.T) / (np.linalg.norm(q, axis=1)[:, None] * np.linalg.norm(x, axis=1)[None] + SIGMA)
    s = oracle.scores(qb, xb, nthreads=nthreads)
    np.testing.assert_allclose(s, ref, rtol=0, atol=1e-12)
    k = 12
    ids, sc, pred = oracle.sps(qb, xb, act, k, nthreads=nthreads)
    for i in range(qb.shape[0]):
        order = np.lexsort((np.arange(n), -s[i]))[:k]   # library sort of the (independent) scores
        order_ref = np.lexsort((np.arange(n), -ref[i]))[:k]
        assert list(ids[i]) == list(order) == list(order_ref)
        w = scipy_softmax(ref[i, order])
        np.testing.assert_allclose(pred[i], np.einsum("r,rle->le", w, act[order].astype(np.float64)),
                                   rtol=0, atol=1e-12)
    if per < n:
        assert ids[0, 0] == per - 1 and ids[0, 1] == per  # duplicate pair: lower id first


# ---------------------------------------------------------------- NEXT-N4 JS divergence

def test_js_divergence_pins():
    """Identical -> 0; disjoint supports -> 1 (base-2 maximum); [.5,.5] vs [.9,.1] ->
    0.146793 (re-derived; SPEC S:249's 0.2089 is wrong); symmetric; equals
    scipy's jensenshannon(base=2)**2 (a library routine) row by row, averaged over layers."""
    from scipy.spatial.distance import jensenshannon
    assert oracle.js_divergence([[0.2, 0.3, 0.5]], [[0.2, 0.3, 0.5]]) == 0.0
    assert abs(oracle.js_divergence([[1.0, 0.0]], [[0.0, 1.0]]) - 1.0) <= 1e-15
    assert abs(oracle.js_divergence([[0.5, 0.5]], [[0.9, 0.1]]) - 0.146793) <= 5e-7
    rng = np.random.default_rng(9)
    for L, E in [(1, 2), (3, 8), (27, 64)]:
        p = rng.random((L, E)); p[rng.random((L, E)) < 0.2] = 0; p /= p.sum(1, keepdims=True)
        q = rng.random((L, E)); q /= q.sum(1, keepdims=True)
        ref = np.mean([jensenshannon(p[l], q[l], base=2) ** 2 for l in range(L)])
        assert abs(oracle.js_divergence(p, q) - ref) <= 1e-12
        assert abs(oracle.js_divergence(p, q) - oracle.js_divergence(q, p)) <= 1e-15
