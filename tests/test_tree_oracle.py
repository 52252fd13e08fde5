"""Pins of the NEXT-N2 oracle (oracle/tree.py: the clustering tree and Algorithm 1)
against what the paper, SPEC and mathematics fix: the degenerate single-leaf tree is BF,
self-retrieval, cluster purity on separated data, k-medoids fixed-point conditions checked
pair by pair, the roulette draw distribution, the splitmix64 reference value, structural
invariants, and the quality/evaluation-count claim."""
import numpy as np
import pytest

import gen
import oracle
from oracle import tree as T


def _bits(x):
    return gen.f32_to_bf16_bits(np.asarray(x, np.float32))


def _corpus(n=2000, d=64, seed=5):
    return gen.store_emb(seed, n, d)


def test_splitmix64_reference_value():
    # the first output of the reference splitmix64 generator seeded with 0
    assert T.splitmix64(0) == 0xE220A8397B1DCDAF
    u = np.array([T.uniform(3, n, j) for n in range(50) for j in range(20)])
    assert u.min() >= 0 and u.max() < 1 and abs(u.mean() - 0.5) < 0.03


def test_under_capacity_is_a_single_leaf():
    # 100 prompts, beta = 150 -> no split
    t = T.build_tree(_corpus(100), beta=150, branching=8, max_iter=10, seed=1)
    assert len(t["begin"]) == 1 and t["nchild"][0] == 0
    assert np.array_equal(t["perm"], np.arange(100))


def _check_structure(t, N, beta):
    perm = t["perm"]
    assert np.array_equal(np.sort(perm), np.arange(N))
    leaves = np.flatnonzero(t["nchild"] == 0)
    assert np.all(t["end"][leaves] - t["begin"][leaves] <= beta)
    assert (t["end"][leaves] - t["begin"][leaves]).sum() == N   # every prompt in exactly one leaf
    for i in np.flatnonzero(t["nchild"] > 0):
        ch = np.arange(t["child0"][i], t["child0"][i] + t["nchild"][i])
        assert ch.size >= 2
        assert t["begin"][ch[0]] == t["begin"][i] and t["end"][ch[-1]] == t["end"][i]
        assert np.all(t["end"][ch[:-1]] == t["begin"][ch[1:]])
        assert np.all(t["parent"][ch] == i)
        for c in ch:   # the centroid is a member of its subcluster
            assert t["medoid"][c] in perm[t["begin"][c]:t["end"][c]]


def test_structure_invariants():
    t = T.build_tree(_corpus(), beta=150, branching=8, max_iter=10, seed=2)
    _check_structure(t, 2000, 150)
    assert len(t["begin"]) > 8


def test_kmedoids_fixed_point_pairwise():
    """With max_iter large enough to converge, every split is a k-medoids fixed point:
    each member is at least as close to its own subcluster's centroid as to any sibling
    centroid, and the centroid maximises the summed cosine to its subcluster -- both
    checked pair by pair with an explicit cosine (R25)."""
    x = _corpus(600, 32, seed=9)
    t = T.build_tree(x, beta=100, branching=4, max_iter=100, seed=4)
    X = oracle.widen(x)

    def cos(a, b):
        return float(np.dot(X[a], X[b]) / (np.linalg.norm(X[a]) * np.linalg.norm(X[b])))
    perm = t["perm"]
    for i in np.flatnonzero(t["nchild"] > 0):
        ch = list(range(t["child0"][i], t["child0"][i] + t["nchild"][i]))
        meds = [int(t["medoid"][c]) for c in ch]
        for ci, c in enumerate(ch):
            mem = perm[t["begin"][c]:t["end"][c]]
            for r in mem[::7]:
                own = cos(r, meds[ci])
                assert all(own >= cos(r, mo) - 1e-12 for mo in meds)
            tot = {int(r): sum(cos(r, s) for s in mem) for r in mem}
            assert tot[meds[ci]] >= max(tot.values()) - 1e-9


def test_first_split_recovers_separated_clusters():
    # 4 well-separated clusters, branching 4 -> first split purity >= 90%
    rng = np.random.default_rng(0)
    D = 32
    centers = np.linalg.qr(rng.standard_normal((D, 4)))[0].T * 4.0
    labels = np.repeat(np.arange(4), 100)
    x = centers[labels] + 0.5 * rng.standard_normal((400, D)) / np.sqrt(D)
    t = T.build_tree(_bits(x), beta=150, branching=4, max_iter=20, seed=3)
    assert t["nchild"][0] == 4
    hit = 0
    for c in range(t["child0"][0], t["child0"][0] + 4):
        lab = labels[t["perm"][t["begin"][c]:t["end"][c]]]
        hit += np.bincount(lab, minlength=4).max()
    assert hit / 400 >= 0.9


def test_roulette_draw_distribution():
    """R24: with one medoid chosen, the second is drawn with probability d_i / sum d,
    d_i = 1 - cos(x_i, medoid).  Monte Carlo over 4000 node counters."""
    V = T._unit_rows(np.array([[1, 0, 0], [1, 1, 0], [0, 1, 0], [-1, 0.2, 0], [0.3, 0.3, 1]], float))
    counts = np.zeros(5)
    firsts = np.zeros(5)
    trials = 4000
    for node in range(trials):
        m = T.roulette_init(V, 2, seed=7, node=node)
        firsts[m[0]] += 1
        if m[0] == 0:
            counts[m[1]] += 1
    d = 1 - V @ V[0]
    d[0] = 0
    p = d / d.sum()
    n0 = counts.sum()
    assert abs(n0 / trials - 0.2) < 0.03                     # first pick uniform
    assert counts[0] == 0
    assert np.all(np.abs(counts / n0 - p) < 4 * np.sqrt(p * (1 - p) / n0) + 1e-9)


def test_single_leaf_search_is_brute_force():
    # a single-leaf tree returns exactly the brute-force top-alpha
    x = _corpus(300, 64, seed=11)
    q = gen.queries(11, 12, 300, 64, 24, mode=1)
    t = T.build_tree(x, beta=1000, branching=8, max_iter=10, seed=1)
    ids, sc, leaf, ne = T.search(t, x, q, k=15)
    ref_ids, ref_sc, _ = oracle.sps(q, x, np.zeros((300, 1, 1), np.float32), 15, want_pred=False)
    assert np.array_equal(ids, ref_ids)
    assert np.allclose(sc, ref_sc, rtol=0, atol=1e-15)
    assert np.all(leaf == 0) and np.all(ne == 300)


def test_self_retrieval_and_quality_vs_bf():
    """S:229 self-retrieval; S:231 on a clustered 2000-prompt corpus: mean SCS of the
    tree's top-alpha >= 0.95 x brute force's, with >= 5x fewer Eq. 11 evaluations."""
    N, D, k = 2000, 64, 15
    x = _corpus(N, D, seed=21)
    t = T.build_tree(x, beta=150, branching=8, max_iter=10, seed=5)
    rows = np.arange(0, N, 97)
    ids, _, _, _ = T.search(t, x, x[rows], k)
    assert all(r in ids[i] for i, r in enumerate(rows))
    q = gen.queries(21, 22, N, D, 64, mode=0)
    ids, sc, _, ne = T.search(t, x, q, k)
    _, ref_sc, _ = oracle.sps(q, x, np.zeros((N, 1, 1), np.float32), k, want_pred=False)
    assert sc.mean() >= 0.95 * ref_sc.mean()
    assert ne.mean() * 5 <= N


def test_supplement_from_siblings_hand_tree():
    """R28 on a hand-built tree: root with leaves A (3 rows), B (10), C (10); a query that
    lands in A with alpha = 12 gathers A and the better-scoring sibling only."""
    rng = np.random.default_rng(1)
    D = 16
    base = np.eye(D)[:3] * 3
    x = np.concatenate([base[0] + 0.1 * rng.standard_normal((3, D)),
                        base[1] + 0.1 * rng.standard_normal((10, D)),
                        base[2] + 0.1 * rng.standard_normal((10, D))])
    xb = _bits(x)
    t = dict(perm=np.arange(23), begin=np.array([0, 0, 3, 13]), end=np.array([23, 3, 13, 23]),
             parent=np.array([-1, 0, 0, 0]), child0=np.array([1, -1, -1, -1]),
             nchild=np.array([3, 0, 0, 0]), medoid=np.array([-1, 0, 3, 13]))
    q = _bits(base[0] + 0.6 * base[1] / 3 + 0.1 * base[2] / 3)[None]
    ids, sc, leaf, ne = T.search(t, xb, q, k=12)
    assert leaf[0] == 1
    assert set(ids[0]) <= set(range(13)) and len(set(ids[0])) == 12
    assert ne[0] == 3 + 13
    ids, _, _, _ = T.search(t, xb, q, k=3)       # enough in the leaf: no supplement
    assert set(ids[0]) == {0, 1, 2}


def test_structure_on_duplicates_fallback():
    # R26: identical rows cannot be separated by k-medoids: equal contiguous chunks
    x = np.tile(_corpus(1, 16, seed=3), (40, 1))
    t = T.build_tree(x, beta=10, branching=4, max_iter=5, seed=1)
    _check_structure(t, 40, 10)
    assert t["nchild"][0] == 4 and list(t["end"][1:5] - t["begin"][1:5]) == [10, 10, 10, 10]


def test_supplement_always_fills_alpha():
    """R28 (Alg. 1 line 8, "until alpha samples are obtained"): with alpha far above beta
    the depth-first walk still gathers alpha distinct prompts whenever N >= alpha, and the
    answer is the top-alpha by key of what it gathered."""
    N, D = 900, 40
    x = _corpus(N, D, seed=2)
    t = T.build_tree(x, beta=20, branching=3, max_iter=25, seed=2)
    q = gen.queries(2, 3, N, D, 40, mode=1)
    for k in (64, 300, N):
        ids, sc, _, ne = T.search(t, x, q, k)
        assert np.all(ids >= 0)
        assert all(len(set(r)) == k for r in ids)
        assert np.all(np.diff(sc, axis=1) <= 0)
    ids, sc, _, _ = T.search(t, x, q, N)        # alpha = N gathers everything: BF order
    ref_ids, _, _ = oracle.sps(q, x, np.zeros((N, 1, 1), np.float32), N, want_pred=False)
    assert np.array_equal(ids, ref_ids)
