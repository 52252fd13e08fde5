"""NEXT-N2 on the GPU: the clustering tree (remoe_sps_tree_build) and Algorithm 1
(remoe_sps_tree_query) vs the oracle (oracle/tree.py, numpy fp64, pinned in
test_tree_oracle.py).

* Build: the exported tree equals the oracle's tree array for array (every integer
  decision is taken in fp64 on both sides; exact ties do not occur in these inputs).
* Search: same leaf and evaluation count per query (a differing leaf is accepted only
  where the descent had a near tie, |gap| <= 1e-4), ids/scores/pred by the BF parity
  protocol (tests/parity.py) against the oracle's search on the same tree.
* Full size (1M x 1024, the c3 store): structural invariants, k-medoids fixed-point
  checks on sampled members, and sampled queries searched by the oracle on the GPU's
  tree."""
import numpy as np
import pytest

import gen
import oracle
from oracle import tree as T
from parity import compare

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("remoe_lib_built")]
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_18674_b200 as remoe  # noqa: E402

FIELDS = ("perm", "begin", "end", "parent", "child0", "nchild", "medoid")


def _sps(x, act, max_k=64, **kw):
    return remoe.Sps(torch.from_numpy(x.view(np.int16)).cuda(), torch.from_numpy(act).cuda(), max_k=max_k,
                     max_batch=256, **kw)


def _q(q):
    return torch.from_numpy(q.view(np.int16)).cuda()


def _assert_same_tree(g, o):
    for f in FIELDS:
        np.testing.assert_array_equal(np.asarray(g[f], np.int64), np.asarray(o[f], np.int64), err_msg=f)


def _descent_gaps(tree, x, q, sigma=oracle.SIGMA):
    """Smallest gap between the best and second-best child score along each query's
    oracle descent (near ties may legitimately send fp32 and fp64 different ways)."""
    gaps = []
    Q = oracle.widen(q)
    for b in range(q.shape[0]):
        node, g = 0, np.inf
        qn = np.sqrt(Q[b] @ Q[b])
        while tree["nchild"][node] > 0:
            ch = np.arange(tree["child0"][node], tree["child0"][node] + tree["nchild"][node])
            s = T._score(Q[b], qn, x, tree["medoid"][ch], sigma)
            o = np.argsort(-s, kind="stable")
            g = min(g, s[o[0]] - s[o[1]])
            node = int(ch[o[0]])
        gaps.append(g)
    return np.array(gaps)


CASES = [  # N, D, beta, branching, max_iter, seed
    (3000, 128, 150, 8, 10, 5),
    (2000, 64, 60, 4, 0, 1),
    (1500, 1024, 100, 16, 10, 3),
    (5000, 256, 150, 8, 10, 9),
    (900, 40, 20, 3, 25, 2),
]


@pytest.mark.parametrize("case", CASES)
def test_tree_build_matches_oracle(case):
    N, D, beta, br, it, seed = case
    x = gen.store_emb(seed, N, D)
    act = gen.store_act(seed, N, 2, 8, 2)
    s = _sps(x, act)
    info = s.tree_build(beta, br, it, seed)
    o = T.build_tree(x, beta, br, it, seed)
    _assert_same_tree(s.tree_export(), o)
    assert info.n_nodes == len(o["begin"])
    assert info.max_leaf <= beta


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("k", [1, 15, 64])
def test_tree_search_matches_oracle(case, k):
    N, D, beta, br, it, seed = case
    x = gen.store_emb(seed, N, D)
    act = gen.store_act(seed, N, 3, 16, 2)
    s = _sps(x, act)
    s.tree_build(beta, br, it, seed)
    tree = s.tree_export()
    q = gen.queries(seed, seed + 100, N, D, 96, mode=1)
    ids, sc, pred, leaf, ne = s.tree_query(_q(q), k)
    ids, sc, pred = ids.cpu().numpy(), sc.cpu().numpy(), pred.cpu().numpy()
    leaf, ne = leaf.cpu().numpy(), ne.cpu().numpy()
    o_ids, o_sc, o_leaf, o_ne = T.search(tree, x, q, k)
    same = leaf == o_leaf
    if not same.all():
        gaps = _descent_gaps(tree, x, q)
        assert np.all(gaps[~same] <= 1e-4), "leaf differs without a near tie in the descent"
    assert same.mean() >= 0.9
    np.testing.assert_array_equal(ne[same], o_ne[same])
    sel = np.flatnonzero(same)
    o_pred = np.stack([oracle.predict(o_ids[i], oracle.softmax(o_sc[i]), act) for i in sel])
    rep = compare(q[sel], x, act, k, ids[sel], sc[sel], pred[sel],
                  oracle_out=(o_ids[sel], o_sc[sel], o_pred))
    assert rep.ok(), rep.failures[:5]


def test_single_leaf_tree_is_brute_force():
    """beta >= N -> the tree search returns the BF top-k (compared with the BF
    oracle by the parity protocol) and evaluates every row exactly once."""
    N, D, k = 1200, 256, 32
    x = gen.store_emb(4, N, D)
    act = gen.store_act(4, N, 2, 8, 2)
    s = _sps(x, act)
    info = s.tree_build(1500, 8, 10, 1)
    assert info.n_nodes == 1
    q = gen.queries(4, 5, N, D, 64, mode=1)
    ids, sc, pred, leaf, ne = s.tree_query(_q(q), k)
    assert np.all(ne.cpu().numpy() == N) and np.all(leaf.cpu().numpy() == 0)
    rep = compare(q, x, act, k, ids.cpu().numpy(), sc.cpu().numpy(), pred.cpu().numpy())
    assert rep.ok(), rep.failures[:5]


def test_self_retrieval_and_supplement():
    """S:229 self-retrieval, and alpha > beta (every query needs sibling leaves, R28)."""
    N, D = 3000, 128
    x = gen.store_emb(8, N, D)
    act = gen.store_act(8, N, 2, 8, 2)
    s = _sps(x, act, max_k=128)
    s.tree_build(40, 4, 10, 8)
    rows = np.arange(0, N, 31)
    ids, _, _, _, _ = s.tree_query(_q(np.ascontiguousarray(x[rows])), 100)
    ids = ids.cpu().numpy()
    assert all(r in ids[i] for i, r in enumerate(rows))
    assert np.all(ids >= 0) and all(len(set(r)) == 100 for r in ids)


def test_duplicate_rows_fallback():
    x = np.concatenate([np.tile(gen.store_emb(3, 1, 16), (40, 1)), gen.store_emb(4, 30, 16)])
    act = gen.store_act(3, 70, 1, 4, 1)
    s = _sps(x, act, max_k=8)
    s.tree_build(10, 4, 5, 1)
    o = T.build_tree(x, 10, 4, 5, 1)
    _assert_same_tree(s.tree_export(), o)


def test_tree_errors():
    x = gen.store_emb(1, 500, 64)
    act = gen.store_act(1, 500, 1, 4, 1)
    s = _sps(x, act, max_k=64)
    q = _q(gen.queries(1, 2, 500, 64, 4))
    with pytest.raises(remoe.RemoeError) as e:
        s.tree_query(q, 4)
    assert e.value.status == 6          # STATE: no tree yet
    for beta, br, it in ((0, 4, 1), (50, 1, 1), (50, 17, 1), (50, 4, -1)):
        with pytest.raises(remoe.RemoeError) as e:
            s.tree_build(beta, br, it, 0)
        assert e.value.status == 1
    with pytest.raises(remoe.RemoeError) as e:
        s.tree_build(2000, 4, 1, 0)     # beta + max_k - 1 > 2048
    assert e.value.status == 5
    s.tree_build(50, 4, 3, 0)
    ids, *_ = s.tree_query(q[:0], 4)
    assert ids.shape == (0, 4)
    with pytest.raises(remoe.RemoeError):
        s.tree_query(q, 501)


@pytest.mark.slow
def test_tree_full_size_c3():
    """The c3 store (1M x 1024, the bench workload), beta = 150, branching 8 (P:675's
    beta): invariants, fixed-point checks on sampled members, and 16 sampled queries
    searched by the oracle on the GPU's tree (ids by the parity protocol)."""
    cfg = gen.CONFIGS["c3"]
    N, D = cfg.n, cfg.dim
    x = gen.store_emb(cfg.store_seed, N, D)
    act = gen.store_act(cfg.store_seed, N, cfg.layers, cfg.experts, cfg.moe_topk)
    s = _sps(x, act, max_k=32)
    info = s.tree_build(150, 8, 10, 7)
    t = s.tree_export()
    assert info.max_leaf <= 150
    assert np.array_equal(np.sort(t["perm"]), np.arange(N))
    leaves = np.flatnonzero(t["nchild"] == 0)
    assert (t["end"][leaves] - t["begin"][leaves]).sum() == N
    rng = np.random.default_rng(0)
    # assignment fixed point: a sampled member is at least as close (fp64) to its own
    # centroid as to every sibling centroid, up to 1e-12
    for node in rng.choice(np.flatnonzero(t["parent"] >= 0), 40, replace=False):
        p = t["parent"][node]
        sib = np.arange(t["child0"][p], t["child0"][p] + t["nchild"][p])
        meds = oracle.widen(x[t["medoid"][sib]])
        meds /= np.linalg.norm(meds, axis=1, keepdims=True)
        mem = t["perm"][t["begin"][node]:t["end"][node]]
        r = oracle.widen(x[rng.choice(mem, min(8, mem.size), replace=False)])
        r /= np.linalg.norm(r, axis=1, keepdims=True)
        cos = r @ meds.T
        own = int(np.flatnonzero(sib == node)[0])
        assert np.all(cos[:, own] >= cos.max(axis=1) - 1e-12)
    k = 15
    q = gen.queries(cfg.store_seed, cfg.query_seed, N, D, 16, mode=0)
    ids, sc, pred, leaf, ne = s.tree_query(_q(q), k)
    o_ids, o_sc, o_leaf, o_ne = T.search(t, x, q, k)
    same = leaf.cpu().numpy() == o_leaf
    assert same.mean() >= 0.9
    sel = np.flatnonzero(same)
    o_pred = np.stack([oracle.predict(o_ids[i], oracle.softmax(o_sc[i]), act) for i in sel])
    rep = compare(q[sel], x, act, k, ids.cpu().numpy()[sel], sc.cpu().numpy()[sel], pred.cpu().numpy()[sel],
                  oracle_out=(o_ids[sel], o_sc[sel], o_pred))
    assert rep.ok(), rep.failures[:5]
    assert ne.cpu().numpy().mean() * 10 < N
