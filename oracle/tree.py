"""NEXT-N2 oracle: the multi-fork clustering tree and Algorithm 1 (§IV-B,
lines 386-417), plain numpy fp64, one node and one step at a time.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/ alone; it shares no
code with the CUDA path (the counter-based generator below is implemented separately on
each side, as the tier rules allow).

Paper text followed (P = PAPER.md line):
  P:389  "any node (cluster) with more than beta prompts is recursively partitioned.  The
          partition is based on a customized k-medoids clustering algorithm using
          prompt-level semantic similarity as distance metric, where roulette wheel
          sampling-based centroid initialization and subcluster-level centroid updating
          are conducted."
  P:391  "the tree is traversed to a leaf by successively selecting the semantically
          closest subcluster centroid.  If there are enough prompts in the leaf, top-alpha
          semantically similar ones are returned; otherwise, we turn to the leaf's
          siblings for supplement."   (Algorithm 1)

Readings (R24-R28):
  R24 roulette init: the first medoid is the member at floor(u0 n); medoid j >= 1 is
      drawn with probability proportional to d_i = max(0, 1 - max_{chosen m} cos(x_i, x_m))
      (distance mass to the nearest chosen medoid; chosen medoids get d = 0): the first
      i with cumsum(d)[i] > u_j * sum(d).  sum(d) == 0 stops the init early.
  R25 k-medoids "distance" is 1 - cos with the sigma-free cosine x_i . x_j / (|x_i||x_j|)
      (sigma only guards Eq. 11's division; the medoid objective
      sum_{t in C} cos(x_i, x_t) is then exactly x^_i . sum_t x^_t).  Assignment: the
      most similar medoid, ties -> lower slot.  Update ("subcluster-level"): per cluster,
      the member maximising the summed cosine to its cluster; values within
      1e-10 * |cluster| of the maximum are ties: the current medoid stays if it is one,
      else the earliest tied member wins; an empty cluster keeps its medoid.  Stop when the medoids do not change or after
      max_iter updates; the final assignment is to the final medoids.
  R26 children are the non-empty clusters in slot order, members in their original
      order (a stable partition of the node's range); a split with < 2 non-empty
      clusters (duplicate rows) falls back to c equal contiguous chunks.
  R27 search scores are Eq. 11 (sigma included, fp64 here); the closest child is the one
      with the larger (score, lower global id) key -- the same key order as BF.
  R28 supplement ("add samples into PROM until alpha samples are obtained", Alg. 1
      line 8): the siblings of the current node in descending key order, each subtree
      explored depth-first with children in descending key order, whole leaves added,
      until >= alpha candidates; if the siblings run out, the same at the parent's level,
      and so on up to the root (so alpha <= N always fills).  The answer is the
      top-alpha by key of the gathered candidates.
Node numbering is breadth-first (root 0, children appended in the order their parents
split); u(seed, node, j) is the counter-based uniform below.
"""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1
TIE_TOL = 1e-10   # medoid-update tie window per member (R25)


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def uniform(seed: int, node: int, j: int) -> float:
    """u in [0, 1) with 53 random bits for draw j of node `node` (R24)."""
    h = splitmix64((seed ^ ((node * 0x9E3779B97F4A7C15 + j) & _M64)) & _M64)
    return (h >> 11) * (1.0 / (1 << 53))


def _unit_rows(x: np.ndarray) -> np.ndarray:
    n = np.sqrt((x * x).sum(axis=1))
    out = np.zeros_like(x)
    nz = n > 0
    out[nz] = x[nz] / n[nz, None]
    return out


def roulette_init(V: np.ndarray, c: int, seed: int, node: int) -> list[int]:
    """R24: medoid positions (within the node) by roulette-wheel sampling."""
    n = V.shape[0]
    m = [min(n - 1, int(np.floor(uniform(seed, node, 0) * n)))]
    best = V @ V[m[0]]
    for j in range(1, c):
        d = np.maximum(0.0, 1.0 - best)
        d[m] = 0.0
        cs = np.cumsum(d)
        total = cs[-1]
        if not total > 0:
            break
        t = uniform(seed, node, j) * total
        p = int(np.searchsorted(cs, t, side="right"))   # first i with cs[i] > t
        m.append(min(p, n - 1))
        best = np.maximum(best, V @ V[m[-1]])
    return m


def assign(V: np.ndarray, m: list[int]) -> np.ndarray:
    """R25: label of every member = most similar medoid (first max -> lower slot)."""
    return np.argmax(V @ V[m].T, axis=1)


def update(V: np.ndarray, lab: np.ndarray, m: list[int]) -> list[int]:
    """R25: subcluster-level medoid update: the member maximising the summed cosine within
    the cluster (computed literally from the cluster's Gram matrix).  Members within
    TIE_TOL * max(1, |cluster|) of the maximum count as maximisers: the current medoid is
    kept if it is one, else the earliest maximiser wins (a 2-member cluster is an exact
    tie by symmetry, so this rule is needed for a reproducible result)."""
    out = []
    for j in range(len(m)):
        idx = np.flatnonzero(lab == j)
        if idx.size == 0:
            out.append(m[j])
            continue
        G = V[idx] @ V[idx].T
        obj = G.sum(axis=1)
        near = obj >= obj.max() - TIE_TOL * max(1, idx.size)
        cur = np.flatnonzero(idx == m[j])
        if cur.size and near[cur[0]]:
            out.append(m[j])
        else:
            out.append(int(idx[np.argmax(near)]))
    return out


def kmedoids(V: np.ndarray, c: int, max_iter: int, seed: int, node: int):
    m = roulette_init(V, c, seed, node)
    for _ in range(max_iter):
        new = update(V, assign(V, m), m)
        if new == m:
            break
        m = new
    return m, assign(V, m)


def build_tree(x_bits: np.ndarray, beta: int, branching: int, max_iter: int, seed: int) -> dict:
    """The clustering tree over store rows (bf16 bits [N, D]).  Returns flat arrays:
    perm [N] (row ids; every node owns perm[begin:end]), begin, end, parent, child0,
    nchild, medoid (row id of the node's centroid; -1 for the root)."""
    from oracle import widen
    X = widen(np.asarray(x_bits, np.uint16))
    Xh = _unit_rows(X)
    N = X.shape[0]
    perm = np.arange(N, dtype=np.int64)
    begin, end, parent, child0, nchild, medoid = [0], [N], [-1], [-1], [0], [-1]
    i = 0
    while i < len(begin):
        b, e = begin[i], end[i]
        n = e - b
        if n > beta:
            pos = perm[b:e].copy()
            V = Xh[pos]
            c = min(branching, n)
            m, lab = kmedoids(V, c, max_iter, seed, i)
            slots = [j for j in range(len(m)) if np.any(lab == j)]
            child0[i] = len(begin)
            if len(slots) >= 2:
                order = np.argsort(lab, kind="stable")
                perm[b:e] = pos[order]
                at = b
                for j in slots:
                    cnt = int(np.sum(lab == j))
                    begin.append(at); end.append(at + cnt); parent.append(i)
                    child0.append(-1); nchild.append(0); medoid.append(int(pos[m[j]]))
                    at += cnt
                nchild[i] = len(slots)
            else:   # R26 fallback: c equal contiguous chunks, medoid = first member
                bounds = [b + (n * j) // c for j in range(c + 1)]
                for j in range(c):
                    begin.append(bounds[j]); end.append(bounds[j + 1]); parent.append(i)
                    child0.append(-1); nchild.append(0); medoid.append(int(perm[bounds[j]]))
                nchild[i] = c
        i += 1
    a = lambda v: np.asarray(v, np.int64)  # noqa: E731
    return dict(perm=perm, begin=a(begin), end=a(end), parent=a(parent), child0=a(child0),
                nchild=a(nchild), medoid=a(medoid))


def _score(q: np.ndarray, qn: float, x_bits: np.ndarray, rows, sigma: float) -> np.ndarray:
    """Eq. 11 on prompt vectors, fp64 (R27); widens only the rows it scores."""
    from oracle import widen
    rows = np.asarray(rows, np.int64)
    X = widen(x_bits[rows])
    xn = np.sqrt((X * X).sum(axis=1))
    return (X @ q) / (qn * xn + sigma)


def _order(scores: np.ndarray, gids: np.ndarray) -> np.ndarray:
    """Indices by key: score descending, then lower global id."""
    return np.lexsort((gids, -scores))


def search(tree: dict, x_bits: np.ndarray, q_bits: np.ndarray, k: int, sigma: float = 1e-6,
           id_offset: int = 0):
    """Algorithm 1 for every query.  Returns ids int64 [B, k], scores fp64 [B, k],
    leaf int64 [B] (the leaf the descent reached), n_eval int64 [B] (Eq. 11 evaluations)."""
    from oracle import widen
    x_bits = np.asarray(x_bits, np.uint16)
    Q = widen(np.asarray(q_bits, np.uint16))
    B = Q.shape[0]
    ids = np.full((B, k), -1, np.int64)
    sc = np.full((B, k), -np.inf)
    leaves = np.zeros(B, np.int64)
    evals = np.zeros(B, np.int64)
    child0, nchild, medoid = tree["child0"], tree["nchild"], tree["medoid"]
    begin, end, perm = tree["begin"], tree["end"], tree["perm"]
    for bq in range(B):
        q = Q[bq]
        qn = float(np.sqrt(q @ q))
        ne = 0

        def ranked_children(node):
            nonlocal ne
            ch = np.arange(child0[node], child0[node] + nchild[node])
            s = _score(q, qn, x_bits, medoid[ch], sigma)
            ne += ch.size
            return ch[_order(s, medoid[ch] + id_offset)]

        def descend(node):
            path = []
            while nchild[node] > 0:
                order = ranked_children(node)
                path.append((node, order))
                node = int(order[0])
            return node, path

        leaf, path = descend(0)
        leaves[bq] = leaf
        chosen = [leaf]
        count = end[leaf] - begin[leaf]

        def explore(node):          # R28: depth-first in key order, whole leaves
            nonlocal count
            if nchild[node] == 0:
                chosen.append(node)
                count += end[node] - begin[node]
                return
            for c in ranked_children(node):
                if count >= k:
                    return
                explore(int(c))

        cur = leaf
        for lvl in range(len(path) - 1, -1, -1):
            if count >= k:
                break
            for c in path[lvl][1]:
                if count >= k:
                    break
                if c != cur:
                    explore(int(c))
            cur = path[lvl][0]
        rows = np.concatenate([perm[begin[lf]:end[lf]] for lf in chosen])
        s = _score(q, qn, x_bits, rows, sigma)
        ne += rows.size
        o = _order(s, rows + id_offset)[:k]
        ids[bq, :o.size] = rows[o] + id_offset
        sc[bq, :o.size] = s[o]
        evals[bq] = ne
    return ids, sc, leaves, evals
