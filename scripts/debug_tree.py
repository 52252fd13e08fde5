"""Debug helper: compare the GPU tree build with the oracle node by node (REMOE_TREE_DEBUG)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from oracle import tree as T  # noqa: E402

N, D, beta, br, it, seed = (int(v) for v in (sys.argv[1:] or [3000, 128, 150, 8, 10, 5]))
x = gen.store_emb(seed, N, D)
Xh = T._unit_rows(gen.bf16_bits_to_f32(x).astype(np.float64))
# oracle with a trace of every node's init and iterations
perm = np.arange(N)
begin, end = [0], [N]
i = 0
while i < len(begin):
    b, e = begin[i], end[i]
    n = e - b
    if n > beta:
        pos = perm[b:e].copy()
        V = Xh[pos]
        c = min(br, n)
        m = T.roulette_init(V, c, seed, i)
        print("ORACLE init node %d:" % i, " ".join(str(pos[j]) for j in m))
        for _ in range(it):
            new = T.update(V, T.assign(V, m), m)
            print("ORACLE iter node %d:" % i, " ".join(str(pos[j]) for j in new))
            if new == m:
                break
            m = new
        lab = T.assign(V, m)
        slots = [j for j in range(len(m)) if np.any(lab == j)]
        order = np.argsort(lab, kind="stable")
        perm[b:e] = pos[order]
        at = b
        for j in slots:
            cnt = int(np.sum(lab == j))
            begin.append(at); end.append(at + cnt)
            at += cnt
    i += 1
