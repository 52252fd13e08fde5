#!/usr/bin/env python
"""Small workload for compute-sanitizer (scripts/sanitize.sh): tiny and a 20k-row c2
store, each scan kernel forced in turn (streaming, resident-slab tensor core, CTA pair),
seeded and unseeded, k in {5, 64}, plus a 3-rank loopback group (the multi-rank stages)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import torch  # noqa: E402
import paper_2512_18674_b200 as remoe  # noqa: E402

for name, n, B in (("tiny", 1000, 16), ("c2", 40_000, 40)):
    c = gen.CONFIGS[name]
    x = gen.store_emb(c.store_seed, n, c.dim)
    a = gen.store_act(c.store_seed, n, c.layers, c.experts, c.moe_topk)
    q = torch.from_numpy(gen.queries(c.store_seed, c.query_seed, n, c.dim, B, mode=1).view(np.int16)).cuda()
    s = remoe.Sps(x, a, max_k=64, max_batch=64)
    for kern in (remoe.KERNEL_STREAM, remoe.KERNEL_TC, remoe.KERNEL_PAIR):
        try:
            s.set_kernel(kern)
        except remoe.RemoeError:
            continue
        for k in (5, 64):
            ids, sc, pred = s.query(q, k)
            torch.cuda.synchronize()
            print(f"{name} kernel={kern} k={k}: ok, last_kernel={s.info().last_scan_kernel}", flush=True)
    s.close()
    g_shards = []
    for r in range(3):
        off, nl = gen.shard_range(n, 3, r)
        g_shards.append((x[off:off + nl].copy(), a[off:off + nl].copy()))
    g = remoe.LoopbackGroup([u for u, _ in g_shards], [v for _, v in g_shards], n, max_k=16, max_batch=64)
    ids, sc, pred = g.query(q, 10)
    torch.cuda.synchronize()
    g.close()
    print(f"{name} loopback G=3: ok", flush=True)
