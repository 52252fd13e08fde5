#!/usr/bin/env python
"""NEXT-N2 timing: clustering-tree search (Algorithm 1) vs the exact BF scan on one
store.  Reports the build time, per-batch device time of both paths (CUDA events,
L2 flushed between iterations), recall@k of the tree vs BF and the Eq. 11 evaluations.

  python scripts/tree_bench.py [--config c3] [--batch 64] [--k 16] [--beta 150] [--branching 8]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402


def main():
    import torch

    import paper_2512_18674_b200 as remoe
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--k", type=int, default=16)
    ap.add_argument("--beta", type=int, default=150)
    ap.add_argument("--branching", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    c = gen.CONFIGS[args.config]
    x = gen.store_emb(c.store_seed, c.n, c.dim)
    a = gen.store_act(c.store_seed, c.n, c.layers, c.experts, c.moe_topk)
    sps = remoe.Sps(torch.from_numpy(x.view(np.int16)).cuda(), torch.from_numpy(a).cuda(),
                    max_k=max(32, args.k), max_batch=max(256, args.batch))
    del x, a
    info = sps.tree_build(args.beta, args.branching, 10, 7)
    q = torch.from_numpy(gen.queries(c.store_seed, c.query_seed, c.n, c.dim, args.batch).view(np.int16)).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn):
        for _ in range(3):
            fn()
        ms = []
        for _ in range(args.iters):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return float(np.median(ms)), out
    bf_ms, (bf_ids, _, _) = timed(lambda: sps.query(q, args.k))
    tr_ms, (t_ids, _, _, _, n_eval) = timed(lambda: sps.tree_query(q, args.k))
    bf_ids, t_ids = bf_ids.cpu().numpy(), t_ids.cpu().numpy()
    recall = float(np.mean([len(set(u) & set(v)) / args.k for u, v in zip(bf_ids, t_ids)]))
    print(json.dumps({"config": args.config, "n": c.n, "dim": c.dim, "batch": args.batch, "k": args.k,
                      "beta": args.beta, "branching": args.branching, "n_nodes": info.n_nodes,
                      "n_leaves": info.n_leaves, "depth": info.depth, "build_ms": round(info.build_ms, 1),
                      "bf_ms": round(bf_ms, 4), "tree_ms": round(tr_ms, 4), "speedup": round(bf_ms / tr_ms, 2),
                      "recall_vs_bf": round(recall, 4), "mean_evals": float(n_eval.float().mean()),
                      "evals_ratio_bf": round(c.n / float(n_eval.float().mean()), 1)}))


if __name__ == "__main__":
    main()
