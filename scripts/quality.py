#!/usr/bin/env python
"""NEXT-N4: prediction-quality harness (the methodology of the paper's
fig:predict_method_compare, on synthetic data).

History = the first N prompts of a generated store; held-out queries = the next H
prompts of the same generator, whose own activation tables are the ground truth.
Predictors: SPS (this library, exact BF top-alpha + softmax weighting, alpha = 15 as in
P:675), TREE (NEXT-N2: the paper's clustering-tree search, beta = 150),
EF (uniform 1/E, P:672 baseline 5), DOP (historical mean, P:672 baseline 3).
Metric: mean base-2 JS divergence over layers (remoe_js_divergence on the GPU).

  python scripts/quality.py [--config c2] [--n 100000] [--held-out 512] [--k 15]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402


def evaluate(cfg_name="c2", n=100_000, held_out=512, k=15, seed_offset=0, beta=150, branching=8):
    import torch

    import paper_2512_18674_b200 as remoe
    c = gen.CONFIGS[cfg_name]
    seed = c.store_seed + seed_offset
    total = n + held_out
    x = gen.store_emb(seed, total, c.dim)
    a = gen.store_act(seed, total, c.layers, c.experts, c.moe_topk)
    hist_x, hist_a = x[:n], a[:n]
    q, truth = x[n:], a[n:]
    sps = remoe.Sps(hist_x, hist_a, max_k=max(16, k), max_batch=256)
    qd = torch.from_numpy(q.view(np.int16)).cuda()
    bf_ids, _, pred = sps.query(qd, k)
    info = sps.tree_build(beta, branching, 10, seed)
    t_ids, _, t_pred, _, n_eval = sps.tree_query(qd, k)
    bf_ids, t_ids = bf_ids.cpu().numpy(), t_ids.cpu().numpy()
    recall = float(np.mean([len(set(a) & set(b)) / k for a, b in zip(bf_ids, t_ids)]))
    truth_d = torch.from_numpy(truth).cuda()
    ef = torch.full((c.layers, c.experts), 1.0 / c.experts, device="cuda")
    dop = torch.from_numpy(hist_a.astype(np.float64).mean(0).astype(np.float32)).cuda()
    res = {}
    for name, P in (("SPS", pred), ("TREE", t_pred), ("DOP", dop.expand_as(truth_d).contiguous()),
                     ("EF", ef.expand_as(truth_d).contiguous())):
        js = remoe.js_divergence(P, truth_d)
        res[name] = float(js.mean())
    res["tree"] = {"recall_vs_bf": recall, "mean_evals": float(n_eval.float().mean()),
                   "evals_bf": n, "n_nodes": info.n_nodes, "depth": info.depth,
                   "build_ms": round(info.build_ms, 1), "beta": beta, "branching": branching}
    torch.cuda.synchronize()
    sps.close()
    return res, pred.cpu().numpy(), truth


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--held-out", type=int, default=512)
    ap.add_argument("--k", type=int, default=15)
    args = ap.parse_args()
    res, _, _ = evaluate(args.config, args.n, args.held_out, args.k)
    print(json.dumps({"config": args.config, "history": args.n, "held_out": args.held_out,
                      "alpha": args.k, "mean_js_base2": res}))


if __name__ == "__main__":
    main()
