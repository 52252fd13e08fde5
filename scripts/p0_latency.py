#!/usr/bin/env python
"""p0: the paper's own SPS scale (5,000 stored prompts, alpha = 15, one
request at a time -- serverless) on one B200, for context next to the paper's only
SPS claims (tree build <= 0.5 s; SPS "more than 10 times faster than BF"; BF the more
accurate).  Two shapes: GPT2-moe (D = 768, table 12 x 8) and
DeepSeek-V2-Lite (D = 2048, table 26 x 64; D > 1536 runs the streaming kernel).

Reports, per shape: exact BF (remoe_sps_query) single-query latency on the device
(CUDA events, graphed path, p10/p50/p90) and end to end through remoe_sps_query_host
(host buffers, copies included); the clustering tree (alpha = 15, beta = 150) build time
and query latency; writes profiles/<tag>_p0_latency.json.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402


def pct(v):
    return {f"p{q}": float(np.percentile(v, q)) for q in (10, 50, 90)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r02")
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    import torch
    import paper_2512_18674_b200 as remoe

    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    out = {"what": "paper scale (P:675): 5,000 history, alpha = 15, B = 1; device latency (graphed "
                   "remoe_sps_query, CUDA events) and end to end (remoe_sps_query_host, pinned host buffers)",
           "shapes": []}
    for name in ("p0_gpt2", "p0_dsv2"):
        c = gen.CONFIGS[name]
        x = gen.store_emb(c.store_seed, c.n, c.dim)
        a = gen.store_act(c.store_seed, c.n, c.layers, c.experts, c.moe_topk)
        qs = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, args.iters, mode=0)
        sps = remoe.Sps(x, a, max_batch=16, max_k=32)
        k = c.k
        ids = torch.empty((1, k), dtype=torch.int64, device=dev)
        sc = torch.empty((1, k), dtype=torch.float32, device=dev)
        pr = torch.empty((1, c.layers, c.experts), dtype=torch.float32, device=dev)
        qd = torch.from_numpy(qs.view(np.int16)).to(dev)
        qbuf = torch.empty((1, c.dim), dtype=torch.int16, device=dev)
        for i in range(10):
            qbuf.copy_(qd[i:i + 1])
            remoe.remoe_sps_query(sps.handle, qbuf, 1, k, ids, sc, pr, stream)
        torch.cuda.synchronize()
        dev_ms = []
        for i in range(args.iters):
            qbuf.copy_(qd[i:i + 1])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            remoe.remoe_sps_query(sps.handle, qbuf, 1, k, ids, sc, pr, stream)
            e1.record(stream)
            e1.synchronize()
            dev_ms.append(e0.elapsed_time(e1))
        qh = torch.from_numpy(qs.view(np.int16)).pin_memory()
        ih = torch.empty((1, k), dtype=torch.int64).pin_memory()
        sh = torch.empty((1, k), dtype=torch.float32).pin_memory()
        ph = torch.empty((1, c.layers, c.experts), dtype=torch.float32).pin_memory()
        for i in range(10):
            remoe.remoe_sps_query_host(sps.handle, qh[i:i + 1], 1, k, ih, sh, ph, stream)
        e2e_ms = []
        for i in range(args.iters):
            t0 = time.perf_counter()
            remoe.remoe_sps_query_host(sps.handle, qh[i:i + 1], 1, k, ih, sh, ph, stream)
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        info = sps.info()
        t0 = time.perf_counter()
        ti = sps.tree_build(beta=150, branching=8, max_iter=10, seed=0)
        build_s = time.perf_counter() - t0
        tree_ms = []
        for i in range(args.iters):
            qbuf.copy_(qd[i:i + 1])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sps.tree_query(qbuf, k)
            e1.record(stream)
            e1.synchronize()
            tree_ms.append(e0.elapsed_time(e1))
        r = {"shape": name, "n": c.n, "dim": c.dim, "table": f"{c.layers}x{c.experts}", "alpha": k,
             "bf_kernel": {1: "k_scan_simt (streaming)", 2: "k_scan_tc", 3: "k_scan_pair"}[info.last_scan_kernel],
             "bf_device_ms": pct(dev_ms), "bf_e2e_ms": pct(e2e_ms),
             "tree_build_s": build_s, "tree_nodes": ti.n_nodes, "tree_depth": ti.depth,
             "tree_device_ms": pct(tree_ms)}
        out["shapes"].append(r)
        print(json.dumps(r), flush=True)
        sps.close()
    out["paper"] = ("PAPER.md P:675: the clustering tree is built in <= 0.5 s and SPS is 'more than 10 times "
                    "faster than BF'; BF is the more accurate (testbed: 2x Xeon + 2x A100, P:662)")
    path = os.path.join(ROOT, "profiles", f"{args.tag}_p0_latency.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
