"""Reproduce the c5-sweep slowdown: time c3 B=1 k=2 before and after other (B, k) points on one handle."""
import os, sys, json
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen
import paper_2512_18674_b200 as remoe

c = gen.CONFIGS["c3"]
x = gen.store_emb(c.store_seed, c.n, c.dim)
a = gen.store_act(c.store_seed, c.n, c.layers, c.experts, c.moe_topk)
sps = remoe.Sps(x, a, max_batch=1024, max_k=128)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
q = torch.from_numpy(gen.queries(c.store_seed, c.query_seed, c.n, c.dim, 4096, mode=0).view(np.int16)).to(dev)

def run(B, k, n=10):
    ids = torch.empty((B, k), dtype=torch.int64, device=dev)
    sc = torch.empty((B, k), dtype=torch.float32, device=dev)
    pr = torch.empty((B, c.layers, c.experts), dtype=torch.float32, device=dev)
    ts = []
    for i in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        remoe.remoe_sps_query(sps.handle, q[:B], B, k, ids, sc, pr, st)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[2:])), ids.cpu().numpy(), sc.cpu().numpy()

seq = [(1, 2), (64, 1), (1, 2), (1024, 1), (1, 2), (2048, 1), (1, 2), (4096, 1), (1, 2), (8, 16), (256, 2), (1, 2)]
ref = None
for B, k in seq:
    ms, ids, sc = run(B, k)
    note = ""
    if (B, k) == (1, 2):
        if ref is None: ref = (ids, sc)
        else: note = "ids_same=%s" % np.array_equal(ids, ref[0])
    print(f"B={B} k={k} ms={ms:.4f} kernel={sps.info().last_scan_kernel} {note}", flush=True)
