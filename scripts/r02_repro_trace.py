"""Trace c3 B=1 k=2 scan phases before/after a chunked B=4096 query (REMOE_TC_TRACE=1 REMOE_NO_GRAPH=1)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen
import paper_2512_18674_b200 as remoe

c = gen.CONFIGS["c3"]
x = gen.store_emb(c.store_seed, c.n, c.dim)
a = gen.store_act(c.store_seed, c.n, c.layers, c.experts, c.moe_topk)
sps = remoe.Sps(x, a, max_batch=int(os.environ.get("MB", "1024")), max_k=128)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
q = torch.from_numpy(gen.queries(c.store_seed, c.query_seed, c.n, c.dim, 4096, mode=0).view(np.int16)).to(dev)

def run(B, k, n):
    ids = torch.empty((B, k), dtype=torch.int64, device=dev)
    sc = torch.empty((B, k), dtype=torch.float32, device=dev)
    pr = torch.empty((B, c.layers, c.experts), dtype=torch.float32, device=dev)
    for i in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        remoe.remoe_sps_query(sps.handle, q[:B], B, k, ids, sc, pr, st)
        e1.record(st)
        torch.cuda.synchronize()
        print(f"B={B} k={k} ms={e0.elapsed_time(e1):.4f}", file=sys.stderr, flush=True)

import subprocess, time
for arg in ["1,2,3"] + sys.argv[1:] + ["1,2,3"]:
    if arg.startswith("sleep"):
        time.sleep(float(arg[5:]))
        continue
    if arg == "smi":
        print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_throttle_reasons.active",
                              "--format=csv,noheader"], capture_output=True, text=True).stdout.strip(), file=sys.stderr)
        continue
    B, k, n = map(int, arg.split(","))
    run(B, k, n)
