"""cuBLAS ceiling for the pair scan's contraction shape: Q [B x D] @ X^T [D x N] in bf16
(fp32 accumulate, bf16 out -- the library GEMM alone, no top-k), c3 shape N = 1M, D = 1024,
B in {256, 512, 1024}; CUDA events, best and median of 20.  Context for the pair scan's
tensor fraction (profiles/r02_cublas_shape.json)."""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
dev = torch.device("cuda", 0)
N, D = 1_000_000, 1024
X = torch.randn(N, D, device=dev, dtype=torch.bfloat16)
out = {"what": __doc__.strip().splitlines()[0], "N": N, "D": D, "points": []}
for B in (256, 512, 1024, 2048):
    Q = torch.randn(B, D, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(Q, X.t())
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(Q, X.t()); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    fl = 2.0 * B * N * D
    p = {"B": B, "best_ms": ts[0], "median_ms": ts[len(ts) // 2], "tflops_best": fl / ts[0] / 1e9,
         "tflops_median": fl / ts[len(ts) // 2] / 1e9}
    out["points"].append(p)
    print(json.dumps(p), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "cublas_shape.json"), "w"), indent=1)
