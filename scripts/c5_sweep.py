#!/usr/bin/env python
"""BASELINE configs[4] (c5): the k sweep 1-128 x batch sweep 1-4096 on the c3 store
(1M x 1024, 24x60 table), one GPU, plus a forced-kernel sweep over the batch for the
resident-slab (k_scan_tc) and CTA-pair (k_scan_pair) scans, to place the HBM -> tensor
crossover.  Writes profiles/<tag>_c5_sweep.json and a markdown table next to it.

Per point: W warm-up steps, then K device-timed steps (CUDA events on the query stream,
L2 flushed between steps); the library's graphed path for the step time, and a second
pass with the live scan events for the S2+S3 phase time.  Roofline fractions use the
algorithmic bytes / flops of SURVEY §8(d) against MEASURED_PEAKS.json.

  python scripts/c5_sweep.py [--tag r02] [--steps 10] [--warmup 3] [--quick]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r02")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--cooldown", type=float, default=1.0, help="seconds idle before each point")
    args = ap.parse_args()
    import torch
    import paper_2512_18674_b200 as remoe

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm, tc = peaks["hbm_gbs"], peaks["bf16_tflops"]
    c = gen.CONFIGS["c3"]
    x = gen.store_emb(c.store_seed, c.n, c.dim)
    a = gen.store_act(c.store_seed, c.n, c.layers, c.experts, c.moe_topk)
    Bs = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]
    ks = [1, 2, 4, 8, 16, 32, 64, 128]
    if args.quick:
        Bs, ks = [1, 64, 1024], [1, 16, 128]
    sps = remoe.Sps(x, a, max_batch=1024, max_k=128)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    qall = gen.queries(c.store_seed, c.query_seed, c.n, c.dim, max(Bs), mode=0)
    q = torch.from_numpy(qall.view(np.int16)).to(dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    fl_w = torch.empty(2 * l2 // 4 + 1024, dtype=torch.int32, device=dev)
    fl_r = torch.zeros_like(fl_w)

    try:
        import pynvml
        pynvml.nvmlInit()
        nvh = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    except Exception:
        nvh = None

    def clocks():
        if nvh is None:
            return None
        return {"sm_mhz": pynvml.nvmlDeviceGetClockInfo(nvh, pynvml.NVML_CLOCK_SM),
                "reasons_mask": int(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(nvh))}

    def run_point(B, k, kernel=0):
        # cool-down: the tensor-bound points draw ~1 kW; a light point measured right after
        # one ran up to 1.6x slower on the same box (power-cap transient, scripts/r02_repro_*)
        time.sleep(args.cooldown)
        sps.set_kernel(kernel)
        ids = torch.empty((B, k), dtype=torch.int64, device=dev)
        sc = torch.empty((B, k), dtype=torch.float32, device=dev)
        pr = torch.empty((B, c.layers, c.experts), dtype=torch.float32, device=dev)
        qb = q[:B]
        for _ in range(args.warmup):
            remoe.remoe_sps_query(sps.handle, qb, B, k, ids, sc, pr, stream)

        def one_pass(profile):
            sps.profile(profile)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            for i in range(args.steps):
                fl_w.fill_(i)
                fl_r.amax()
                ev[i][0].record(stream)
                remoe.remoe_sps_query(sps.handle, qb, B, k, ids, sc, pr, stream)
                ev[i][1].record(stream)
            torch.cuda.synchronize()
            scan_ms, phases = sps.profile(False)
            return [s.elapsed_time(e) for s, e in ev], scan_ms, phases

        step, _, _ = one_pass(False)
        clk = clocks()
        _, scan_ms, phases = one_pass(True)
        info = sps.info()
        chunks = max(1, phases // args.steps)
        alg = c.n * (2 * c.dim + 4) * chunks + B * 2 * c.dim          # bytes per step
        flops = 2.0 * B * c.n * c.dim
        med = float(np.median(step))
        scan = scan_ms / args.steps
        return {
            "B": B, "k": k, "kernel": {1: "stream", 2: "tc", 3: "pair"}[info.last_scan_kernel],
            "forced": kernel != 0, "launches": info.last_launches,
            "step_ms_p10": float(np.percentile(step, 10)), "step_ms_p50": med,
            "step_ms_p90": float(np.percentile(step, 90)), "scan_ms": scan,
            "qps": B / (med / 1e3),
            "hbm_frac_scan": alg / (scan / 1e3) / 1e9 / hbm, "hbm_frac_step": alg / (med / 1e3) / 1e9 / hbm,
            "tensor_frac_scan": flops / (scan / 1e3) / 1e12 / tc,
            "tensor_frac_step": flops / (med / 1e3) / 1e12 / tc,
            "intensity_flop_per_byte": flops / alg,
            "bound_by_roofline": "tensor" if flops / alg > tc * 1e12 / (hbm * 1e9) else "hbm",
            "clocks_after_step_pass": clk,
        }

    t0 = time.time()
    pts = []
    for k in ks:
        for B in Bs:
            r = run_point(B, k)
            pts.append(r)
            print(json.dumps(r), flush=True)
    forced = []
    for B in ([64, 128, 256, 512, 1024] if not args.quick else [128, 1024]):
        for kern in (2, 3):
            r = run_point(B, 16, kern)
            forced.append(r)
            print(json.dumps(r), flush=True)
    sps.close()
    ridge = tc * 1e12 / (hbm * 1e9)
    out = {"config": "c5: c3 store (1,000,000 x 1024, table 24x60), one B200", "peaks": {"hbm_gbs": hbm,
           "bf16_tflops": tc}, "ridge_flop_per_byte": ridge, "steps": args.steps, "warmup": args.warmup,
           "l2": "flushed between steps", "points": pts, "forced_kernel": forced, "wall_s": time.time() - t0}
    # crossovers: the batch where the roofline bound switches (intensity ~ B passes the
    # ridge), and where the measured step stops being flat in B (HBM-bound: time ~ const)
    out["hbm_to_tensor_crossover_B_roofline"] = ridge
    k16 = sorted([p for p in pts if p["k"] == 16], key=lambda p: p["B"])
    base = k16[0]["step_ms_p50"] if k16 else None
    out["measured_flat_until_B"] = max([p["B"] for p in k16 if p["step_ms_p50"] <= 1.15 * base], default=None)
    path = os.path.join(ROOT, "profiles", f"{args.tag}_c5_sweep.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    with open(path.replace(".json", ".md"), "w") as f:
        f.write(f"# c5 sweep ({args.tag}): c3 store, 1 GPU; q/s (step p50), HBM / tensor fraction of the scan\n\n")
        f.write(f"ridge = {ridge:.0f} flop/byte; step = S1-S7 device time, L2 flushed between steps\n\n")
        f.write("| k \\\\ B | " + " | ".join(str(B) for B in Bs) + " |\n|" + "---|" * (len(Bs) + 1) + "\n")
        for k in ks:
            row = []
            for B in Bs:
                p = next(p for p in pts if p["B"] == B and p["k"] == k)
                fr = p["hbm_frac_scan"] if p["bound_by_roofline"] == "hbm" else p["tensor_frac_scan"]
                row.append(f"{p['qps']:.3g} ({'H' if p['bound_by_roofline'] == 'hbm' else 'T'} {fr:.2f})")
            f.write(f"| {k} | " + " | ".join(row) + " |\n")
        f.write("\nForced kernel at k = 16 (tc = resident query slab, pair = CTA pairs):\n\n"
                "| B | kernel | step ms | scan ms | HBM frac | tensor frac |\n|---|---|---|---|---|---|\n")
        for p in forced:
            f.write(f"| {p['B']} | {p['kernel']} | {p['step_ms_p50']:.3f} | {p['scan_ms']:.3f} | "
                    f"{p['hbm_frac_scan']:.2f} | {p['tensor_frac_scan']:.2f} |\n")
    print("wrote", path)


if __name__ == "__main__":
    main()
