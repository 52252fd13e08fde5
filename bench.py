#!/usr/bin/env python
"""SPS benchmark (driver contract).

A step = one pass of the whole hot path (S1-S7: query norms, similarity scan with
fused top-k, local merge, [cross-rank merge + row exchange], softmax + weighted
reduce) over one batch of B synthetic queries against the whole store, through
the C ABI, inputs resident in HBM.  Default workload: BASELINE config c3
(1M prompts x 1024, Qwen1.5-MoE 24x60 table, B=64, k=16) -- the config the
metric "SPS queries/s at 1/2/4/8 B200" is quoted on.  With N GPUs the store is
sharded row-wise (strong scaling: N_total fixed), queries are replicated.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--batch B] [--k K]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
  python bench.py --impl reference      # the oracle (CPU), same config/metric
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gen  # noqa: E402

METRIC = "SPS queries/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(gen.CONFIGS))
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--kernel", default="auto", choices=["auto", "stream", "tc", "pair"])
    ap.add_argument("--no-flush", action="store_true", help="do not flush L2 between steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-scan-events", action="store_true",
                    help="debug: no per-scan CUDA events inside the timed steps (no roofline)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--shard-of", type=int, default=1,
                    help="N = 1 only: run the step on shard 0 of a G-way row split (the per-GPU "
                         "work of G GPUs: S1-S7 on that shard, no exchange); a diagnostic line")
    ap.add_argument("--exchange", default="fused", choices=["fused", "nccl"],
                    help="N > 1: the fused peer-memory exchange (DESIGN.md §8; falls back to NCCL "
                         "if a rank cannot map its peers) or NCCL collectives")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks sampler

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.dev)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ helpers

def workload(cfg, B, k):
    return {"workload": f"{cfg.name}: {cfg.n:,} prompts x D={cfg.dim}, table {cfg.layers}x{cfg.experts}"
                        f" (MoE top-{cfg.moe_topk}), batch {B}, k={k}",
            "n_prompts": cfg.n, "dim": cfg.dim, "layers": cfg.layers, "experts": cfg.experts,
            "batch": B, "k": k}


def algorithmic_bytes_per_launch(n_loc, D, nq):
    """S2 scan: the store rows + their fp32 norms + the queries of the launch
    (SURVEY §8(d) per-unit figure N_loc*(2D+4), x units = rows of the shard)."""
    return n_loc * (2 * D + 4) + nq * 2 * D


def algorithmic_flops_per_launch(n_loc, D, nq):
    """S2 scan: 2*D flops per (query, row) pair; the Eq. 11 scaling and the
    top-k compare are O(1) per pair and not counted."""
    return 2.0 * nq * n_loc * D


def cpu_baseline(cfg, B, k, seconds, x, a):
    """The oracle as it stands, on this host's cores, on a bounded sample."""
    import oracle
    qs = gen.queries(cfg.store_seed, cfg.query_seed, cfg.n, cfg.dim, max(B, 1), mode=0)
    t0 = time.perf_counter()
    oracle.sps(qs[:1], x, a, k)
    t1 = time.perf_counter() - t0
    n = int(max(1, min(B, seconds / max(t1, 1e-6))))
    t0 = time.perf_counter()
    oracle.sps(qs[:n], x, a, k)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "queries/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"{n} of the {B} queries of one batch against the full {cfg.n:,}-row store "
                      f"(fp64 C oracle, {os.cpu_count()} threads, {dt:.2f} s)"}


# ------------------------------------------------------------------ reference arm (oracle)

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    cfg = gen.CONFIGS[args.config]
    B = args.batch or cfg.batch
    k = args.k or cfg.k
    x = gen.store_emb(cfg.store_seed, cfg.n, cfg.dim)
    a = gen.store_act(cfg.store_seed, cfg.n, cfg.layers, cfg.experts, cfg.moe_topk)
    qs = gen.queries(cfg.store_seed, cfg.query_seed, cfg.n, cfg.dim, B, mode=0)
    # per-step sample sized from one probe so that warmup+steps ends within minutes
    t0 = time.perf_counter()
    oracle.sps(qs[:1], x, a, k)
    t1 = time.perf_counter() - t0
    budget = 150.0 / max(1, args.steps + args.warmup)
    nq = int(max(1, min(B, budget / max(t1, 1e-6))))
    for i in range(args.warmup):
        oracle.sps(qs[:nq], x, a, k)
    t0 = time.perf_counter()
    for i in range(args.steps):
        oracle.sps(qs[(i * nq) % B:][:nq] if B - (i * nq) % B >= nq else qs[:nq], x, a, k)
    dt = time.perf_counter() - t0
    value = nq * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {**workload(cfg, B, k), "sample_queries_per_step": nq},
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": os.cpu_count(),
                         "kind": "oracle",
                         "sample": f"{nq} queries per step of the {B}-query batch, full store"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2512_18674_b200 as remoe

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ["REMOE_FUSED_COMM"] = "1" if args.exchange == "fused" else "0"  # read at build
        dist.init_process_group("nccl", device_id=dev)
    cfg = gen.CONFIGS[args.config]
    B = args.batch or cfg.batch
    k = args.k or cfg.k
    off, n_loc = gen.shard_range(cfg.n, world, rank)
    if args.shard_of > 1:
        if world > 1:
            raise SystemExit("--shard-of is a one-GPU diagnostic")
        off, n_loc = gen.shard_range(cfg.n, args.shard_of, 0)

    # ---- inputs: this rank's shard, generated on the host, copied into HBM at build
    x = gen.store_emb(cfg.store_seed, cfg.n, cfg.dim, off, n_loc)
    a = gen.store_act(cfg.store_seed, cfg.n, cfg.layers, cfg.experts, cfg.moe_topk, off, n_loc)
    if world > 1:
        from paper_2512_18674_b200.dist import build_sharded
        sps = build_sharded(x, a, cfg.n, device=local, max_batch=max(B, 1), max_k=max(k, 1))
    else:  # (with --shard-of: the shard alone, as a one-rank store of n_loc rows)
        sps = remoe.Sps(x, a, max_batch=max(B, 1), max_k=max(k, 1), device=local)
    if args.kernel != "auto":
        sps.set_kernel({"stream": remoe.KERNEL_STREAM, "tc": remoe.KERNEL_TC,
                        "pair": remoe.KERNEL_PAIR}[args.kernel])

    # a rotating pool of distinct query batches (fresh cluster members)
    pool = 4
    qall = gen.queries(cfg.store_seed, cfg.query_seed, cfg.n, cfg.dim, B * pool, mode=0)
    qdev = [torch.from_numpy(qall[i * B:(i + 1) * B].view(np.int16)).to(dev) for i in range(pool)]
    ids = torch.empty((B, k), dtype=torch.int64, device=dev)
    scores = torch.empty((B, k), dtype=torch.float32, device=dev)
    pred = torch.empty((B, cfg.layers, cfg.experts), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.empty(2 * l2 // 4 + 1024, dtype=torch.int32, device=dev)
    # the write pass leaves L2 full of dirty lines whose write-back would otherwise land
    # inside the next step; a read pass over a second 2xL2 buffer evicts them before the
    # step starts, so every step begins with a clean, cold L2 (as after a previous
    # read-only query).  (The ~50 MB of scan DRAM writes ncu showed were the scan's own
    # local-memory stores, fixed by sel32 in common.cuh, not this.)
    flush_rd = torch.zeros(2 * l2 // 4 + 1024, dtype=torch.int32, device=dev)
    flush = not args.no_flush

    def flush_l2(i):
        flush_buf.fill_(i)
        flush_rd.amax()

    def step(i):
        remoe.remoe_sps_query(sps.handle, qdev[i % pool], B, k, ids, scores, pred, stream)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)

    # ---- timed region: K steps, per-step CUDA events (L2 flushed between steps, outside the
    # events).  Pass 1 is the headline: the library's normal path (one-chunk device queries
    # replay a cached CUDA graph).  Pass 2 repeats the K steps with the library's live scan
    # timing on (CUDA events around the S2+S3 phase on the query stream; the graph is off
    # while events are recorded) for the roofline's kernel time and its share of the step.
    def interleaved_passes():
        """The graphed steps (value) and the profiled steps (live scan events, graphs off) in
        ONE loop, alternating which comes first: both see the same power/thermal state (a
        c4 run hit sw_power_cap during a second, separate pass and its kernel time came out
        17% above the first pass's whole step)."""
        g_start = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        g_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        p_start = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        p_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        scan_total, scan_l = 0.0, 0
        g_launches = 0
        barrier()
        torch.cuda.synchronize(dev)
        for i in range(args.steps):
            for mode in ((0, 1) if i % 2 == 0 else (1, 0)):
                if flush:
                    flush_l2(i)
                if mode == 0:
                    g_start[i].record(stream)
                    step(i)
                    g_end[i].record(stream)
                    g_launches = sps.info().last_launches
                elif not args.no_scan_events:
                    sps.profile(True)
                    p_start[i].record(stream)
                    step(i)
                    p_end[i].record(stream)
                    torch.cuda.synchronize(dev)
                    ms, nl = sps.profile(False)
                    scan_total += ms
                    scan_l += nl
        torch.cuda.synchronize(dev)
        barrier()
        g = [s.elapsed_time(e) for s, e in zip(g_start, g_end)]
        pr = [s.elapsed_time(e) for s, e in zip(p_start, p_end)] if not args.no_scan_events else g
        return g, pr, (scan_total, scan_l), g_launches

    clocks = ClockSampler(local)
    clocks.start()
    step_ms, prof_step_ms, (scan_ms, scan_launches), launches_per_step = interleaved_passes()
    clk = clocks.stop()
    total_ms = float(sum(step_ms))
    t = torch.tensor([total_ms, scan_ms, float(sum(prof_step_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, scan_ms_max, prof_total_ms = float(t[0]), float(t[1]), float(t[2])
    value = B * args.steps / (total_ms / 1e3)
    pct = {f"p{q}": float(np.percentile(step_ms, q)) for q in (10, 50, 90)}

    # ---- end to end through the public host API: pinned host in, host out, synced
    q_host = torch.from_numpy(qall[:B].view(np.int16)).pin_memory()
    ids_h = torch.empty((B, k), dtype=torch.int64).pin_memory()
    sc_h = torch.empty((B, k), dtype=torch.float32).pin_memory()
    pr_h = torch.empty((B, cfg.layers, cfg.experts), dtype=torch.float32).pin_memory()
    for i in range(max(1, args.warmup // 2)):
        remoe.remoe_sps_query_host(sps.handle, q_host, B, k, ids_h, sc_h, pr_h, stream)
    e2e_ms = []
    barrier()
    for i in range(args.steps):
        if flush:
            flush_l2(i)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        remoe.remoe_sps_query_host(sps.handle, q_host, B, k, ids_h, sc_h, pr_h, stream)
        s1.record(stream)
        s1.synchronize()
        e2e_ms.append(s0.elapsed_time(s1))
    barrier()
    te = torch.tensor([float(sum(e2e_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = B * args.steps / (float(te[0]) / 1e3)

    info = sps.info()
    kern = {1: "k_scan_simt (CUDA cores, TMA bulk staging)", 2: "k_scan_tc (tcgen05 + TMA)",
            3: "k_scan_pair (tcgen05 cta_group::2 + TMA)"}.get(info.last_scan_kernel, "?")
    per_launch_ms = max(scan_ms_max / max(1, scan_launches), 1e-9)
    nq_per_launch = B / max(1, scan_launches // max(1, args.steps))
    alg = algorithmic_bytes_per_launch(n_loc, cfg.dim, nq_per_launch)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    tc_peak = peaks.get("bf16_tflops", 2250.0)
    achieved = alg / (per_launch_ms / 1e3) / 1e9
    flops = algorithmic_flops_per_launch(n_loc, cfg.dim, nq_per_launch)
    # the bound: arithmetic intensity (flop per algorithmic byte, ~B) against the ridge
    tensor_bound = flops / alg > tc_peak * 1e12 / (hbm_peak * 1e9)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"{cfg.name}:B{B}:k{k}:G{world}:{info.last_scan_kernel}")
    except (OSError, ValueError):
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "ms_per_step_pct": pct, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (clustered bf16 embeddings, Zipf activation tables; gen/)",
        "config": {**workload(cfg, B, k), "parallelism": f"store row-sharded x{world}",
                   **({"exchange": "fused peer-memory (CUDA IPC over NVLink)" if info.fused_exchange
                       else "NCCL collectives"} if world > 1 else {}),
                   **({"shard": f"diagnostic: shard 0 of {args.shard_of} ({n_loc:,} rows) alone on one GPU -- "
                                f"the per-GPU scan work of {args.shard_of} GPUs, S1-S7 without the exchanges"}
                      if args.shard_of > 1 else {}),
                   "l2": "flushed between steps (write 2xL2, then read 2xL2: cold and clean)" if flush else "not flushed",
                   "scan_kernel": kern},
        "roofline": ({"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                      "frac": achieved / hbm_peak, "traffic": traffic,
                      "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650"}
                     if not tensor_bound else
                     {"bound": "tensor", "achieved": flops / (per_launch_ms / 1e3) / 1e12, "peak": tc_peak,
                      "unit": "TFLOP/s", "frac": flops / (per_launch_ms / 1e3) / 1e12 / tc_peak,
                      "traffic": traffic,
                      "frac_of_sustained": flops / (per_launch_ms / 1e3) / 1e12
                      / peaks.get("bf16_tflops_sustained", tc_peak),
                      "hbm_achieved_gbs": achieved,
                      "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" if peaks
                      else "fallback 2250 (nominal)"}) | {
                     "kernel": kern, "kernel_ms_per_launch": per_launch_ms,
                     "algorithmic_bytes_per_launch": alg, "algorithmic_flops_per_launch": flops,
                     "kernel_share_of_step": scan_ms_max / max(prof_total_ms, 1e-9),
                     "frac_of_nominal_8tbs": achieved / 8000.0,
                     "step_frac_of_peak": ((alg * max(1, scan_launches // max(1, args.steps)))
                                           / (total_ms / args.steps / 1e3) / 1e9 / hbm_peak),
                     "timing": "kernel time from pass 2 (live CUDA events around the scan phase, "
                               "graphs off); value from pass 1 (the library's graphed path)"},
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": B * cfg.dim * 2,
                "d2h_bytes_per_step": B * k * 12 + B * cfg.layers * cfg.experts * 4},
        "gpu_launches": launches_per_step * args.steps,
        "profiled_ms_per_step": prof_total_ms / args.steps,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, B, k, args.cpu_seconds, x, a)
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                json.dump(line, f, indent=1)
    sps.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
