#!/usr/bin/env python
"""Turn a gpurun_out/<tag>/ evidence directory (scripts/round_profile.sh) into the
committed summaries under profiles/: the per-launch list (ncu gpu__time_duration,
cold-cache and serialised -> compare shares), key metrics of the full ncu capture
of the scan kernel, and the per-launch DRAM traffic bench.py reports.

usage: python scripts/summarize_profile.py <tag> <round, e.g. r01>
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEY_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__cycles_active.avg", "sm__cycles_elapsed.avg",
    "smsp__inst_executed.sum", "l1tex__m_l1tex2xbar_req_cycles_active_op_tma.sum",
]


def launches(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    per = OrderedDict()
    for r in rd:
        key = (r["ID"], r["Kernel Name"])
        per.setdefault(key, {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
    for (i, name), m in per.items():
        t, unit = m.get("gpu__time_duration.sum", ("0", "ns"))
        t = float(t.replace(",", "")) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1.0)
        rb = float(m.get("dram__bytes_read.sum", ("0", ""))[0].replace(",", "") or 0)
        wb = float(m.get("dram__bytes_write.sum", ("0", ""))[0].replace(",", "") or 0)
        scale = lambda v, u: v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        rb = scale(rb, m.get("dram__bytes_read.sum", ("", "byte"))[1])
        wb = scale(wb, m.get("dram__bytes_write.sum", ("", "byte"))[1])
        rows.append((int(i), name.split("(")[0], t, rb, wb))
    return rows


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return {}
    h, u = r[0], r[1]
    # several captured launches (e.g. the threshold-seeding scan and the main scan): keep the longest
    it = h.index("gpu__time_duration.sum")
    v = max(r[2:], key=lambda row: float(row[it].replace(",", "") or 0))
    res = OrderedDict()
    for name in KEY_METRICS:
        if name in h:
            i = h.index(name)
            res[name] = (v[i], u[i])
    res["Kernel Name"] = (v[h.index("Kernel Name")], "") if "Kernel Name" in h else ("?", "")
    return res


def to_bytes(val, unit):
    v = float(str(val).replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    tag, rnd = sys.argv[1], sys.argv[2]
    src = os.path.join(ROOT, "gpurun_out", tag)
    dst = os.path.join(ROOT, "profiles")
    os.makedirs(dst, exist_ok=True)
    bench = json.load(open(os.path.join(src, "bench.json")))
    lines = []
    lines.append(f"# {rnd} {tag}: evidence summary\n")
    lines.append("bench.py line (device-timed, CUDA events, L2 flushed between steps):\n")
    lines.append("```json\n" + json.dumps(bench, indent=1) + "\n```\n")
    if os.path.exists(os.path.join(src, "gpu.txt")):
        lines.append("GPU: `" + open(os.path.join(src, "gpu.txt")).read().strip().replace("\n", " | ") + "`\n")
    L = launches(os.path.join(src, "launches.csv"))
    with open(os.path.join(dst, f"{rnd}_{tag}_launches.csv"), "w") as f:
        f.write("id,kernel,duration_us,dram_read_bytes,dram_write_bytes\n")
        for i, n, t, rb, wb in L:
            f.write(f"{i},{n},{t:.3f},{rb:.0f},{wb:.0f}\n")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for _, n, t, _, _ in L:
        tot[n] += t
        cnt[n] += 1
    allt = sum(tot.values())
    lines.append("\n## Launch list share (ncu --metrics gpu__time_duration.sum --clock-control none)\n")
    lines.append("Cold-cache, serialised per-launch times of the whole bench process (setup + warm-up +"
                 " steps); compare SHARES with bench.py's kernel_share_of_step, not absolutes.\n")
    lines.append("| kernel | launches | total us | share |\n|---|---|---|---|")
    for n in sorted(tot, key=lambda x: -tot[x]):
        lines.append(f"| `{n}` | {cnt[n]} | {tot[n]:.1f} | {tot[n] / allt:.3f} |")
    M = full_metrics(os.path.join(src, "scan.ncu-rep"))
    if M:
        lines.append("\n## Full capture of one scan launch (ncu --set full --clock-control none)\n")
        lines.append(f"Kernel: `{M['Kernel Name'][0]}`\n")
        lines.append("| metric | value | unit |\n|---|---|---|")
        for k_, (v, u) in M.items():
            if k_ != "Kernel Name":
                lines.append(f"| `{k_}` | {v} | {u} |")
        traffic = to_bytes(*M["dram__bytes_read.sum"]) + to_bytes(*M["dram__bytes_write.sum"])
        alg = bench["roofline"]["algorithmic_bytes_per_launch"]
        lines.append(f"\nDRAM traffic per launch {traffic:.4g} B vs algorithmic {alg:.4g} B "
                     f"(ratio {traffic / alg:.4f}).\n")
        tpath = os.path.join(dst, "traffic.json")
        tj = json.load(open(tpath)) if os.path.exists(tpath) else {}
        c = bench["config"]
        sk = c.get("scan_kernel", "")
        kern = 3 if "pair" in sk else 2 if "tc" in sk else 1
        tj[f"c{c['workload'].split(':')[0][1:]}:B{c['batch']}:k{c['k']}:G{bench['n_gpus']}:{kern}"] = traffic
        json.dump(tj, open(tpath, "w"), indent=1, sort_keys=True)
    with open(os.path.join(dst, f"{rnd}_{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
