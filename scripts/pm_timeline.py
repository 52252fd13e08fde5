"""Print the PM-sampling timeline (DRAM throughput, tensor pipe, issue) of an ncu report:
python scripts/pm_timeline.py report.ncu-rep [bins]"""
import sys
sys.path.insert(0, "/opt/nvidia/nsight-compute/2025.2.1/extras/python")
import ncu_report

ctx = ncu_report.load_report(sys.argv[1])
bins = int(sys.argv[2]) if len(sys.argv) > 2 else 40
a = ctx.range_by_idx(0).action_by_idx(0)
keys = {"dram%": "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "tensor%": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "inst%": "TPC.TriageCompute.sm__inst_executed_realtime.avg.pct_of_peak_sustained_elapsed",
        "l2hit%": "LTS.TriageCompute.lts__average_t_sector_hit_rate_realtime.pct"}
series = {}
for k, n in keys.items():
    m = a.metric_by_name(n)
    series[k] = [m.as_double(i) for i in range(m.num_instances())]
n = len(series["dram%"])
print(a.name(), "samples", n)
step = max(1, n // bins)
print("bin  " + "  ".join(f"{k:>8}" for k in keys))
for b in range(0, n, step):
    print(f"{b:4d} " + "  ".join(f"{sum(series[k][b:b+step])/len(series[k][b:b+step]):8.1f}" for k in keys))
