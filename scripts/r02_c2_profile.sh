#!/bin/bash
# c2 (100k x 768) small-store breakdown: bench lines, launch lists, per-CTA phase trace
out=gpurun_out/${1:-r02_c2}; mkdir -p $out
for B in 1 16 64 256; do
  timeout 200 python bench.py --config c2 --batch $B --k 10 --steps 20 --warmup 5 --no-cpu-baseline --json-out $out/bench_B$B.json > $out/bench_B$B.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file $out/ll_B$B.csv \
     python bench.py --config c2 --batch $B --k 10 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
REMOE_TC_TRACE=1 REMOE_NO_GRAPH=1 timeout 120 python bench.py --config c2 --batch 16 --k 10 --steps 2 --warmup 1 --no-cpu-baseline --no-scan-events > $out/trace_B16.log 2>&1
REMOE_TC_TRACE=1 REMOE_NO_GRAPH=1 REMOE_SEED=0 timeout 120 python bench.py --config c2 --batch 16 --k 10 --steps 2 --warmup 1 --no-cpu-baseline --no-scan-events > $out/trace_B16_noseed.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 6 -c 1 -o $out/scan_B16 -f \
    python bench.py --config c2 --batch 16 --k 10 --steps 2 --warmup 3 --no-cpu-baseline > $out/ncu_full.log 2>&1
echo done
