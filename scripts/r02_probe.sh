#!/bin/bash
# round-2 baseline probe: phase traces of the current scans (c2 B=16/64, c3 B=64) and a c2 launch list
out=gpurun_out/r02_probe; mkdir -p $out
nvidia-smi > $out/smi.txt 2>&1
for spec in "c2 16 10" "c2 64 10" "c3 64 16" "c3 1 16"; do
  set -- $spec
  REMOE_TC_TRACE=1 timeout 120 python bench.py --config $1 --batch $2 --k $3 --steps 1 --warmup 3 --no-cpu-baseline > $out/trace_$1_$2.log 2>&1
  timeout 120 python bench.py --config $1 --batch $2 --k $3 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$1_$2.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/ll_c2_16.csv python bench.py --config c2 --batch 16 --k 10 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
