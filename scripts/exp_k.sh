#!/bin/bash
# k > 32 breakdown at c3 B=64: bench lines, phase trace, insert stats, launch list.
out=gpurun_out/expk; mkdir -p $out
bash scripts/sweep_env.sh expk ":c3:64:16" ":c3:64:32" ":c3:64:33" ":c3:64:64" ":c3:64:128" ":c3:1:128" ":c3:1024:128" > $out/sweep.txt 2>&1
for k in 32 64 128; do
  REMOE_TC_TRACE=1 REMOE_TC_STATS=1 timeout 120 python bench.py --config c3 --batch 64 --k $k --steps 1 --warmup 3 --no-cpu-baseline > $out/trace_$k.log 2>&1
done
bash scripts/launch_list.sh expk ":c3:64:128" ":c3:64:32" > $out/ll.txt 2>&1
