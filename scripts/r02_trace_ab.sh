#!/bin/bash
# REMOE_TC_TRACE phase stamps of one c2 B=16 query, working tree vs old_head/
out=gpurun_out/${1:-r02_trace_ab}; mkdir -p $out
for dir in . old_head; do
  specs=${2:-"c2:16:10 c3:64:16"}
  for spec in $specs; do
    IFS=: read cfg B K <<< "$spec"
    echo "== $dir $spec" >> $out/trace.txt
    (cd $dir && REMOE_TC_TRACE=1 REMOE_NO_GRAPH=1 timeout 120 python bench.py --config $cfg --batch $B --k $K --steps 1 --warmup 1 --no-cpu-baseline --no-scan-events 2>&1) | grep -A19 "tc trace" | tail -20 >> $out/trace.txt
  done
done
cat $out/trace.txt
