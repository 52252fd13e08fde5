#!/bin/bash
# stage-ring depth sweep (REMOE_TC_STAGES caps the ring of 32 KB unit stages)
out=gpurun_out/${1:-r02_stages}; mkdir -p $out
for r in 1 2; do
for spec in ${SPECS:-c3:1:16 c3:16:16 c3:32:16 c2:16:10 c2:64:10 c4:1:32 c3:16:128}; do
  IFS=: read cfg B K <<< "$spec"
  for v in ${VALS:-2 3 4 6}; do
    REMOE_TC_STAGES=$v timeout 200 python bench.py --config $cfg --batch $B --k $K --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d['roofline']; print('$spec'.ljust(10), 'stages $v', 'step %.4f p50 %.4f scan %.4f frac %.3f' % (d['ms_per_step'], d['ms_per_step_pct']['p50'], r['kernel_ms_per_launch'], r['frac']))
except Exception as e: print('$spec $v failed', e)
" >> $out/stages.txt
  done
done; done
cat $out/stages.txt
