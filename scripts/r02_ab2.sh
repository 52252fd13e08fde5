#!/bin/bash
# A/B the working tree against old_head/ on a list of bench argument sets (alternating, 2 reps)
for rep in 1 2; do
for a in "$@"; do
  for dir in . old_head; do
    (cd $dir && timeout 200 python bench.py --no-cpu-baseline --steps 20 --warmup 5 $a) 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$dir'.ljust(9), '$a'.ljust(28), 'step p50 %.4f scan %.4f frac %.3f' % (d['ms_per_step_pct']['p50'], r['kernel_ms_per_launch'], r['frac']))"
  done
done; done
