#!/bin/bash
# A/B the working tree against old_head/ (a worktree of HEAD), alternating, same box
for rep in 1 2; do
for dir in . old_head; do
  for a in "--config c2 --batch 16" "--batch 64"; do
    (cd $dir && timeout 200 python bench.py --no-cpu-baseline --steps 30 --warmup 5 $a) 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$dir'.ljust(9), '$a'.ljust(24), 'step p50 %.4f scan %.4f frac %.3f' % (d['ms_per_step_pct']['p50'], r['kernel_ms_per_launch'], r['frac']))"
  done
done; done
