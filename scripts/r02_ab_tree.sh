#!/bin/bash
# A/B the working tree against old_head/ (a worktree of the previous commit, built), alternating
# on the same box.  usage: scripts/r02_ab_tree.sh outdir "cfg:B:k ..."
out=gpurun_out/${1:-r02_ab}; mkdir -p $out
specs=${2:-"c3:64:16 c3:32:16 c3:1:16 c2:16:10 c2:64:10 c3:64:128"}
for r in 1 2; do
for spec in $specs; do
  IFS=: read cfg B K <<< "$spec"
  for dir in . old_head; do
    (cd $dir && timeout 200 python bench.py --config $cfg --batch $B --k $K --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null) | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d['roofline']; print('$spec'.ljust(10), '$dir'.ljust(9), 'step %.4f p50 %.4f scan %.4f frac %.3f' % (d['ms_per_step'], d['ms_per_step_pct']['p50'], r['kernel_ms_per_launch'], r['frac']))
except Exception as e: print('$spec $dir failed', e)
" >> $out/ab.txt
  done
done; done
if [ -n "$TESTS$KEXPR" ]; then
  timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q -x --timeout 600 ${KEXPR:+-k "$KEXPR"} > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
fi
cat $out/ab.txt; tail -3 $out/pytest.log 2>/dev/null
