#!/bin/bash
# A/B of one environment knob on the same box: each spec alternates knob on / off R times.
# usage: KNOB=REMOE_TC_HIROWS ON=1 OFF=0 scripts/r02_ab_knob.sh outdir "c3:64:16 c2:16:10 ..."
out=gpurun_out/${1:-r02_ab}; mkdir -p $out
specs=${2:-"c3:64:16 c3:32:16 c3:16:16 c3:1:16 c2:16:10 c2:64:10 c3:64:128"}
for r in 1 2; do
for spec in $specs; do
  IFS=: read cfg B K <<< "$spec"
  for v in $ON $OFF; do
    env $KNOB=$v timeout 200 python bench.py --config $cfg --batch $B --k $K --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d['roofline']; print('$spec $KNOB=$v step %.4f p50 %.4f scan %.4f frac %.3f' % (d['ms_per_step'], d['ms_per_step_pct']['p50'], r['kernel_ms_per_launch'], r['frac']))
except Exception as e: print('$spec $KNOB=$v failed', e)
" >> $out/ab.txt
  done
done
done
if [ -n "$TESTS$KEXPR" ]; then
  timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -q -x --timeout 600 ${KEXPR:+-k "$KEXPR"} > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
fi
cat $out/ab.txt; tail -3 $out/pytest.log 2>/dev/null
