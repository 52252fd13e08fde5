#!/bin/bash
# quick check after a scan change: c2 trace + stats, bench lines (c2 B=16/64, c3 B=1/64), parity subset
out=gpurun_out/${1:-r02_quick}; mkdir -p $out
REMOE_TC_TRACE=1 REMOE_NO_GRAPH=1 timeout 120 python bench.py --config c2 --batch 16 --k 10 --steps 1 --warmup 1 --no-cpu-baseline --no-scan-events 2>&1 | grep -A17 "tc trace" | tail -18 > $out/trace_c2_16.txt
REMOE_TC_STATS=1 REMOE_NO_GRAPH=1 timeout 120 python bench.py --config c2 --batch 16 --k 10 --steps 1 --warmup 1 --no-cpu-baseline --no-scan-events 2>&1 | grep "tc stats" | tail -1 > $out/stats_c2_16.txt
for spec in c2:16:10 c2:64:10 c3:1:16 c3:64:16 ${EXTRA}; do
  IFS=: read cfg B K <<< "$spec"
  timeout 200 python bench.py --config $cfg --batch $B --k $K --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d['roofline']; print('$spec step %.4f p50 %.4f scan %.4f frac %.3f e2e %.0f' % (d['ms_per_step'], d['ms_per_step_pct']['p50'], r['kernel_ms_per_launch'], r['frac'], d['e2e']['value']))
except Exception as e: print('$spec failed', e)
" >> $out/bench.txt
done
# TESTS: test files (default tests/), KEXPR: a pytest -k expression
if [ -n "$TESTS$KEXPR" ]; then
  timeout 1200 python -m pytest ${TESTS:-tests} -m gpu -q -x --timeout 600 ${KEXPR:+-k "$KEXPR"} > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
fi
cat $out/trace_c2_16.txt $out/stats_c2_16.txt $out/bench.txt; tail -3 $out/pytest.log 2>/dev/null
