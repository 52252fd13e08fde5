#!/bin/bash
# in-kernel seeding: parity suite, then phase traces / DBG knobs on c3 B=64 and c2 B=16
out=gpurun_out/${1:-r02_seed}; mkdir -p $out
export REMOE_PARITY_LOG=$out/parity.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -rs > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
for spec in "c3 64 16" "c2 16 10" "c2 64 10" "c3 64 128"; do
  set -- $spec
  REMOE_TC_TRACE=1 timeout 120 python bench.py --config $1 --batch $2 --k $3 --steps 1 --warmup 3 --no-cpu-baseline > $out/trace_$1_$2_$3.log 2>&1
  timeout 120 python bench.py --config $1 --batch $2 --k $3 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$1_$2_$3.log 2>&1
done
for d in 1 2; do
  REMOE_TC_DBG=$d REMOE_TC_TRACE=1 timeout 120 python bench.py --config c3 --batch 64 --k 16 --steps 1 --warmup 3 --no-cpu-baseline > $out/trace_dbg$d.log 2>&1
done
for ns in 4 5; do
  REMOE_TC_STAGES=$ns timeout 120 python bench.py --config c3 --batch 64 --k 16 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_st$ns.log 2>&1
done
echo done
