#!/bin/bash
# in-kernel vs launch seeding, phase traces and insert stats
out=gpurun_out/${1:-r02_seed2}; mkdir -p $out
run() { # tag env... -- config B k
  local tag=$1; shift
  env "$@" timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$tag.log 2>&1
  env "$@" REMOE_TC_TRACE=1 REMOE_TC_STATS=1 timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1
}
CFG=c3 B=64 K=16
run c3_64_16_ink REMOE_SEED_INKERNEL=1
run c3_64_16_launch REMOE_SEED_INKERNEL=0
run c3_64_16_noseed REMOE_SEED=0
CFG=c3 B=64 K=128
run c3_64_128_ink REMOE_SEED_INKERNEL=1
run c3_64_128_launch REMOE_SEED_INKERNEL=0
CFG=c2 B=16 K=10
run c2_16_10_ink REMOE_SEED_INKERNEL=1
run c2_16_10_launch REMOE_SEED_INKERNEL=0
CFG=c3 B=64 K=16
run c3_dbg1 REMOE_TC_DBG=1
run c3_dbg2 REMOE_TC_DBG=2
echo done
