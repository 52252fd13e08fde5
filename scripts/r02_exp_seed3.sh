#!/bin/bash
# in-kernel seeding (seeding warp) vs launch seeding; the in-kernel stream ceiling (DBG=3)
out=gpurun_out/${1:-r02_seed3}; mkdir -p $out
run() { # tag env...
  local tag=$1; shift
  env "$@" timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$tag.log 2>&1
  env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1
}
CFG=c3 B=64 K=16
run c3_64_16_ink REMOE_SEED_INKERNEL=1
run c3_64_16_launch REMOE_SEED_INKERNEL=0
run c3_dbg3 REMOE_TC_DBG=3
run c3_dbg2 REMOE_TC_DBG=2
CFG=c3 B=1 K=16
run c3_1_16_ink REMOE_SEED_INKERNEL=1
run c3_1_16_seed REMOE_SEED=1
CFG=c3 B=64 K=128
run c3_64_128_ink REMOE_SEED_INKERNEL=1
run c3_64_128_launch REMOE_SEED_INKERNEL=0
CFG=c2 B=16 K=10
run c2_16_10_ink REMOE_SEED_INKERNEL=1
run c2_16_10_launch REMOE_SEED_INKERNEL=0
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -m gpu -q -x --timeout 500 > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
echo done
