#!/bin/bash
# MMA-latency hypothesis (DBG bits) + the epilogue's seeded-threshold wait
out=gpurun_out/${1:-r02_mma}; mkdir -p $out
b() { local tag=$1; shift; env "$@" timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$tag.log 2>&1; }
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
CFG=c3 B=64 K=16
for d in 2 3 10 18 26; do b dbg$d REMOE_TC_DBG=$d; done
b ink REMOE_SEED_INKERNEL=1; t ink REMOE_SEED_INKERNEL=1
b launch REMOE_SEED_INKERNEL=0
CFG=c3 B=64 K=128
b k128_ink; t k128_ink
CFG=c2 B=16 K=10
b c2_16_ink; t c2_16_ink
b c2_16_launch REMOE_SEED_INKERNEL=0
CFG=c3 B=1 K=16
b c3_1
echo done
