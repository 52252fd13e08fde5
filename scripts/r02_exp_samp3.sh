#!/bin/bash
out=gpurun_out/${1:-r02_samp3}; mkdir -p $out
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
CFG=c2 B=16 K=10; t nowait REMOE_TC_DBG=256; t relaxed REMOE_TC_DBG=512; t nowait_nomma REMOE_TC_DBG=257; t seedoff REMOE_SEED=0
echo done
