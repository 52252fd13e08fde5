#!/bin/bash
out=gpurun_out/${1:-r02_samp2}; mkdir -p $out
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
CFG=c2 B=16 K=10; t c2_16_notmem REMOE_TC_DBG=128; t c2_16_nomma REMOE_TC_DBG=1
echo done
