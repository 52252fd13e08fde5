#!/bin/bash
out=gpurun_out/${1:-r02_samp}; mkdir -p $out
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
CFG=c2 B=16 K=10; t c2_16; t c2_16_noins REMOE_TC_DBG=64
CFG=c3 B=64 K=16; t c3_64
echo done
