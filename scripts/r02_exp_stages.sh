#!/bin/bash
# ring depth (REMOE_TC_MAX_STAGES) at small B; effective SM clock in the scan (trace)
out=gpurun_out/${1:-r02_stages}; mkdir -p $out
b() { local tag=$1; shift; env "$@" timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$tag.log 2>&1; }
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
CFG=c3 K=16
for B in 1 16 32; do for ms in 6 8 12; do b B${B}_ms$ms REMOE_TC_MAX_STAGES=$ms; done; done
B=64
b B64; t B64; t B64_dbg2 REMOE_TC_DBG=2; t B64_dbg3 REMOE_TC_DBG=3
B=1; t B1_ms12; t B1_ms6 REMOE_TC_MAX_STAGES=6
echo done
