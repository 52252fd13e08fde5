#!/bin/bash
out=gpurun_out/${1:-r02_box3}; mkdir -p $out
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config c3 --batch $B --k 16 --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
B=64
t dbg34 REMOE_TC_DBG=34
t dbg2 REMOE_TC_DBG=2
t normal
B=1
t b1_normal
t b1_dbg34 REMOE_TC_DBG=34
echo done
