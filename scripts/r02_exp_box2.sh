#!/bin/bash
out=gpurun_out/${1:-r02_box2}; mkdir -p $out
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config c3 --batch 64 --k 16 --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
t dbg34 REMOE_TC_DBG=34
t dbg34_sleep REMOE_TC_DBG=34 REMOE_EPI_SLEEP=1
t dbg2 REMOE_TC_DBG=2
t dbg2_sleep REMOE_TC_DBG=2 REMOE_EPI_SLEEP=1
t normal
t normal_sleep REMOE_EPI_SLEEP=1
t noseed_dbg34 REMOE_TC_DBG=34 REMOE_SEED=0
echo done
