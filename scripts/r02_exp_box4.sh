#!/bin/bash
out=gpurun_out/${1:-r02_box4}; mkdir -p $out
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config c3 --batch $B --k 16 --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
b() { local tag=$1; shift; env "$@" timeout 120 python bench.py --config c3 --batch $B --k 16 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$tag.log 2>&1; }
B=64
t dbg34 REMOE_TC_DBG=34
t dbg2 REMOE_TC_DBG=2
t dbg3 REMOE_TC_DBG=3
t normal
b normal
b launch REMOE_SEED_INKERNEL=0
B=1
t b1
b b1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x -m gpu --timeout 600 > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
echo done
