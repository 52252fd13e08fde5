#!/bin/bash
out=gpurun_out/${1:-r02_seed4}; mkdir -p $out
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
b() { local tag=$1; shift; env "$@" timeout 180 python bench.py --config $CFG --batch $B --k $K --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$tag.log 2>&1; }
CFG=c2 B=16 K=10; t c2_16; b c2_16
CFG=c2 B=64 K=10; t c2_64; b c2_64
CFG=c3 B=64 K=16; t c3_64; b c3_64
CFG=c3 B=64 K=128; b c3_64_128; b c3_64_128_launch REMOE_SEED_INKERNEL=0
CFG=c3 B=1 K=16; b c3_1
CFG=tiny B=16 K=5; b tiny
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -x -m gpu --timeout 600 > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
echo done
