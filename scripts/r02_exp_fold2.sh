#!/bin/bash
out=gpurun_out/${1:-r02_fold2}; mkdir -p $out
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
b() { local tag=$1; shift; env "$@" timeout 180 python bench.py --config $CFG --batch $B --k $K --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$tag.log 2>&1; }
CFG=c2 B=16 K=10; t c2_16; b c2_16
CFG=c3 B=64 K=16; t c3_64; b c3_64
CFG=c3 B=1 K=16; b c3_1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_merge -s 2 -c 1 -o $out/merge_c3 python bench.py --config c3 --batch 64 --k 16 --steps 1 --warmup 1 --no-cpu-baseline --no-scan-events > $out/ncu_merge.log 2>&1
timeout 900 python -m pytest tests -q -x -m gpu --timeout 800 > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
echo done
