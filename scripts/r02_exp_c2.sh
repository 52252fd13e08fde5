#!/bin/bash
out=gpurun_out/${1:-r02_c2}; mkdir -p $out
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config $CFG --batch $B --k $K --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
b() { local tag=$1; shift; env "$@" timeout 180 python bench.py --config $CFG --batch $B --k $K --steps 20 --warmup 5 --no-cpu-baseline "${EXTRA[@]}" > $out/bench_$tag.log 2>&1; }
CFG=c2 B=16 K=10; t c2_16; t c2_16_noseed REMOE_SEED=0; b c2_16_noseed REMOE_SEED=0
CFG=c2 B=64 K=10; t c2_64
CFG=c3 B=128 K=16; EXTRA=(--kernel tc); b c3_128_tc; EXTRA=(--kernel pair); b c3_128_pair
CFG=c3 B=256 K=16; EXTRA=(--kernel tc); b c3_256_tc; EXTRA=(--kernel pair); b c3_256_pair
EXTRA=()
for spec in "c3 64 16" "c2 16 10"; do
  set -- $spec
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/ll_$1_$2.csv python bench.py --config $1 --batch $2 --k $3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
echo done
