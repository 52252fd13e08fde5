#!/bin/bash
# usage: scripts/profile_tc.sh <tag> [bench args...]   (run under gpurun; 1 GPU)
tag=$1; shift
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 \
    -o gpurun_out/prof_$tag -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/prof_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/launches_$tag.log 2>&1
