#!/bin/bash
# Collect the round's evidence on one GPU: bench line, launch list, one full ncu capture of the scan.
# usage: scripts/round_profile.sh <tag> [bench args]
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
python bench.py --steps 20 --warmup 5 --json-out $out/bench.json "$@" > $out/bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > $out/launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_scan -s 6 -c 2 -o $out/scan -f \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > $out/ncu_full.log 2>&1
ls -la $out
