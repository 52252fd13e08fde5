#!/bin/bash
# usage: scripts/launch_list.sh <tag> "<ENV=..,..>:<config>:<B>:<k>" ...  (ncu per-launch durations)
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for spec in "$@"; do
  IFS=: read envs cfg B k <<< "$spec"
  f=$out/ll_${cfg}_${B}_${k}_${envs//[=,]/_}.csv
  env ${envs//,/ } timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
    --log-file $f python bench.py --config $cfg --batch $B --k $k --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "$spec rc=$?"
done
