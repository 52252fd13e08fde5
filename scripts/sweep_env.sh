#!/bin/bash
# usage: scripts/sweep_env.sh <tag> "<ENV=..,ENV2=..>:<config>:<B>:<k>" ...   one bench line each
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for spec in "$@"; do
  IFS=: read envs cfg B k <<< "$spec"
  log=$out/b_${cfg}_${B}_${k}_${envs//[=,]/_}.log
  env ${envs//,/ } timeout 300 python bench.py --config $cfg --batch $B --k $k --steps 20 --warmup 5 --no-cpu-baseline > $log 2>&1
  echo "$spec rc=$? $(tail -1 $log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), "q/s step_ms", round(d["ms_per_step"],4), "scan_ms", round(r["kernel_ms_per_launch"],4), r["bound"], round(r["frac"],3))' 2>&1 | tail -1)"
done
