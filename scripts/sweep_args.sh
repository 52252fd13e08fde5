#!/bin/bash
# usage: scripts/sweep_args.sh <tag> "<bench args>" ...   (one bench line each)
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
i=0
for a in "$@"; do
  i=$((i+1)); log=$out/a$i.log
  timeout 300 python bench.py $a --steps 20 --warmup 5 --no-cpu-baseline > $log 2>&1
  echo "$a rc=$? $(tail -1 $log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), "q/s step_ms", round(d["ms_per_step"],4), "scan_ms", round(r["kernel_ms_per_launch"],4), "e2e", round(d["e2e"]["value"]))' 2>&1 | tail -1)"
done
