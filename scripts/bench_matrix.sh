#!/bin/bash
# usage: scripts/bench_matrix.sh <tag> "<config:B:k:kernel> ..."   (one bench line each, short timeouts)
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
for spec in $@; do
  IFS=: read cfg B k kern <<< "$spec"
  log=$out/b_${cfg}_${B}_${k}_${kern}.log
  REMOE_VERBOSE=1 timeout 300 python bench.py --config $cfg --batch $B --k $k --kernel $kern --steps 10 --warmup 3 --no-cpu-baseline > $log 2>&1
  echo "$spec rc=$? $(tail -1 $log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), "q/s step_ms", round(d["ms_per_step"],3), "scan_ms", round(r["kernel_ms_per_launch"],3), r["bound"], round(r["frac"],3))' 2>&1 | tail -1)"
done
