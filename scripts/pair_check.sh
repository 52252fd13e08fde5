#!/bin/bash
# CTA-pair scan: parity first (short timeouts: a pipeline deadlock must not hang the box), then timings.
out=gpurun_out/pair; mkdir -p $out
timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "pair and tiny" > $out/t_tiny.log 2>&1; echo "tiny rc=$?"
tail -3 $out/t_tiny.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pair" > $out/t_pair.log 2>&1; echo "pair rc=$?"
tail -3 $out/t_pair.log
for B in 256 1024 4096; do
  for kern in tc pair; do
    REMOE_VERBOSE=1 timeout 300 python bench.py --batch $B --kernel $kern --steps 10 --warmup 3 --no-cpu-baseline > $out/b_${B}_${kern}.log 2>&1
    echo "B=$B $kern rc=$? $(tail -1 $out/b_${B}_${kern}.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]), "q/s scan_ms", round(r["kernel_ms_per_launch"],3), r["bound"], round(r["frac"],3))' 2>&1 | tail -1)"
  done
done
