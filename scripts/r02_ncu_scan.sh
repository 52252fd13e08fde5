#!/bin/bash
# ncu --set full of the c3 B=64 k=16 scan: in-kernel seeding, launch seeding (main scan), DBG=2
out=gpurun_out/${1:-r02_ncu}; mkdir -p $out
for cfg in "ink:REMOE_SEED_INKERNEL=1" "launch:REMOE_SEED_INKERNEL=0" "dbg2:REMOE_TC_DBG=2" "dbg6:REMOE_TC_DBG=6"; do
  tag=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan_tc -s 3 -c 1 \
      -o $out/scan_$tag python bench.py --config c3 --batch 64 --k 16 --steps 1 --warmup 1 --no-cpu-baseline --no-scan-events > $out/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
done
env REMOE_TC_DBG=6 timeout 120 python bench.py --config c3 --batch 64 --k 16 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_dbg6.log 2>&1
echo done
