#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck over scripts/sanitize_driver.py
out=gpurun_out/${1:-r02_sanitize}; mkdir -p $out
for tool in memcheck synccheck racecheck; do
  REMOE_NO_GRAPH=1 timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_driver.py > $out/$tool.log 2>&1
  echo "$tool rc=$?" >> $out/$tool.log
done
echo done
