#!/bin/bash
# pair scan L2 sensitivity: skip the query (128) or store (256) box loads after the first tile (wrong results)
for B in 256 1024; do for d in 0 128 256 384; do
  REMOE_TC_DBG=$d timeout 200 python bench.py --config c3 --batch $B --k 16 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; print('B=$B dbg=$d step %.4f scan %.4f frac %.3f %s' % (d['ms_per_step'], r['kernel_ms_per_launch'], r['frac'], r['bound']))"
done; done
