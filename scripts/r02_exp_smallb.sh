#!/bin/bash
# A/B: small-batch unseeded regression (c3, B 1/8/16, k 2/16): current tree vs round-1 final (old_r1/)
out=gpurun_out/${1:-r02_smallb}; mkdir -p $out
b() { local dir=$1 tag=$2; shift 2; (cd $dir && env "$@" timeout 180 python bench.py --config c3 --batch $B --k $K --steps 10 --warmup 3 --no-cpu-baseline) 2>&1 | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d['roofline']; print('$tag B=$B k=$K step %.4f scan %.4f frac %.3f' % (d['ms_per_step'], r['kernel_ms_per_launch'], r['frac']))
except Exception as e: print('$tag B=$B k=$K failed', e)
" >> $out/res.txt; }
for B in 1 16; do for K in 2 16; do
  b . cur; b old_r1 old; b . cur_seed REMOE_SEED=1; b . cur_nofold REMOE_SEED_INKERNEL=0
done; done
B=1 K=16; b . cur_stats REMOE_TC_STATS=1 REMOE_VERBOSE=1
(cd . && REMOE_TC_STATS=1 REMOE_VERBOSE=1 timeout 120 python bench.py --config c3 --batch 1 --k 16 --steps 2 --warmup 1 --no-cpu-baseline > $out/stats.log 2>&1)
cat $out/res.txt
