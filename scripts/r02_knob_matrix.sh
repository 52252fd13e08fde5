#!/bin/bash
# The parity subset of tests/test_gpu_parity.py (no full-size configs) under each alternative
# launch path / experiment knob; every line must pass.   usage: $0 <outfile under gpurun_out>
out=gpurun_out/${1:-r02_knob_matrix.log}; : > $out
for kv in REMOE_TC_TILED=0 REMOE_SEED=1 REMOE_SEED=0 REMOE_NO_MULTICAST=1 REMOE_NO_GRAPH=1 \
          REMOE_SEED_INKERNEL=0 REMOE_PAIR_LOCKSTEP=1 REMOE_TC_STAGES=2 REMOE_SEED_UNITS_PER_K=1; do
  echo "== $kv" >> $out
  env $kv timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 300 \
      -k "not c3 and not c4 and not c5 and not p0" 2>&1 | tail -1 >> $out
done
cat $out
