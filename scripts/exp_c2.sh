#!/bin/bash
# small-store fixed costs at c2: seeded vs unseeded, phase trace
out=gpurun_out/expc2; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
bash scripts/sweep_env.sh expc2 ":c2:1:10" ":c2:8:10" "REMOE_SEED=0:c2:8:10" ":c2:16:10" ":c2:64:10" ":c2:256:10" ":c3:64:16" ":c3:64:128" ":c3:1024:16" > $out/sweep.txt 2>&1
REMOE_TC_TRACE=1 timeout 120 python bench.py --config c2 --batch 16 --steps 1 --warmup 3 --no-cpu-baseline > $out/trace_16.log 2>&1
