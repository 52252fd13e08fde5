#!/bin/bash
# sel32 change: gpu tests, c3 B=64 evidence, B=1024 (pair scan), k=128
o=gpurun_out/r1s6c; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $o/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
timeout 900 bash scripts/round_profile.sh r1s6c/c3_b64
timeout 400 python bench.py --steps 20 --warmup 5 --config c3 --batch 1024 --no-cpu-baseline > $o/c3_b1024.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --config c3 --batch 64 --k 128 --no-cpu-baseline > $o/c3_b64_k128.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --config c2 --batch 16 --no-cpu-baseline > $o/c2_b16.log 2>&1
