#!/bin/bash
# One GPU call: full gpu tests, smoke, and the default-config evidence.
mkdir -p gpurun_out/r1s6
nvidia-smi > gpurun_out/r1s6/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r1s6/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1s6/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s6/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1s6/smoke.log
timeout 900 bash scripts/round_profile.sh r1s6/c3_b64
timeout 600 bash scripts/round_profile.sh r1s6/c3_b64_k128 --config c3 --batch 64 --k 128
timeout 600 bash scripts/round_profile.sh r1s6/c2_b16 --config c2 --batch 16
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1s6/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/r1s6/bench_ref.log
