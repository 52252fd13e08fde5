#!/bin/bash
# refresh the secondary evidence on the sel32 kernels
timeout 600 bash scripts/round_profile.sh r1s6d/c3_b1024 --config c3 --batch 1024
timeout 600 bash scripts/round_profile.sh r1s6d/c3_b64_k128 --config c3 --batch 64 --k 128
timeout 400 bash scripts/round_profile.sh r1s6d/c2_b16 --config c2 --batch 16
timeout 300 python bench.py --steps 20 --warmup 5 --config c3 --batch 1 --no-cpu-baseline > gpurun_out/r1s6d/c3_b1.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --config c3 --batch 256 --no-cpu-baseline > gpurun_out/r1s6d/c3_b256.log 2>&1
