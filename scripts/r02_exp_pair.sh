#!/bin/bash
out=gpurun_out/${1:-r02_pair}; mkdir -p $out
b() { local tag=$1; shift; env "$@" timeout 180 python bench.py --config c3 --batch $B --k $K --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_$tag.log 2>&1; }
K=16
for B in 128 256 1024; do b B$B; done
B=1024 K=128; b B1024_k128
B=64 K=128; b B64_k128; b B64_k128_s1 REMOE_SEED_SEGS=1; b B64_k128_s4 REMOE_SEED_SEGS=4; b B64_k128_launch REMOE_SEED_INKERNEL=0
B=64 K=32; b B64_k32
B=64 K=64; b B64_k64
B=16 K=16; b B16
B=32 K=16; b B32
timeout 120 python bench.py --config c2 --batch 16 --k 10 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_c2_16.log 2>&1
timeout 120 python bench.py --config c2 --batch 64 --k 10 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_c2_64.log 2>&1
timeout 120 python bench.py --config c2 --batch 256 --k 10 --steps 20 --warmup 5 --no-cpu-baseline > $out/bench_c2_256.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu --timeout 600 -k "pair or c5 or c4 or seeded" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
echo done
