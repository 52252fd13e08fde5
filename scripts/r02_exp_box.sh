#!/bin/bash
# same-box A/B of the scan's pieces: stream only, MMA only, both; plus the box's stream/UMMA micro ceilings
out=gpurun_out/${1:-r02_box}; mkdir -p $out
nvidia-smi -q -d CLOCK,POWER,PERFORMANCE > $out/smi.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bs scripts/micro/bench_stream.cu && timeout 120 /tmp/bs 2 > $out/stream.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2512_18674_b200/csrc -o /tmp/bu scripts/micro/bench_umma.cu && timeout 60 /tmp/bu > $out/umma.txt 2>&1
t() { local tag=$1; shift; env "$@" REMOE_TC_TRACE=1 timeout 120 python bench.py --config c3 --batch 64 --k 16 --steps 1 --warmup 2 --no-cpu-baseline --no-scan-events > $out/trace_$tag.log 2>&1; }
t normal
for d in 2 3 34 35; do t dbg$d REMOE_TC_DBG=$d; done
nvidia-smi -q -d CLOCK,POWER,PERFORMANCE > $out/smi_after.txt 2>&1
echo done
