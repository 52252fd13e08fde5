mkdir -p gpurun_out/exp3
ncu --set full --clock-control none --import-source on -k regex:k_scan -s 3 -c 1 -o gpurun_out/exp3/b64 -f \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --batch 64 > gpurun_out/exp3/b64.log 2>&1
ls -la gpurun_out/exp3
