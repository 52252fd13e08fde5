mkdir -p gpurun_out/exp3
ncu --set full --import-source on --sampling-interval 0 --clock-control none -k regex:k_merge -s 3 -c 1 -o gpurun_out/exp3/merge -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config c2 --batch 1 --k 10 > /dev/null 2>&1
