timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/m4_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/m4_parity.log
bash scripts/bench_matrix.sh m4 c3:1024:64:pair c3:1024:128:pair c3:64:64:tc c3:64:128:tc c3:1024:16:pair c3:4096:128:pair c3:1:128:tc
