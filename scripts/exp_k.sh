#!/bin/bash
# k > 32 at c3: parity of the large-k paths, then bench lines and a launch list.
out=gpurun_out/expk; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "large_k or c5 or k_sweep or tiny or small_stores" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
bash scripts/sweep_env.sh expk ":c3:64:16" ":c3:64:32" ":c3:64:33" ":c3:64:64" ":c3:64:128" ":c3:1:128" ":c3:1024:128" ":c2:16:10" > $out/sweep.txt 2>&1
bash scripts/launch_list.sh expk ":c3:64:128" ":c3:64:64" > $out/ll.txt 2>&1
