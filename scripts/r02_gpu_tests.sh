#!/bin/bash
# round-2 GPU check: full -m gpu suite (parity log), smoke, default bench, read-stream ceiling
out=gpurun_out/${1:-r02_t1}; mkdir -p $out
export REMOE_PARITY_LOG=$out/parity.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -rs > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 300 python bench.py > $out/bench.log 2>&1; echo "bench rc=$?" >> $out/bench.log
if [ -n "$2" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bs scripts/micro/bench_stream.cu && timeout 120 /tmp/bs 2 > $out/stream_ceiling.txt 2>&1
fi
echo done
