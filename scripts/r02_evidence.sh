#!/bin/bash
# Round-2 evidence on one GPU: -m gpu suite, smoke, default bench, launch list, one full ncu
# capture of the scan, then c5 sweep, p0 latency and the sanitizers.  usage: $0 <tag> [sweep]
tag=${1:-r02_ev}; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
export REMOE_PARITY_LOG=$out/parity.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -rs > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 300 python bench.py --json-out $out/bench.json > $out/bench.log 2>&1; echo "bench rc=$?" >> $out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $out/launches.log 2>&1
echo "launches rc=$?" >> $out/launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 6 -c 1 -o $out/scan -f \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $out/ncu_full.log 2>&1
echo "ncu rc=$?" >> $out/ncu_full.log
if [ -n "$2" ]; then
  timeout 600 python scripts/p0_latency.py --tag $tag > $out/p0.log 2>&1; echo "p0 rc=$?" >> $out/p0.log
  timeout 1200 python scripts/c5_sweep.py --tag $tag > $out/c5.log 2>&1; echo "c5 rc=$?" >> $out/c5.log
  cp profiles/${tag}_* $out/ 2>/dev/null
  bash scripts/sanitize.sh $tag/san
fi
ls -la $out
