#!/bin/bash
# Round-2 final evidence on one GPU (summarised by scripts/summarize_profile.py):
#   suite + smoke; per config: bench line, ncu launch list, one ncu --set full capture of the scan;
#   c5 sweep, p0 latency, shard diagnostics.   usage: $0 <prefix>
pre=${1:-r02f}
root=gpurun_out; mkdir -p $root/${pre}_suite
export REMOE_PARITY_LOG=$root/${pre}_suite/parity.jsonl
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rs > $root/${pre}_suite/pytest.log 2>&1; echo "pytest rc=$?" >> $root/${pre}_suite/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $root/${pre}_suite/smoke.log 2>&1; echo "smoke rc=$?" >> $root/${pre}_suite/smoke.log
cap() {  # tag, regex, bench args...
  local tag=$1 rx=$2; shift 2; local out=$root/${pre}_$tag; mkdir -p $out
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
  timeout 400 python bench.py --json-out $out/bench.json "$@" > $out/bench.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > $out/launches.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s 2 -c 1 -o $out/scan -f \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > $out/ncu_full.log 2>&1
}
cap c3_b64 k_scan
cap c2_b16 k_scan --config c2 --batch 16 --no-cpu-baseline
cap c3_b1024 'k_scan_pair<.int.0, .int.16>' --batch 1024 --no-cpu-baseline  # not the seed-scan launch <0, 8>
cap c4_b1 k_scan --config c4 --batch 1 --k 32 --no-cpu-baseline
mkdir -p $root/${pre}_extra
line() { local tag=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --json-out $root/${pre}_extra/$tag.json "$@" > /dev/null 2>&1; }
line c3_g2 --shard-of 2; line c3_g4 --shard-of 4; line c3_g8 --shard-of 8
line c4_g8_b1 --config c4 --batch 1 --k 32 --shard-of 8; line c4_g8_b1024 --config c4 --batch 1024 --k 32 --shard-of 8
line c2_b64 --config c2 --batch 64; line c2_b256 --config c2 --batch 256; line c3_b1 --batch 1; line c3_b64_k128 --k 128
timeout 600 python scripts/p0_latency.py --tag ${pre} > $root/${pre}_extra/p0.log 2>&1
timeout 1800 python scripts/c5_sweep.py --tag ${pre} > $root/${pre}_extra/c5.log 2>&1
cp profiles/${pre}_* $root/${pre}_extra/ 2>/dev/null
ls $root/${pre}_*
