#!/bin/bash
# Round-2 check: -m gpu suite, smoke, default bench, per-GPU shard diagnostics (c3 at G = 2/4/8,
# c4 at G = 8: the north star's 10M store over 8 GPUs), c2 lines.  usage: $0 <tag>
out=gpurun_out/${1:-r02_round}; mkdir -p $out
export REMOE_PARITY_LOG=$out/parity.jsonl
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 -rs > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 300 python bench.py --json-out $out/bench.json > $out/bench.log 2>&1; echo "bench rc=$?" >> $out/bench.log
line() { local tag=$1; shift; timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --json-out $out/$tag.json "$@" > $out/$tag.log 2>&1
  python -c "
import json; d=json.load(open('$out/$tag.json')); r=d['roofline']
print('%-22s step p50 %.4f ms  scan %.4f ms  %s frac %.3f  e2e %.0f q/s  value %.0f q/s' % ('$tag', d['ms_per_step_pct']['p50'], r['kernel_ms_per_launch'], r['bound'], r['frac'], d['e2e']['value'], d['value']))" >> $out/lines.txt 2>&1; }
line c3_g2 --shard-of 2
line c3_g4 --shard-of 4
line c3_g8 --shard-of 8
line c4_g8_b1 --config c4 --batch 1 --k 32 --shard-of 8
line c4_g8_b1024 --config c4 --batch 1024 --k 32 --shard-of 8
line c4_g1_b1 --config c4 --batch 1 --k 32
line c2_b16 --config c2 --batch 16
line c2_b64 --config c2 --batch 64
line c2_b256 --config c2 --batch 256
line c3_b1024 --batch 1024
cat $out/lines.txt; tail -2 $out/pytest.log; cat $out/smoke.log
