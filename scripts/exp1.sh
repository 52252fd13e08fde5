mkdir -p gpurun_out/exp1
i=0
run() { i=$((i+1)); timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/exp1/r$i.json "$@" > gpurun_out/exp1/r$i.log 2>&1; python -c "import json,sys; d=json.load(open('gpurun_out/exp1/r$i.json')); r=d['roofline']; print('$*', '| scan ms', round(r['kernel_ms_per_launch'],4), 'frac', round(r['frac'],3), '| step ms', round(d['ms_per_step'],4), 'q/s', round(d['value']))" 2>/dev/null || (echo "FAIL $*"; grep -v '^\s*$' gpurun_out/exp1/r$i.log | tail -3); }
