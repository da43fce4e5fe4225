#!/bin/bash
# Parity tests + one bench line per config (+ the default bench line) into <outdir>.
out=${1:-gpurun_out/bench}
mkdir -p $out
timeout 600 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $out/pytest_gpu.log
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 16 2>&1 | tail -1 > $out/bench_$c.json
  python -c "import json; d=json.load(open('$out/bench_$c.json')); print('$c', round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'Gev/s', 'e2e', round(d.get('e2e',{}).get('value',0)/1e9,2), round(d.get('e2e',{}).get('ms_per_step',0),3), 'ms frac', round(d['roofline']['frac'],4), 'xu', round(d['roofline']['xu_pipe']['frac'],3), 'launches', d['gpu_launches'])" || cat $out/bench_$c.json
done
timeout 600 python bench.py > $out/bench_default.json 2> $out/bench_default.err; tail -c 400 $out/bench_default.json
