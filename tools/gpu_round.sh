#!/bin/bash
# One GPU-box pass: parity tests, bench lines for every config, the ncu launch list of
# the default bench command, and full ncu captures of the dominant kernels.
# usage: bash tools/gpu_round.sh <outdir>   (outdir under gpurun_out/)
out=${1:-gpurun_out/round}
mkdir -p $out
timeout 600 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $out/pytest_gpu.log
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 16 2>&1 | tail -1 > $out/bench_$c.json
  python -c "import json; d=json.load(open('$out/bench_$c.json')); print('$c', round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'Gev/s', 'e2e', round(d.get('e2e',{}).get('value',0)/1e9,2), 'frac', round(d['roofline']['frac'],4), 'xu', round(d['roofline']['xu_pipe']['frac'],3), 'launches', d['gpu_launches'])" || cat $out/bench_$c.json
done
timeout 600 python bench.py > $out/bench_default.json 2> $out/bench_default.err; tail -c 600 $out/bench_default.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:dvr_kernel -s 3 -c 1 --export $out/ncu_dvr_cfg2 -f python bench.py --config cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:dvr_tc_kernel -s 3 -c 1 --export $out/ncu_tc_cfg3 -f python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:sample_kernel -s 3 -c 1 --export $out/ncu_decode_cfg4 -f python bench.py --config cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls $out
