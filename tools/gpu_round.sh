#!/bin/bash
# One GPU-box pass: bench lines for every config (with CPU baselines of the reference,
# benchmark.csv + manifest), the reference arm, a 2-rank one-GPU bench line (multi-rank
# code path), the ncu launch list of the default bench command and full ncu captures of
# the dominant kernels (raw + source pages).
# usage: bash tools/gpu_round.sh <outdir>   (outdir under gpurun_out/)
out=${1:-gpurun_out/round}
mkdir -p $out
for c in cfg1 cfg3 cfg4 cfg5 cfg2; do
  timeout 900 python bench.py --config $c --steps 16 --csv $out/benchmark.csv 2> $out/bench_$c.err | tail -1 > $out/bench_$c.json
  python -c "import json; d=json.load(open('$out/bench_$c.json')); print('$c', round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'Gev/s', 'e2e', round(d.get('e2e',{}).get('value',0)/1e9,2), round(d.get('e2e',{}).get('ms_per_step',0),3), 'ms frac', round(d['roofline']['frac'],4), 'xu', round(d['roofline']['xu_pipe']['frac'],3), 'cpu', d.get('cpu_baseline',{}).get('value'), d.get('cpu_baseline',{}).get('kind'))" || tail -3 $out/bench_$c.err
done
timeout 600 python bench.py > $out/bench_default.json 2> $out/bench_default.err; tail -c 300 $out/bench_default.json; echo
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > $out/bench_reference.json 2> $out/bench_reference.err; tail -c 400 $out/bench_reference.json; echo
FVSRN_BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 8 --check-frame --no-cpu-baseline > $out/bench_2ranks_onegpu.json 2> $out/bench_2ranks.err; tail -c 300 $out/bench_2ranks_onegpu.json; echo
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# full captures of each config's dominant kernel (the one bench.py reports in roofline.kernel)
for spec in "cfg2:dvr_tc_kernel" "cfg3:dvr_tc_kernel" "cfg5:dvr_tc_kernel" "cfg1:dvr_pair_kernel" "cfg4:decode_tc_kernel"; do
  c=${spec%%:*}; k=${spec#*:}
  timeout 400 ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 --export $out/ncu_$c -f python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  ncu -i $out/ncu_$c.ncu-rep --page raw --csv > $out/ncu_${c}_raw.csv 2>/dev/null
  ncu -i $out/ncu_$c.ncu-rep --page source --csv --print-source sass > $out/ncu_${c}_src.csv 2>/dev/null
  rm -f $out/ncu_$c.ncu-rep
done
ls $out
