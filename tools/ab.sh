#!/bin/bash
# A/B bench on the GPU box: tools/ab.sh "cfg2 cfg3" default build/libfvsrn_x.so FVSRN_WS=0 "FVSRN_WS=0,build/libfvsrn_x.so" ...
# Each entry: "default", a library path, ENV=value settings, or a comma-separated mix.
cfgs=$1; shift
for ent in "$@"; do
  for c in $cfgs; do
    envs=(); L=""
    IFS=',' read -ra parts <<< "$ent"
    for p in "${parts[@]}"; do
      case "$p" in default) ;; *=*) envs+=("$p") ;; *) L=$p ;; esac
    done
    timeout 120 env "${envs[@]}" FVSRN_LIB=$L python bench.py --config $c --no-cpu-baseline --no-e2e --steps 16 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$ent', '$c', round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'Gev/s', d['clocks'].get('sm_mhz'))" || echo "$ent $c FAILED"
  done
done
