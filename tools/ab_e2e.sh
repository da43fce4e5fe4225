#!/bin/bash
# A/B of device and end-to-end ms/frame: tools/ab_e2e.sh "cfg1 cfg2" "FVSRN_X=0" "FVSRN_X=1" ...
cfgs=$1; shift
for ent in "$@"; do
  for c in $cfgs; do
    envs=(); IFS=',' read -ra parts <<< "$ent"
    for p in "${parts[@]}"; do case "$p" in default) ;; *) envs+=("$p") ;; esac; done
    timeout 180 env "${envs[@]}" python bench.py --config $c --no-cpu-baseline --steps 30 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$ent', '$c', round(d['ms_per_step'],3), 'ms  e2e', round(d['e2e']['ms_per_step'],3), 'ms')" || echo "$ent $c FAILED"
  done
done
