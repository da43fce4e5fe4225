#!/bin/bash
# A/B bench of library variants on the GPU box: tools/ab.sh "cfg2 cfg3" default build/libfvsrn_x.so ...
cfgs=$1; shift
for lib in "$@"; do
  for c in $cfgs; do
    if [ "$lib" = default ]; then L=""; else L=$lib; fi
    FVSRN_LIB=$L python bench.py --config $c --no-cpu-baseline --no-e2e --steps 16 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$c', round(d['ms_per_step'],3), 'ms', round(d['value']/1e9,2), 'Gev/s')" || echo "$lib $c FAILED"
  done
done
