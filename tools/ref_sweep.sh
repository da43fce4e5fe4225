#!/bin/bash
# Thread settings of the reference's CPU path on this box (bench.py REF_BEST): one bench
# step of each config (the same row sample the bench uses) through oracle/ref_runner.py per
# candidate (render_image threads, NUMBA_NUM_THREADS, BLAS threads).
C=$(python -c 'import os; print(len(os.sched_getaffinity(0)))')
H=$((C / 2)); Q=$((C / 4)); [ $Q -lt 1 ] && Q=1
echo "cores $C, $(grep -m1 'model name' /proc/cpuinfo)"
run() {  # config threads numba blas stride
  r=$(env NUMBA_NUM_THREADS=$3 OMP_NUM_THREADS=$4 OPENBLAS_NUM_THREADS=$4 MKL_NUM_THREADS=$4 \
      timeout 400 python -m oracle.ref_runner --config $1 --threads $2 $5 2>/dev/null | tail -1)
  echo "$1 threads=$2 numba=$3 blas=$4: $(echo $r | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), "M evals/s", round(d["seconds"],1), "s", d["sample"])' 2>/dev/null || echo failed)"
}
for cfg in "cfg1 --full" "cfg2 --row-stride=2" "cfg5 --row-stride=64" "cfg3 --row-stride=64"; do
  set -- $cfg
  for cand in "$C 1 1" "1 $C $C" "$H 2 2" "$Q 4 4" "1 1 $C"; do
    run $1 $cand $2
  done
done
for cand in "1 $C $C" "1 1 $C" "1 $C 1"; do
  run cfg4 $cand --row-stride=16
done
