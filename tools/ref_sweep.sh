#!/bin/bash
# Thread settings of the reference's CPU path on this box (bench.py REF_BEST): one bench
# step of each config through oracle/ref_runner.py per candidate
# (render_image threads, NUMBA_NUM_THREADS, BLAS threads).
C=$(nproc)
run() {  # config threads numba blas stride
  r=$(env NUMBA_NUM_THREADS=$3 OMP_NUM_THREADS=$4 OPENBLAS_NUM_THREADS=$4 MKL_NUM_THREADS=$4 \
      timeout 300 python -m oracle.ref_runner --config $1 --threads $2 --row-stride $5 2>/dev/null | tail -1)
  echo "$1 threads=$2 numba=$3 blas=$4: $(echo $r | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,3), "M evals/s", d["kind"], d["sample"])' 2>/dev/null || echo failed)"
}
echo "cores $C, $(grep -m1 'model name' /proc/cpuinfo)"
for cfg in "cfg1 8" "cfg2 16" "cfg5 256" "cfg3 128"; do
  set -- $cfg
  for cand in "$C 1 1" "$C 1 $C" "1 $C $C" "4 4 4" "8 2 2" "1 1 $C"; do
    run $1 $cand $2
  done
done
for cand in "1 $C $C" "1 $C 1" "1 1 $C"; do
  r=$(env NUMBA_NUM_THREADS=$(echo $cand | cut -d' ' -f2) OMP_NUM_THREADS=$(echo $cand | cut -d' ' -f3) OPENBLAS_NUM_THREADS=$(echo $cand | cut -d' ' -f3) timeout 300 python -m oracle.ref_runner --config cfg4 --threads 1 --row-stride 16 | tail -1)
  echo "cfg4 $cand: $r"
done
