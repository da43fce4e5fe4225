#!/bin/bash
# compute-sanitizer over tools/sanitize_smoke.py: memcheck for each small-frame kernel
# (8 / 4 / 2 lanes per ray), racecheck / synccheck / initcheck once.  usage: bash tools/sanitize_all.sh out.txt
out=${1:-gpurun_out/sanitizer.txt}
: > $out
for env in "" "FVSRN_OCTO_FRAC=0" "FVSRN_OCTO_FRAC=0 FVSRN_QUAD_FRAC=0"; do
  echo "memcheck ${env:-(default)}:" >> $out
  env $env timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_smoke.py 2>&1 | grep -E "ERROR SUMMARY|smoke done|Error" | head -5 >> $out
done
for tool in racecheck synccheck initcheck; do
  echo "$tool:" >> $out
  timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_smoke.py 2>&1 | grep -E "SUMMARY|smoke done|Error" | head -5 >> $out
done
cat $out
