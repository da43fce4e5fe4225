#!/usr/bin/env bash
# Stages the UNMODIFIED reference package (fvsrn 0.1.0, /root/reference/pkg) into
# oracle/_ref so bench.py's CPU legs (--impl reference, cpu_baseline) can run the real
# reference on the GPU box, where /root/reference does not exist.  Test infrastructure:
# oracle/_ref is git-ignored (never committed) but not gpurun-ignored (it travels with
# the snapshot like the built .so).  The reference source tree is read-only, so the
# build runs from a copy under /tmp; dependencies (numpy, scipy, numba, Pillow) are the
# image's own.  No-op when /root/reference is absent (e.g. on the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "stage_ref: $SRC absent, keeping $HERE/_ref as is"; exit 0; }
TMP="$(mktemp -d /tmp/fvsrn_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg"
echo "stage_ref: fvsrn staged into $HERE/_ref"
