"""bench.py's multi-rank path on one GPU (FVSRN_BENCH_ONE_GPU=1: every rank on cuda:0 over
gloo): `--gpus 2` re-launches itself under torch.distributed.run, renders with the
peer-memory frame (default) and with the NCCL-style gather + reassembly
(FVSRN_MULTI=gather), and the assembled frame must be bit-identical to a 1-GPU render."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["peer", "gather"])
def test_bench_two_ranks_one_gpu(mode):
    env = dict(os.environ, FVSRN_BENCH_ONE_GPU="1", FVSRN_MULTI=mode)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "cfg1",
                        "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--check-frame"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["config"]["frame_bit_identical_to_1gpu"] is True
    assert line["value"] > 0 and line["e2e"]["value"] > 0
