"""CPU legs of bench.py (the reference arm and ``cpu_baseline``) -- TEST INFRASTRUCTURE ONLY.

Runs the UNMODIFIED reference package staged into ``oracle/_ref`` by
``oracle/stage_ref.sh`` (fvsrn 0.1.0 from /root/reference/pkg, pip-installed with the
image's numpy/scipy/numba) through its own public functions, exactly as its
``render_image`` composes them (render.py:314-332): ``camera_rays`` for the frame, the
rays split into ``threads * 4`` chunks on a ``ThreadPoolExecutor``, each chunk through
``render_rays`` -> ``raymarch_forward`` with ``ModelSource(model, tf, use_fused=True)``
(``use_fused=False`` for 6x64, whose fused plan raises CapacityError, fused.py:84-89).
``decode_volume`` (model.py:385-398) is called as is.  The evaluated-sample count is
the reference's own: ``ModelSource.sample`` calls.

A bounded sample of a frame is a deterministic set of its rows (every k-th row): rays
are independent, so those rows cost and evaluate exactly what they do inside the full
frame.  When ``oracle/_ref`` is absent the numpy/numba port ``oracle/fvsrn_oracle.py``
runs instead and the result says ``kind: "port"``.

Only bench.py calls this module (in-process for the reference arm, as a subprocess
under ``taskset`` for the single-core figure).  The product package never imports it.

    python -m oracle.ref_runner --config cfg2 --threads 1 --row-stride 64 --step 0
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"

# BASELINE.json configs (same as bench.CONFIGS; duplicated so the subprocess needs no torch)
CONFIGS = {
    "cfg1": dict(model=dict(layers=4, hidden=32, grid_resolution=16, grid_channels=16, seed=0),
                 res=256, stepsize=1 / 128, kind="dvr"),
    "cfg2": dict(model=dict(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0),
                 res=1024, stepsize=1 / 256, kind="dvr"),
    "cfg3": dict(model=dict(layers=6, hidden=64, grid_resolution=64, grid_channels=16,
                            fourier_m=30, seed=0),
                 res=1024, stepsize=1 / 768, kind="dvr"),
    "cfg4": dict(model=dict(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0),
                 res=256, kind="decode"),
    "cfg5": dict(model=dict(layers=4, hidden=32, grid_resolution=32, grid_channels=16,
                            keyframe_times=[1, 11, 21], seed=0),
                 res=4096, stepsize=1 / 256, kind="dvr", t=6.5),
}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def available() -> bool:
    return (REF_DIR / "fvsrn" / "__init__.py").exists()


class Runner:
    """One configuration on the reference (``kind="reference"``) or the port."""

    def __init__(self, config: str, threads: int, prefer_ref: bool = True):
        self.cfg = CONFIGS[config]
        self.config = config
        self.threads = max(1, int(threads))
        self.kind = "reference" if (prefer_ref and available()) else "port"
        if self.kind == "reference":
            self._init_ref()
        else:
            self._init_port()

    # ---------------------------------------------------------------- reference
    def _init_ref(self):
        if str(REF_DIR) not in sys.path:
            sys.path.insert(0, str(REF_DIR))
        from fvsrn.model import ModelConfig, decode_volume, model_init
        from fvsrn.render import ModelSource, RenderSettings, camera_rays, render_rays
        from fvsrn.train import fibonacci_cameras
        from fvsrn.transfer import TF_PRESETS

        self.model = model_init(ModelConfig(**self.cfg["model"]))
        self._decode = decode_volume
        self._rays = camera_rays
        self._render_rays = render_rays
        lock = threading.Lock()

        class Counting(ModelSource):
            count = 0

            def sample(self, p, d):
                with lock:
                    Counting.count += len(p)
                return super().sample(p, d)

        self._src_cls = Counting
        self._tf = TF_PRESETS["grayscale"]
        self._fused = self.model.config.hidden <= 32
        if self.cfg["kind"] == "dvr":
            self.cams = fibonacci_cameras(8, self.cfg["res"], self.cfg["res"])
            self.settings = RenderSettings(stepsize=self.cfg["stepsize"], threads=self.threads)

    def _rows_ref(self, view: int, rows) -> int:
        from concurrent.futures import ThreadPoolExecutor

        cam = self.cams[view % 8]
        o, d = self._rays(cam)
        w = cam.width
        idx = (np.asarray(rows)[:, None] * w + np.arange(w)[None, :]).reshape(-1)
        src = self._src_cls(self.model, self._tf, t=self.cfg.get("t"), use_fused=self._fused)
        self._src_cls.count = 0
        # render.py:320-331 restricted to the sample rows
        if self.threads <= 1 or len(idx) < 4096:
            self._render_rays(src, o[idx], d[idx], self.settings)
        else:
            chunks = [c for c in np.array_split(idx, self.threads * 4) if len(c)]
            with ThreadPoolExecutor(max_workers=self.threads) as pool:
                futs = [pool.submit(self._render_rays, src, o[c], d[c], self.settings) for c in chunks]
                for f in futs:
                    f.result()
        return int(self._src_cls.count)

    # ---------------------------------------------------------------- port
    def _init_port(self):
        from oracle import fvsrn_oracle as O

        O.set_threads(self.threads)
        self.O = O
        self.model = O.model_init(O.OConfig(**self.cfg["model"]))
        if self.cfg["kind"] == "dvr":
            self.cams = O.fibonacci_cameras(8, self.cfg["res"], self.cfg["res"])

    def _rows_port(self, view: int, rows) -> int:
        cnt = [0]
        self.O.render_image(self.model, self.O.TF_PRESETS["grayscale"], self.cams[view % 8],
                            self.cfg["stepsize"], t=self.cfg.get("t"), counter=cnt, rows=rows,
                            threads=self.threads)
        return cnt[0]

    # ---------------------------------------------------------------- public
    def render_rows(self, view: int, rows):
        """(evals, seconds) for the given rows of view ``view``."""
        t0 = time.perf_counter()
        n = self._rows_ref(view, rows) if self.kind == "reference" else self._rows_port(view, rows)
        return n, time.perf_counter() - t0

    def decode(self, x_stride: int = 1):
        """(evals, seconds): decode_volume of the full lattice (x_stride 1), or the port's
        evaluation of every x_stride-th x slab of it."""
        res = self.cfg["res"]
        t0 = time.perf_counter()
        if self.kind == "reference" and x_stride == 1:
            self._decode(self.model, res)
            return res ** 3, time.perf_counter() - t0
        axis = np.linspace(0.0, 1.0, res)
        gx, gy, gz = np.meshgrid(axis[::x_stride], axis, axis, indexing="ij")
        pts = np.stack([gx, gy, gz], -1).reshape(-1, 3)
        if self.kind == "reference":
            from fvsrn.model import eval_density
        else:
            eval_density = self.O.eval_density
        for lo in range(0, len(pts), 1 << 16):      # decode_volume's chunking (model.py:392)
            eval_density(self.model, pts[lo:lo + (1 << 16)])
        return len(pts), time.perf_counter() - t0

    def render_step(self, step: int, stride: int):
        """One bench step of a DVR config: every stride-th row of view (step mod 8), offset by
        step // 8 (stride 1 = the whole frame).  One view per call keeps the batches the
        reference's thread pool sees close to a full frame's (render.py:320-331)."""
        res = self.cfg["res"]
        return self.render_rows(step % 8, np.arange((step // 8) % stride, res, stride))

    def warm(self):
        """JIT / first-call warm-up on a tiny sample (untimed)."""
        if self.cfg["kind"] == "dvr":
            self.render_rows(0, [self.cfg["res"] // 2])
        else:
            self.decode(x_stride=self.cfg["res"] // 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--row-stride", type=int, default=8)
    ap.add_argument("--full", action="store_true", help="the whole frame / lattice")
    ap.add_argument("--step", type=int, default=0, help="bench step index (render_step)")
    args = ap.parse_args()
    r = Runner(args.config, args.threads)
    r.warm()
    if r.cfg["kind"] == "dvr":
        stride = 1 if args.full else args.row_stride
        n, dt = r.render_step(args.step, stride)
        sample = (f"whole frame of view {args.step % 8}" if stride == 1 else
                  f"every {stride}th row of view {args.step % 8} ({r.cfg['res'] // stride} of "
                  f"{r.cfg['res']} rows)")
    else:
        stride = 1 if args.full else args.row_stride
        n, dt = r.decode(stride)
        sample = ("full lattice decode_volume" if stride == 1
                  else f"x slabs [::{stride}] of the lattice")
    print(json.dumps({"evals": n, "seconds": dt, "value": n / dt, "kind": r.kind,
                      "threads": r.threads, "sample": f"{args.config}: {sample}",
                      "cpu_model": cpu_model(), "cores": len(os.sched_getaffinity(0))}))


if __name__ == "__main__":
    main()
