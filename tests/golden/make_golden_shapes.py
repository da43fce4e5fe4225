"""Golden fixtures at the EXACT BASELINE.json shapes, made by running the REFERENCE.

The bench reports configs 2, 3 and 5 at 1024^2 / 4096^2.  The reference renders those
frames in minutes to hours on the CPU, so this script renders deterministic ROW SUBSETS
of each frame through the reference's own `raymarch_forward` (render.py:203-238) on the
rays `camera_rays` (render.py:72-94) produces for those rows.  Rays are independent in
the reference (per-ray early termination, render.py:219-232), so a row subset is
bit-identical to the same rows of a full `render_image` frame.

Fixtures written next to this file:
  golden_shapes.npz / golden_shapes.json
    cfg2_v{0..7}     config 2: 4x32, R32, 1024^2, stepsize 1/256, all 8 fibonacci views
    cfg3_v{0,5}      config 3: 6x64, R64, m=30, 1024^2, stepsize 1/768 (use_fused=False:
                     the fused plan raises CapacityError, render.py:168-180)
    cfg5_t{..}       config 5: R32, keyframes [1,11,21], 4096^2, stepsize 1/256,
                     t in {1, 6.5, 11, 16.25, 21} (model.py:219-233)
    trained_v{0..7}  a train_world checkpoint (train.py:165-206) of the config-2 shape
                     trained on synth_field("marschner_lobb", 64): all 8 views, 1024^2
    trained_density  eval_density (model.py:368-373) of the trained model at 65,536
                     uniform positions (the oracle is pinned to these; the GPU test then
                     compares at 2^20 positions against the pinned oracle)
    trained3_*       the same for the config-3 shape (6x64, R64; 10 epochs), one view;
                     its checkpoint stores the latent grid as u8 codes (grid.py:157-172)
  trained_cfg2.fvsrn / trained_cfg3.fvsrn  the trained checkpoints, written by the
                     reference (f32 weights, f32 grid)

Each render entry stores the rows, the (len(rows)*W, 4) f32 pixels and the reference's
evaluated-sample count (ModelSource.sample calls).

Run here (where /root/reference exists), read-only import, no source copied:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_shapes.py
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import fvsrn  # noqa: E402
from fvsrn.model import ModelConfig, checkpoint_load, checkpoint_save, eval_density, model_init  # noqa: E402
from fvsrn.render import ModelSource, RenderSettings, camera_rays, raymarch_forward  # noqa: E402
from fvsrn.train import WorldTarget, WorldTrainConfig, fibonacci_cameras, train_world  # noqa: E402
from fvsrn.transfer import TF_PRESETS  # noqa: E402
from fvsrn.volume import synth_field  # noqa: E402

CFG2 = dict(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0)
CFG3 = dict(layers=6, hidden=64, grid_resolution=64, grid_channels=16, fourier_m=30, seed=0)
CFG5 = dict(layers=4, hidden=32, grid_resolution=32, grid_channels=16,
            keyframe_times=[1, 11, 21], time_mode="none", seed=0)
TRAIN = dict(sample_count=64 ** 3, batch_size=16384, epochs=50, lr=0.01, seed=0)
TRAIN3 = dict(sample_count=64 ** 3, batch_size=16384, epochs=10, lr=0.01, seed=0)


class Counting(ModelSource):
    count = 0

    def sample(self, p, d):
        Counting.count += len(p)
        return super().sample(p, d)


def rows_for(h: int, n: int) -> np.ndarray:
    """n deterministic rows spread over the band the unit cube projects into."""
    return np.unique(np.linspace(0.22 * h, 0.78 * h, n).astype(np.int64))


def render_rows(model, tf, cam, settings, rows, t=None, fused=True):
    o, d = camera_rays(cam)
    w = cam.width
    idx = (rows[:, None] * w + np.arange(w)[None, :]).reshape(-1)
    Counting.count = 0
    px, _ = raymarch_forward(Counting(model, tf, t=t, use_fused=fused), o[idx], d[idx], settings)
    return px.astype(np.float32), int(Counting.count)


def cam_meta(cam):
    return {"eye": list(map(float, cam.eye)), "target": list(map(float, cam.target)),
            "up": list(map(float, cam.up)), "fov_y": float(cam.fov_y),
            "width": cam.width, "height": cam.height}


def main():
    meta = {"reference": "fvsrn " + fvsrn.__version__, "models": {"cfg2": CFG2, "cfg3": CFG3,
            "cfg5": CFG5}, "train": TRAIN, "train3": TRAIN3, "renders": {}}
    arrays = {}
    gray = TF_PRESETS["grayscale"]

    def add(tag, model_name, model, tf_name, cam, settings, rows, t=None, fused=True):
        t0 = time.time()
        px, cnt = render_rows(model, TF_PRESETS[tf_name], cam, settings, rows, t, fused)
        arrays[f"px_{tag}"] = px
        arrays[f"rows_{tag}"] = rows
        meta["renders"][tag] = {"model": model_name, "tf": tf_name, "t": t, "count": cnt,
                                "stepsize": settings.stepsize, "camera": cam_meta(cam),
                                "fused": fused}
        print(f"{tag}: rows={len(rows)} count={cnt} {time.time() - t0:.1f}s", flush=True)

    # ---- config 2: all 8 views at 1024^2
    m2 = model_init(ModelConfig(**CFG2))
    cams = fibonacci_cameras(8, 1024, 1024)
    s2 = RenderSettings(stepsize=1 / 256)
    for v, cam in enumerate(cams):
        add(f"cfg2_v{v}", "cfg2", m2, "grayscale", cam, s2, rows_for(1024, 16))

    # ---- config 5: temporal R32, 4096^2, five timesteps (views cycle with t)
    m5 = model_init(ModelConfig(**CFG5))
    cams5 = fibonacci_cameras(8, 4096, 4096)
    for i, t in enumerate((1.0, 6.5, 11.0, 16.25, 21.0)):
        add(f"cfg5_t{t}", "cfg5", m5, "grayscale", cams5[i], s2, rows_for(4096, 8), t=t)

    # ---- config 3: 6x64, R64, 1024^2, stepsize 1/768 through the naive path
    m3 = model_init(ModelConfig(**CFG3))
    s3 = RenderSettings(stepsize=1 / 768)
    for v in (0, 5):
        add(f"cfg3_v{v}", "cfg3", m3, "grayscale", cams[v], s3, rows_for(1024, 16), fused=False)

    # ---- trained config-2 model (train_world on a Marschner-Lobb field)
    mt = model_init(ModelConfig(**CFG2))
    vol = synth_field("marschner_lobb", 64)
    t0 = time.time()
    _, trace = train_world(mt, WorldTarget(vol), WorldTrainConfig(**TRAIN))
    print(f"trained {TRAIN['epochs']} epochs in {time.time() - t0:.1f}s: {trace}", flush=True)
    meta["train_trace"] = [float(x) for x in trace]
    checkpoint_save(mt, HERE / "trained_cfg2.fvsrn", "f32", "f32")
    back = checkpoint_load(HERE / "trained_cfg2.fvsrn")
    p = np.random.default_rng(2024).uniform(0.0, 1.0, size=(65536, 3))
    arrays["trained_p"] = p
    arrays["trained_density"] = eval_density(back, p)
    for v, cam in enumerate(cams):
        add(f"trained_v{v}", "trained", back, "grayscale", cam, s2, rows_for(1024, 16))
    add("trained_v3_warm", "trained", back, "warm", cams[3], s2, rows_for(1024, 16))

    # ---- trained config-3 shape (6x64, R64, m=30): naive path, stepsize 1/768
    m3t = model_init(ModelConfig(**CFG3))
    t0 = time.time()
    _, trace3 = train_world(m3t, WorldTarget(vol), WorldTrainConfig(**TRAIN3))
    print(f"trained cfg3 {TRAIN3['epochs']} epochs in {time.time() - t0:.1f}s: {trace3}", flush=True)
    meta["train3_trace"] = [float(x) for x in trace3]
    checkpoint_save(m3t, HERE / "trained_cfg3.fvsrn", "f32", "u8")   # 4 MiB instead of 16
    back3 = checkpoint_load(HERE / "trained_cfg3.fvsrn")
    arrays["trained3_density"] = eval_density(back3, p[:16384])
    add("trained3_v2", "trained3", back3, "grayscale", cams[2], s3, rows_for(1024, 8), fused=False)

    np.savez_compressed(HERE / "golden_shapes.npz", **arrays)
    with open(HERE / "golden_shapes.json", "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", HERE / "golden_shapes.npz", flush=True)


if __name__ == "__main__":
    main()
