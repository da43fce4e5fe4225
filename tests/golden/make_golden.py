"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

The outputs (*.npz, *.fvsrn, golden.json) are committed; nothing on the GPU
box reads /root/reference.  The reference is imported read-only; no source is
copied.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import fvsrn  # noqa: E402
from fvsrn.imaging import Camera, Image  # noqa: E402
from fvsrn.model import (  # noqa: E402
    ModelConfig, assemble_input, checkpoint_save, decode_volume, eval_color,
    eval_density, model_init)
from fvsrn.render import (  # noqa: E402
    ModelSource, RenderSettings, _march_geometry, camera_rays, raymarch_forward,
    render_image)
from fvsrn.train import fibonacci_cameras  # noqa: E402
from fvsrn.transfer import TF_PRESETS, tf_eval  # noqa: E402
from fvsrn.fused import fused_eval, plan_for_model  # noqa: E402
from fvsrn.render import VolumeSource  # noqa: E402
from fvsrn.volume import ScalarVolume, sample_volume, synth_field  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def model_hashes(m):
    return {
        "weights": [sha(w) for w in m.params.weights],
        "biases": [sha(b) for b in m.params.biases],
        "grids": [sha(g.values) for g in m.grids],
        "b_matrix": sha(m.spatial_encoder.b_matrix),
    }


class Counting(ModelSource):
    count = 0

    def sample(self, p, d):
        Counting.count += len(p)
        return super().sample(p, d)


def counted_render(model, tf, cam, settings, t=None, fused=True):
    Counting.count = 0
    src = Counting(model, tf, t=t, use_fused=fused)
    img = render_image(src, cam, settings)
    return img.data, Counting.count


CONFIGS = {
    # name -> ModelConfig kwargs (BASELINE.json configs + test shapes)
    "cfg1": dict(layers=4, hidden=32, grid_resolution=16, grid_channels=16, seed=0),
    "cfg2": dict(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0),
    "cfg3": dict(layers=6, hidden=64, grid_resolution=64, grid_channels=16, fourier_m=30, seed=0),
    "tiny": dict(layers=2, hidden=16, fourier_m=6, grid_resolution=4, grid_channels=4, seed=7),
    "temporal": dict(layers=4, hidden=32, grid_resolution=8, grid_channels=16,
                     keyframe_times=[1, 11, 21], seed=0),
    "temporal_both": dict(layers=3, hidden=32, grid_resolution=6, grid_channels=8,
                          keyframe_times=[1, 6, 11], time_mode="both", seed=3),
    "color_dirf": dict(head="color", layers=3, hidden=32, grid_resolution=8, grid_channels=8,
                       direction_mode="dirF", fourier_m=12, seed=5),
    "color_pos": dict(head="color", layers=3, hidden=32, grid_resolution=8, grid_channels=16,
                      seed=11),
    "random_fourier": dict(layers=3, hidden=48, fourier_mode="random", fourier_m=20,
                           fourier_sigma=2.0, grid_resolution=8, grid_channels=16, seed=4),
    "relu_nogrid": dict(layers=3, hidden=32, activation="relu", grid_resolution=0, seed=9),
    "snake_f12": dict(layers=3, hidden=32, activation="snake", grid_resolution=5,
                      grid_channels=12, seed=13),
}


def main():
    rng = np.random.default_rng(20211203)
    meta = {"reference": "fvsrn " + fvsrn.__version__, "models": {}, "renders": {}}
    arrays = {}

    models = {k: model_init(ModelConfig(**v)) for k, v in CONFIGS.items()}
    for k, m in models.items():
        meta["models"][k] = {"config": CONFIGS[k], "hashes": model_hashes(m),
                             "input_width": m.config.input_width}

    # --- rays + geometry (render.py:72-106,189-200)
    cams = {
        "fib0": fibonacci_cameras(8, 37, 23)[0],
        "fib5": fibonacci_cameras(8, 37, 23)[5],
        "center": Camera(eye=(0.5, 0.5, 3.5), target=(0.5, 0.5, 0.5), up=(0, 1, 0),
                         fov_y=np.pi / 5, width=33, height=33),
        "inside": Camera(eye=(0.3, 0.6, 0.4), target=(0.9, 0.1, 0.8), up=(0, 0, 1),
                         fov_y=1.2, width=20, height=16),
    }
    for name, cam in cams.items():
        o, d = camera_rays(cam)
        tmin, ds, n = _march_geometry(o, d, RenderSettings(stepsize=1 / 128))
        arrays[f"rays_{name}_o"] = o
        arrays[f"rays_{name}_d"] = d
        arrays[f"rays_{name}_tmin"] = tmin
        arrays[f"rays_{name}_ds"] = ds
        arrays[f"rays_{name}_n"] = n
        meta.setdefault("cameras", {})[name] = {
            "eye": list(map(float, cam.eye)), "target": list(map(float, cam.target)),
            "up": list(map(float, cam.up)), "fov_y": float(cam.fov_y),
            "width": cam.width, "height": cam.height}

    # --- per-sample evaluation (model.py:248-279, 368-382)
    p = rng.uniform(0.0, 1.0, size=(4096, 3))
    p[:8] = [[0, 0, 0], [1, 1, 1], [0, 1, 0], [1, 0, 1], [0.5, 0.5, 0.5],
             [-0.1, 0.5, 1.2], [1.0, 0.999999, 1e-9], [0.25, 0.75, 0.125]]
    dirs = rng.normal(size=(4096, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    arrays["eval_p"] = p
    arrays["eval_d"] = dirs
    for k, m in models.items():
        t = 6.5 if m.is_temporal else None
        x = assemble_input(m, p[:257], dirs[:257] if m.config.direction_mode != "pos" else None, t)
        arrays[f"assemble_{k}"] = x
        if m.config.head == "density":
            if m.is_temporal:
                for tt in (1.0, 6.5, 11.0, 16.25, 21.0, 0.0, 30.0):
                    arrays[f"density_{k}_t{tt}"] = eval_density(m, p, t=tt)
            else:
                arrays[f"density_{k}"] = eval_density(m, p)
        else:
            dd = dirs if m.config.direction_mode != "pos" else None
            arrays[f"color_{k}"] = eval_color(m, p, dd)
    # fused operator (fused.py:281-301)
    for k in ("cfg1", "color_pos", "random_fourier"):
        m = models[k]
        x = rng.uniform(-1, 1, size=(1000, m.config.input_width)).astype(np.float32)
        arrays[f"fused_x_{k}"] = x
        arrays[f"fused_y_{k}"] = fused_eval(plan_for_model(m), m, x)

    # --- transfer functions (transfer.py:57-65)
    dens = np.concatenate([np.linspace(-0.2, 1.2, 141), rng.uniform(0, 1, 200)]).astype(np.float32)
    arrays["tf_density"] = dens
    for name, tf in TF_PRESETS.items():
        rgb, sig = tf_eval(tf, dens)
        arrays[f"tf_{name}_rgb"] = rgb
        arrays[f"tf_{name}_sigma"] = sig

    # --- renders (render.py:314-332), counted evals
    def add_render(tag, model, tf_name, cam, settings, t=None, fused=True):
        tf = TF_PRESETS[tf_name] if tf_name else None
        img, cnt = counted_render(model, tf, cam, settings, t, fused)
        arrays[f"render_{tag}"] = img
        meta["renders"][tag] = {
            "count": int(cnt), "tf": tf_name, "t": t,
            "stepsize": settings.stepsize, "max_steps": settings.max_steps,
            "background": list(settings.background), "et": settings.early_term_alpha,
            "camera": {"eye": list(map(float, cam.eye)), "target": list(map(float, cam.target)),
                       "up": list(map(float, cam.up)), "fov_y": float(cam.fov_y),
                       "width": cam.width, "height": cam.height}}
        print("render", tag, cnt, flush=True)

    s128 = RenderSettings(stepsize=1.0 / 128)
    fib128 = fibonacci_cameras(8, 128, 128)
    add_render("cfg1_v0_gray", models["cfg1"], "grayscale", fib128[0], s128)
    add_render("cfg1_v3_gray", models["cfg1"], "grayscale", fib128[3], s128)
    fib64 = fibonacci_cameras(8, 64, 64)
    add_render("cfg1_v6_warm", models["cfg1"], "warm", fib64[6], s128)
    add_render("cfg1_v1_peaks_bg", models["cfg1"], "two_peaks", fib64[1],
               RenderSettings(stepsize=1.0 / 100, background=(0.2, 0.3, 0.4)))
    add_render("cfg2_v2_gray", models["cfg2"], "grayscale", fib64[2], RenderSettings(stepsize=1 / 256))
    add_render("tiny_center_gray", models["tiny"], "grayscale", cams["center"],
               RenderSettings(stepsize=1 / 64))
    add_render("temporal_t6.5", models["temporal"], "grayscale", fib64[4],
               RenderSettings(stepsize=1 / 128), t=6.5)
    add_render("temporal_both_t3", models["temporal_both"], "warm", fib64[0],
               RenderSettings(stepsize=1 / 96), t=3.0)
    add_render("color_dirf", models["color_dirf"], None, fib64[5], RenderSettings(stepsize=1 / 64))
    add_render("color_pos_et", models["color_pos"], None, fib64[7],
               RenderSettings(stepsize=1 / 128, early_term_alpha=0.5))
    add_render("inside_gray", models["cfg1"], "grayscale", cams["inside"],
               RenderSettings(stepsize=1 / 128))
    add_render("cfg3_v0_gray_48", models["cfg3"], "grayscale", fibonacci_cameras(8, 48, 48)[0],
               RenderSettings(stepsize=1 / 192), fused=False)  # CapacityError on fused
    # ragged frame (neither side a multiple of the 8x8 screen tile), rays capped by
    # max_steps (render.py:196), ET off, coloured background
    add_render("cfg2_ragged_cap", models["cfg2"], "warm", fibonacci_cameras(8, 100, 36)[3],
               RenderSettings(stepsize=1 / 200, max_steps=60, early_term_alpha=1.0,
                              background=(0.05, 0.1, 0.15)))

    # --- ground-truth DVR through VolumeSource (render.py:132-141, volume.py:213-255)
    vols = {
        "sphere32": synth_field("sphere", 32),
        "gauss48": synth_field("gaussians", 48, {"n_components": 8}, seed=42),
        "random975": ScalarVolume(values=np.random.default_rng(1234).uniform(0, 1, size=(9, 7, 5))
                                  .astype(np.float32)),
    }
    for k, v in vols.items():
        arrays[f"volume_{k}"] = v.values
    vol_renders = [("sphere32", "grayscale", fib64[0], 1 / 32, (0, 0, 0)),
                   ("gauss48", "warm", fib64[3], 1 / 48, (0.1, 0.2, 0.3)),
                   ("random975", "two_peaks", fib64[5], 1 / 40, (0, 0, 0))]
    for vname, tfname, cam, step, bg in vol_renders:
        Counting.count = 0
        st = RenderSettings(stepsize=step, background=bg)
        img = render_image(VolumeSource(vols[vname], TF_PRESETS[tfname]), cam, st)
        tag = f"vol_{vname}_{tfname}"
        arrays[f"render_{tag}"] = img.data
        meta["renders"][tag] = {
            "count": None, "tf": tfname, "t": None, "volume": vname,
            "stepsize": st.stepsize, "max_steps": st.max_steps,
            "background": list(st.background), "et": st.early_term_alpha,
            "camera": {"eye": list(map(float, cam.eye)), "target": list(map(float, cam.target)),
                       "up": list(map(float, cam.up)), "fov_y": float(cam.fov_y),
                       "width": cam.width, "height": cam.height}}

    # --- raymarch_forward on explicit rays, max_steps cap (render.py:203-238)
    o = np.column_stack([rng.uniform(0.2, 0.8, 64), rng.uniform(0.2, 0.8, 64), np.full(64, -0.5)])
    d = np.column_stack([rng.uniform(-0.2, 0.2, 64), rng.uniform(-0.2, 0.2, 64), np.ones(64)])
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    arrays["rays_explicit_o"] = o
    arrays["rays_explicit_d"] = d
    px, _ = raymarch_forward(ModelSource(models["cfg1"], TF_PRESETS["warm"], use_fused=True), o, d,
                             RenderSettings(stepsize=1 / 300, max_steps=200))
    arrays["rays_explicit_px"] = px

    # --- decode (model.py:385-398)
    arrays["decode_tiny_9"] = decode_volume(models["tiny"], 9).values
    arrays["decode_cfg1_17"] = decode_volume(models["cfg1"], 17).values
    arrays["decode_temporal_12_t16.25"] = decode_volume(models["temporal"], 12, t=16.25).values

    # --- checkpoints written by the reference (model.py:430-472)
    checkpoint_save(models["tiny"], HERE / "tiny_f32.fvsrn", "f32", "f32")
    checkpoint_save(models["tiny"], HERE / "tiny_f16_u8.fvsrn", "f16", "u8")
    checkpoint_save(models["temporal_both"], HERE / "temporal_both_f32.fvsrn", "f32", "f32")
    from fvsrn.model import checkpoint_load
    for name in ("tiny_f32", "tiny_f16_u8", "temporal_both_f32"):
        back = checkpoint_load(HERE / f"{name}.fvsrn")
        t = 3.0 if back.is_temporal else None
        arrays[f"ckpt_{name}_density"] = eval_density(back, p[:512], t=t)

    # --- u8-quantised grids of the default (fast-path) shapes: the GPU
    # samples the codes directly (RGBA8 textures, dequantised in the kernel)
    checkpoint_save(models["cfg1"], HERE / "cfg1_f16_u8.fvsrn", "f16", "u8")
    checkpoint_save(models["temporal"], HERE / "temporal_f16_u8.fvsrn", "f16", "u8")
    for name, t in (("cfg1_f16_u8", None), ("temporal_f16_u8", 6.5)):
        back = checkpoint_load(HERE / f"{name}.fvsrn")
        arrays[f"ckpt_{name}_density"] = eval_density(back, p[:4096], t=t)
        add_render(f"ckpt_{name}", back, "grayscale", fib128[2], s128, t=t)

    # --- world-space training (train.py:136-206): one-batch gradients of the L1 loss
    # through model_backward (flat, trainable_arrays order) and short loss traces
    from fvsrn.model import color_head_backward, density_head_backward, model_backward
    from fvsrn.train import WorldTarget, WorldTrainConfig, _l1_and_adjoint, _model_predict, train_world
    vol = synth_field("gaussians", 24, {"n_components": 6}, seed=42)
    arrays["train_volume"] = vol.values
    meta["train"] = {}
    for name, tfname in (("cfg1", None), ("color_pos", "warm"), ("relu_nogrid", None), ("tiny", None)):
        model = model_init(ModelConfig(**CONFIGS[name]))
        target = WorldTarget(vol, TF_PRESETS[tfname] if tfname else None)
        pb = np.random.default_rng(77).uniform(0.0, 1.0, size=(512, 3))
        ref = target.reference(pb)
        pred, raw, ctx = _model_predict(model, pb)
        loss, adj = _l1_and_adjoint(pred, ref)
        if model.config.head == "density":
            raw_bar = density_head_backward(raw, adj)
        else:
            raw_bar = color_head_backward(raw, adj)
        grads = model_backward(model, ctx, raw_bar)
        arrays[f"train_pos_{name}"] = pb
        arrays[f"train_ref_{name}"] = np.asarray(ref, dtype=np.float32)
        arrays[f"train_grads_{name}"] = np.concatenate([g.reshape(-1) for g in grads.arrays()])
        meta["train"][name] = {"tf": tfname, "loss": loss}
    for name in ("tiny", "cfg1"):
        model = model_init(ModelConfig(**CONFIGS[name]))
        cfg = WorldTrainConfig(sample_count=4096, batch_size=1024, epochs=4, lr=0.01, seed=0)
        _, trace = train_world(model, WorldTarget(vol), cfg)
        arrays[f"train_trace_{name}"] = np.asarray(trace)
        arrays[f"train_final_{name}"] = np.concatenate([a.reshape(-1) for a in model.trainable_arrays()])
        print("train", name, trace, flush=True)

    # --- screen-space training (train.py:227-262): raymarch_backward (render.py:241-306)
    # of a colour model against a VolumeSource reference view, and a short trace
    from fvsrn.render import raymarch_backward
    from fvsrn.train import ScreenTrainConfig, train_screen

    model = model_init(ModelConfig(**CONFIGS["color_pos"]))
    cam = fibonacci_cameras(8, 12, 12)[1]
    o, d = camera_rays(cam)
    st = RenderSettings(stepsize=0.05)
    ref_px, _ = raymarch_forward(VolumeSource(vol, TF_PRESETS["warm"]), o, d,
                                 RenderSettings.for_voxels(24, 0.5))
    px, states = raymarch_forward(ModelSource(model), o, d, st, want_states=True)
    loss, adj = _l1_and_adjoint(px, ref_px)
    grads = raymarch_backward(model, o, d, st, adj, terminal_states=states)
    arrays["screen_o"], arrays["screen_d"] = o, d
    arrays["screen_px"], arrays["screen_ref"], arrays["screen_adj"] = px, ref_px, adj
    arrays["screen_state_c"], arrays["screen_state_a"] = states.color, states.alpha
    arrays["screen_grads"] = np.concatenate([g.reshape(-1) for g in grads.arrays()])
    meta["screen"] = {"stepsize": 0.05, "loss": loss}
    model = model_init(ModelConfig(**CONFIGS["color_pos"]))
    _, trace = train_screen(model, vol, TF_PRESETS["warm"],
                            ScreenTrainConfig(views=2, resolution=12, stepsize=0.05, epochs=3,
                                              reference_stepsize_voxels=0.5))
    arrays["screen_trace"] = np.asarray(trace)
    print("screen", trace, flush=True)

    # --- temporal training (train.py:265-314): one-batch gradients with per-sample
    # timesteps (keyframe hits and in-between) and a short train_temporal trace
    from fvsrn.train import TemporalTrainConfig, train_temporal

    for name in ("temporal", "temporal_both"):
        model = model_init(ModelConfig(**CONFIGS[name]))
        rng = np.random.default_rng(91)
        pb = rng.uniform(0.0, 1.0, size=(384, 3))
        kt = list(CONFIGS[name]["keyframe_times"])
        tb = np.concatenate([rng.uniform(kt[0], kt[-1], size=256), rng.choice(kt, size=128)])
        ref = sample_volume(vol, pb)
        pred, raw, ctx = _model_predict(model, pb, tb)
        loss, adj = _l1_and_adjoint(pred, ref)
        grads = model_backward(model, ctx, density_head_backward(raw, adj))
        arrays[f"ttrain_pos_{name}"], arrays[f"ttrain_t_{name}"] = pb, tb
        arrays[f"ttrain_ref_{name}"] = np.asarray(ref, dtype=np.float32)
        arrays[f"ttrain_grads_{name}"] = np.concatenate([g.reshape(-1) for g in grads.arrays()])
        meta["train"][f"t_{name}"] = {"loss": loss}
    model = model_init(ModelConfig(**CONFIGS["temporal"]))
    tcfg = TemporalTrainConfig(keyframe_times=[1, 11, 21], train_times=[1, 6, 11, 16, 21],
                               world=WorldTrainConfig(sample_count=4096, batch_size=1024, epochs=3,
                                                      lr=0.01, seed=0))
    provider = lambda t: synth_field("gaussians", 20, {"n_components": 5}, t=t / 21.0, seed=42)  # noqa: E731
    _, trace = train_temporal(model, provider, tcfg)
    arrays["ttrain_trace"] = np.asarray(trace)
    for tt in tcfg.train_times:
        arrays[f"ttrain_vol_{tt}"] = provider(tt).values
    print("temporal", trace, flush=True)

    # --- evaluation metrics (imaging.py:156-177, train.py:317-341): SSIM of seeded image
    # pairs (rgb, gray, identical) and a 2-view evaluate_views of cfg1 vs the train volume
    from fvsrn.imaging import metric_ssim
    from fvsrn.train import evaluate_views, metrics_csv

    rng = np.random.default_rng(123)
    a = rng.uniform(0, 1, size=(24, 20, 4)).astype(np.float32)
    b = np.clip(a + rng.normal(0, 0.1, size=a.shape), 0, 1).astype(np.float32)
    g1, g2 = rng.uniform(0, 1, size=(16, 33)), rng.uniform(0, 1, size=(16, 33))
    arrays["ssim_a"], arrays["ssim_b"], arrays["ssim_g1"], arrays["ssim_g2"] = a, b, g1, g2
    meta["ssim"] = {"rgb": metric_ssim(Image(a), Image(b)), "gray": metric_ssim(g1, g2),
                    "same": metric_ssim(Image(a), Image(a))}
    model = model_init(ModelConfig(**CONFIGS["cfg1"]))
    rows = evaluate_views(model, vol, TF_PRESETS["grayscale"], n_views=2, resolution=32)
    meta["evaluate_views"] = {"model": "cfg1", "tf": "grayscale", "n_views": 2, "resolution": 32,
                              "rows": rows, "csv": metrics_csv(rows)}
    print("evaluate_views", rows, flush=True)

    # --- grid_sample_backward (grid.py:123-137) on cfg1's latent grid: positions incl.
    # the faces / corners / outside the cube (clamped), random adjoints
    from fvsrn.grid import grid_sample_backward

    g1 = models["cfg1"].grid
    rng = np.random.default_rng(55)
    gp = rng.uniform(-0.1, 1.1, size=(300, 3))
    gp[:4] = [[0, 0, 0], [1, 1, 1], [1, 0, 0.5], [0.999999, 1e-9, 0.25]]
    gz = rng.normal(size=(300, g1.channels)).astype(np.float32)
    gg = np.zeros_like(g1.values)
    grid_sample_backward(g1, gp, gz, gg)
    arrays["gsb_pos"], arrays["gsb_zbar"], arrays["gsb_grad"] = gp, gz, gg

    # --- mlp_forward / mlp_backward (nn.py:179-193, 234-256) of plain MLPs
    from fvsrn.nn import init_params, mlp_backward, mlp_forward

    for tag, (lc, hid, din, dout, act) in {"snake4": (3, 16, 10, 4, "snake_alt"),
                                          "relu1": (4, 24, 7, 1, "relu"),
                                          "snake2": (2, 8, 5, 2, "snake"), "softplus3": (3, 12, 6, 3, "softplus")}.items():
        prm = init_params(lc, hid, din, dout, seed=3, activation=act)
        rng = np.random.default_rng(66)
        for b in prm.biases:
            b[...] = rng.normal(scale=0.1, size=b.shape).astype(np.float32)
        xm = rng.normal(size=(64, din)).astype(np.float32)
        ym, cm = mlp_forward(prm, xm)
        yb = rng.normal(size=ym.shape).astype(np.float32)
        xb, gm = mlp_backward(prm, cm, yb)
        arrays[f"mlp_{tag}_x"], arrays[f"mlp_{tag}_y"], arrays[f"mlp_{tag}_ybar"] = xm, ym, yb
        arrays[f"mlp_{tag}_xbar"] = xb
        arrays[f"mlp_{tag}_grads"] = np.concatenate([g.reshape(-1) for g in gm.arrays()])
        arrays[f"mlp_{tag}_biases"] = np.concatenate([b.reshape(-1) for b in prm.biases])
        arrays[f"mlp_{tag}_pre0"] = cm.preacts[0]
        meta.setdefault("mlp", {})[tag] = [lc, hid, din, dout, act]

    # --- fourier_encode (nn.py:96-105), f64 and f32 inputs
    from fvsrn.nn import fourier_encode, fourier_make

    fv = np.random.default_rng(12).uniform(-1, 2, size=(33, 3))
    arrays["fenc_v"] = fv
    for mode, mm in (("nerf", 12), ("random", 7)):
        enc = fourier_make(mode, mm, 3, sigma=2.0, seed=5)
        arrays[f"fenc_{mode}_f64"] = fourier_encode(enc, fv)
        arrays[f"fenc_{mode}_f32"] = fourier_encode(enc, fv.astype(np.float32))

    np.savez_compressed(HERE / "golden.npz", **arrays)
    with open(HERE / "golden.json", "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", HERE / "golden.npz", os.path.getsize(HERE / "golden.npz"), "bytes")


if __name__ == "__main__":
    main()
