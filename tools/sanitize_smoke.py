"""Small invocations of every kernel family, for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
(the small frame takes the eight-lanes-per-ray kernel; FVSRN_OCTO_FRAC=0 the four-lane one,
FVSRN_OCTO_FRAC=0 FVSRN_QUAD_FRAC=0 the two-lane one)"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2112_01579_b200 as P
from paper_2112_01579_b200 import device as D

cam = P.fibonacci_cameras(8, 40, 24)[2]
s = P.RenderSettings(stepsize=1 / 64)
for kw in (dict(layers=4, hidden=32, grid_resolution=8, seed=0),
           dict(layers=6, hidden=64, grid_resolution=8, fourier_m=30, seed=0),
           dict(layers=3, hidden=32, grid_resolution=6, grid_channels=8, keyframe_times=[1, 6, 11],
                time_mode="both", seed=3)):
    m = P.model_init(P.ModelConfig(**kw))
    t = 3.0 if m.is_temporal else None
    src = P.ModelSource(m, P.TF_PRESETS["warm"], t=t)
    for sampler in ("auto", "ldg"):    # texture units / exact-weight LDG.256 sampler
        D.set_grid_sampler(sampler)
        for k in ("auto", "warp", "tc"):   # auto on this small frame: the lane-group kernels
            D.set_dvr_kernel(k)
            P.render_image(src, cam, s)
            P.decode_volume(m, 12, t=t)    # tcgen05 decode (tc / auto) or mma.sync (warp)
        D.set_dvr_kernel("auto")
    D.set_grid_sampler("auto")
    p = np.random.default_rng(0).uniform(0, 1, (100, 3))
    P.eval_density(m, p, t=t)
vol = P.ScalarVolume(np.random.default_rng(1).uniform(0, 1, (9, 7, 5)).astype(np.float32))
P.render_image(P.VolumeSource(vol, P.TF_PRESETS["grayscale"]), cam, s)
m = P.model_init(P.ModelConfig(layers=3, hidden=32, grid_resolution=8, seed=0))
P.train_world(m, P.WorldTarget(vol), P.WorldTrainConfig(sample_count=2048, batch_size=512, epochs=1))
mc = P.model_init(P.ModelConfig(head="color", layers=3, hidden=32, grid_resolution=8, seed=11))
P.train_screen(mc, vol, P.TF_PRESETS["warm"],
               P.ScreenTrainConfig(views=2, resolution=12, stepsize=0.05, epochs=1, reference_stepsize_voxels=0.5))
mt = P.model_init(P.ModelConfig(layers=3, hidden=32, grid_resolution=6, keyframe_times=[1, 11], seed=0))
P.train_temporal(mt, lambda t: vol, P.TemporalTrainConfig(keyframe_times=[1, 11], train_times=[1, 6, 11],
                 world=P.WorldTrainConfig(sample_count=1024, batch_size=512, epochs=1)))
print("sanitize smoke done")
