"""Where the e2e-vs-device gap of render_image goes: python-level wall time per call,
the C entry's host phases (FVSRN_DEBUG_TIMING) and the device time of the same frame."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_2112_01579_b200 as P
from paper_2112_01579_b200 import device as D

for kw, res, ss in [(dict(layers=4, hidden=32, grid_resolution=16, seed=0), 256, 1/128),
                    (dict(layers=4, hidden=32, grid_resolution=32, seed=0), 1024, 1/256)]:
    m = P.model_init(P.ModelConfig(**kw)); src = P.ModelSource(m, P.TF_PRESETS["grayscale"])
    cams = P.fibonacci_cameras(8, res, res); fb = P.pinned_empty((res, res, 4)); s = P.RenderSettings(stepsize=ss)
    for i in range(10): P.render_image(src, cams[0], s, out=fb)
    wall = []
    for i in range(20):
        t0 = time.perf_counter(); P.render_image(src, cams[0], s, out=fb); wall.append(time.perf_counter() - t0)
    dm = D.device_model(m)
    import cProfile, pstats
    pr = cProfile.Profile(); pr.enable()
    for i in range(20): P.render_image(src, cams[0], s, out=fb)
    pr.disable()
    print(f"res {res}: python wall median {np.median(wall)*1e3:.3f} ms min {np.min(wall)*1e3:.3f}")
    st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(12)
