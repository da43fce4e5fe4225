"""Debug the two-lanes-per-ray kernel on a tiny frame (run under timeout)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2112_01579_b200 as P
m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0))
src = P.ModelSource(m, P.TF_PRESETS["grayscale"])
for res in (8, 16, 40):
    cam = P.fibonacci_cameras(8, res, res)[2]
    st = P.RenderSettings(stepsize=1 / 128)
    print("rendering", res, flush=True)
    img = P.render_image(src, cam, st).data
    o, d = P.camera_rays(cam)
    px, _ = P.raymarch_forward(src, o, d, st)
    print(res, "equal", np.array_equal(px.reshape(res, res, 4), img), flush=True)
