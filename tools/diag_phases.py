import os, sys
sys.path.insert(0, os.getcwd())
import paper_2112_01579_b200 as P
from paper_2112_01579_b200 import device as D
for kw, res, ss in [(dict(layers=4, hidden=32, grid_resolution=16, seed=0), 256, 1/128), (dict(layers=4, hidden=32, grid_resolution=32, seed=0), 1024, 1/256)]:
    m = P.model_init(P.ModelConfig(**kw)); src = P.ModelSource(m, P.TF_PRESETS["grayscale"])
    cams = P.fibonacci_cameras(8, res, res); fb = P.pinned_empty((res, res, 4)); s = P.RenderSettings(stepsize=ss)
    for i in range(6): P.render_image(src, cams[i % 8], s, out=fb)
