"""/render latency of the GPU service at 512^2 and 1024^2 (config-2 model), in-process
TestClient: X-Render-Millis (render + device quantisation + transfer) and the whole
request (incl. PNG encode)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
from fastapi.testclient import TestClient

import paper_2112_01579_b200 as P
from paper_2112_01579_b200.service import SessionState, create_app

m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0))
c = TestClient(create_app(SessionState(model=m, default_tf=P.TF_PRESETS["grayscale"],
                                       native_resolution=256)))
for res in (512, 1024):
    body = {"camera": {"eye": [0.5, 1.2, 2.4], "target": [0.5, 0.5, 0.5], "up": [0, 1, 0],
                       "fov_y_deg": 45.0}, "width": res, "height": res, "stepsize_voxels": 1.0}
    for _ in range(3):
        c.post("/render", json=body)
    rm, tot, size = [], [], 0
    for _ in range(10):
        t0 = time.perf_counter()
        r = c.post("/render", json=body)
        tot.append(1e3 * (time.perf_counter() - t0))
        rm.append(float(r.headers["X-Render-Millis"]))
        size = len(r.content)
    rm.sort(); tot.sort()
    print(f"{res}^2: X-Render-Millis median {rm[5]:.2f} ms, request median {tot[5]:.2f} ms, png {size} B")
