"""Where does the host-side time of render_image go? (run on the GPU box)"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2112_01579_b200 as P
from paper_2112_01579_b200 import device as D

for res, step in ((256, 1 / 128), (1024, 1 / 256), (4096, 1 / 256)):
    m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=32, grid_channels=16))
    src = P.ModelSource(m, P.TF_PRESETS["grayscale"])
    cam = P.fibonacci_cameras(8, res, res)[0]
    s = P.RenderSettings(stepsize=step)
    fb = P.pinned_empty((res, res, 4))
    for _ in range(3):
        P.render_image(src, cam, s, out=fb)
    n = 10
    t0 = time.perf_counter()
    for _ in range(n):
        P.render_image(src, cam, s, out=fb)
    t_api = (time.perf_counter() - t0) / n
    t0 = time.perf_counter()
    for _ in range(n):
        D.camera_desc(cam); D.settings_desc(s); D.tf_desc(src.tf)
    t_py = (time.perf_counter() - t0) / n
    np_out = np.empty((res, res, 4), np.float32)
    P.render_image(src, cam, s, out=np_out)
    t0 = time.perf_counter()
    for _ in range(n):
        P.render_image(src, cam, s, out=np_out)
    t_page = (time.perf_counter() - t0) / n
    import torch
    dev = torch.empty((res, res, 4), device="cuda")
    host = torch.from_numpy(fb)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        host.copy_(dev); torch.cuda.synchronize()
    t_d2h = (time.perf_counter() - t0) / n
    print(f"res {res}: api(pinned) {t_api*1e3:.3f} ms  api(pageable) {t_page*1e3:.3f} ms  "
          f"py descs {t_py*1e3:.3f} ms  torch D2H->pinned {t_d2h*1e3:.3f} ms  evals {src.last_eval_count}")
