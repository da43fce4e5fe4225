"""Break down render_image wall time (host setup, kernels, copy) on the GPU box."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import paper_2112_01579_b200 as P
from paper_2112_01579_b200 import _lib as L
from paper_2112_01579_b200 import device as D

for cfgname, kw, res, ss in [("cfg2", dict(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0), 1024, 1 / 256)]:
    m = P.model_init(P.ModelConfig(**kw))
    src = P.ModelSource(m, P.TF_PRESETS["grayscale"], use_fused=True)
    cams = P.fibonacci_cameras(8, res, res)
    s = P.RenderSettings(stepsize=ss)
    fb = P.pinned_empty((res, res, 4))
    dm = src.device_model
    frame = torch.empty((res, res, 4), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    for i in range(3):
        P.render_image(src, cams[i], s, out=fb)
    def wall(fn, n=8):
        ts = []
        for i in range(n):
            t0 = time.perf_counter(); fn(i); ts.append(1e3 * (time.perf_counter() - t0))
        return sorted(ts)[n // 2]
    print("render_image(out=mapped pinned)  %.3f ms" % wall(lambda i: P.render_image(src, cams[i], s, out=fb)))
    print("dm.render (ctypes only)          %.3f ms" % wall(lambda i: dm.render(src.tf, cams[i], s, None, out=fb)))
    def dev(i):
        dm.render_device(src.tf, cams[i], s, None, frame.data_ptr(), None, st.cuda_stream); torch.cuda.synchronize()
    print("render_device + sync             %.3f ms" % wall(dev))
    def dev_copy(i):
        dm.render_device(src.tf, cams[i], s, None, frame.data_ptr(), None, st.cuda_stream)
        torch.from_numpy(fb).copy_(frame, non_blocking=True); torch.cuda.synchronize()
    print("render_device + D2H + sync       %.3f ms" % wall(dev_copy))
    D.kernel_timer(True)
    dev(0)
    print("kernel only                      %.3f ms" % D.kernel_timer_read()[0])
    D.kernel_timer(False)
    def desc_only(i):
        D.tf_desc(src.tf); D.camera_desc(cams[i]); D.settings_desc(s)
    print("python descriptors               %.3f ms" % wall(desc_only))
