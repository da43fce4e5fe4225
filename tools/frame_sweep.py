"""Device ms/frame of the config-2 model across frame sizes (CUDA events around
render_device, L2 flushed between frames), for tuning the small-frame paths:
    FVSRN_PAIR_FRAC=0 python tools/frame_sweep.py ; python tools/frame_sweep.py
    FVSRN_QUAD_FRAC=5 python tools/frame_sweep.py   (four lanes per ray)
    python tools/frame_sweep.py 128 256 384        (sizes)"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2112_01579_b200 as P

m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0))
src = P.ModelSource(m, P.TF_PRESETS["grayscale"])
st = P.RenderSettings(stepsize=1 / 256)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for res in ([int(a) for a in sys.argv[1:]] or (128, 192, 256, 320, 384, 448, 512, 640, 768)):
    cams = P.fibonacci_cameras(8, res, res)
    frame = torch.empty((res, res, 4), dtype=torch.float32, device="cuda")
    for i in range(3):
        src.device_model.render_device(src.tf, cams[i], st, None, frame.data_ptr(), None, s.cuda_stream)
    ts = []
    for i in range(16):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        src.device_model.render_device(src.tf, cams[i % 8], st, None, frame.data_ptr(), None, s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{res}x{res} slots {res * res:7d}: {ts[len(ts) // 2]:.3f} ms", flush=True)
