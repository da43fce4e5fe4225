"""World-space training throughput on the GPU: config-2 model (4x32, 32^3x16 grid),
the reference's default WorldTrainConfig sizes (64^3 samples, batch 16384), a 64^3
gaussians volume.  Prints samples/s and ms per epoch (after one warm-up epoch)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_2112_01579_b200 as P
from paper_2112_01579_b200.train import WorldTrainer, sample_world_dataset

x, y, z = np.meshgrid(*(np.linspace(0, 1, 64),) * 3, indexing="ij")
v = np.zeros_like(x)
rng = np.random.default_rng(42)
for _ in range(8):
    c = rng.uniform(0.2, 0.8, 3)
    v += rng.uniform(0.3, 1.0) * np.exp(-((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2) / (2 * 0.08 ** 2))
vol = P.ScalarVolume(np.clip(v, 0, 1).astype(np.float32))
m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0))
target = P.WorldTarget(vol)
n, bs = 64 ** 3, 16384
pos, val = sample_world_dataset(target, n, "uniform", 0)
tr = WorldTrainer(m)
pos_d = torch.as_tensor(pos, device=tr.dev)
val_d = torch.as_tensor(val, dtype=torch.float32, device=tr.dev).reshape(n, -1)
gen = np.random.default_rng(0)


def epoch():
    perm = torch.as_tensor(gen.permutation(n), device=tr.dev)
    tot = 0.0
    for lo in range(0, n, bs):
        idx = perm[lo:lo + bs]
        tot += tr.gradients(pos_d[idx], val_d[idx]) * len(idx)
        tr.adam(0.01)
    return tot / n


epoch()
torch.cuda.synchronize()
ts = []
for e in range(5):
    t0 = time.perf_counter()
    loss = epoch()
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    print(f"epoch {e} loss {loss:.5f} {1e3 * ts[-1]:.1f} ms")
print(f"train_world epoch (64^3 samples, batch 16384): median {1e3 * sorted(ts)[2]:.1f} ms "
      f"-> {n / sorted(ts)[2] / 1e6:.1f} M samples/s")

# ---- screen space: colour model (4x32, 32^3x16 grid), 256^2 views, stepsize 0.02
from paper_2112_01579_b200.train import ScreenTrainer  # noqa: E402

mc = P.model_init(P.ModelConfig(head="color", layers=4, hidden=32, grid_resolution=32,
                                grid_channels=16, seed=0))
st = ScreenTrainer(mc)
settings = P.RenderSettings(stepsize=0.02)
cams = P.fibonacci_cameras(8, 256, 256)
vsrc = P.VolumeSource(vol, P.TF_PRESETS["warm"])
refs = []
for cam in cams:
    o, d = P.camera_rays(cam)
    pix, _ = P.raymarch_forward(vsrc, o, d, P.RenderSettings.for_voxels(64, 0.1))
    refs.append((o, d, torch.as_tensor(pix, device=st.dev)))


def screen_epoch():
    tot = 0.0
    for o, d, ref in refs:
        pix, state = st.forward(o, d, settings)
        diff = pix - ref
        tot += float(diff.abs().mean())
        st.backward(state, settings, torch.sign(diff) / diff.numel())
        st.adam(0.01)
    return tot / len(refs)


screen_epoch()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    loss = screen_epoch()
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 3
print(f"train_screen epoch (8 views 256^2, stepsize 0.02): {1e3 * dt:.1f} ms ({1e3 * dt / 8:.2f} ms/view), loss {loss:.5f}")
