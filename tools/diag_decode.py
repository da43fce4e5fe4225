"""decode_volume(256) host paths on the GPU box: mapped pinned vs copy."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2112_01579_b200 as P
from paper_2112_01579_b200 import device as D
m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0))
vb = P.pinned_empty((256, 256, 256))
for i in range(2): P.decode_volume(m, 256, out=vb)
D.kernel_timer(True)
ts = []
for i in range(6):
    t0 = time.perf_counter(); P.decode_volume(m, 256, out=vb); ts.append(1e3 * (time.perf_counter() - t0))
print("decode e2e ms", [round(x, 2) for x in ts], "kernel ms/launch", D.kernel_timer_read()[0] / 6)
