"""Screen-tile sharding across ranks: tile assignment + gather + reassembly.

The GPU kernel's slot->pixel mapping is mirrored by ``shard_pixel_index``; here
two gloo ranks on CPU render their shares with the CPU oracle (test-only
renderer), gather to rank 0 and reassemble; the frame must equal a 1-rank
render.  The CUDA path of the same plumbing is tested in test_gpu_parity.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2112_01579_b200.sharding import reassemble_host, shard_pixel_index


@pytest.mark.parametrize("w,h,world", [(64, 64, 2), (123, 77, 3), (8, 8, 8), (1, 1, 4), (1024, 1024, 8)])
def test_every_pixel_exactly_once(w, h, world):
    seen = np.concatenate([shard_pixel_index(w, h, r, world) for r in range(world)])
    seen = seen[seen >= 0]
    assert len(seen) == w * h
    assert np.array_equal(np.sort(seen), np.arange(w * h))


def test_round_robin_balance():
    counts = [(shard_pixel_index(1024, 1024, r, 8) >= 0).sum() for r in range(8)]
    assert max(counts) - min(counts) <= 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import fvsrn_oracle as O

    m = O.model_init(O.OConfig(layers=2, hidden=16, fourier_m=6, grid_resolution=4,
                               grid_channels=4, seed=7))
    cam = O.fibonacci_cameras(8, 37, 29)[3]
    o, d = O.camera_rays(cam)
    idx = shard_pixel_index(cam.width, cam.height, rank, world)
    px = np.zeros((len(idx), 4), np.float32)
    ok = idx >= 0
    px[ok] = O.raymarch_forward(m, O.TF_PRESETS["warm"], o[idx[ok]], d[idx[ok]], 1 / 64)
    t = torch.from_numpy(px)
    gl = [torch.zeros_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, gather_list=gl, dst=0)
    if rank == 0:
        frame = reassemble_host(torch.stack(gl).numpy(), cam.width, cam.height)
        full = O.raymarch_forward(m, O.TF_PRESETS["warm"], o, d, 1 / 64).reshape(frame.shape)
        q.put(float(np.abs(frame - full).max()))
    dist.destroy_process_group()


def test_gloo_two_rank_gather_reassembles_frame():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert err <= 1e-6
