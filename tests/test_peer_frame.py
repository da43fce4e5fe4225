"""Peer-memory framebuffer assembly (sharding.PeerFrameRenderer): two processes share
one GPU here (CUDA IPC works across processes on one device just as across NVLink
peers); rank 1's kernel writes its tiles straight into rank 0's frame.  The result must
be bit-identical to a single-process render and the evaluated-sample counts must add up."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2112_01579_b200 as P
    from paper_2112_01579_b200.sharding import PeerFrameRenderer

    m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=16, seed=0))
    src = P.ModelSource(m, P.TF_PRESETS["warm"])
    r = PeerFrameRenderer(src)
    cam = P.fibonacci_cameras(8, 203, 157)[3]
    out = r.render(cam, P.RenderSettings(stepsize=1 / 128), count=True)
    if rank == 0:
        q.put((out.cpu().numpy(), r.last_eval_count))
    dist.barrier()
    r.close()
    dist.barrier()
    dist.destroy_process_group()


def test_peer_frame_two_processes_bit_identical():
    import paper_2112_01579_b200 as P

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    frame, count = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=16, seed=0))
    src = P.ModelSource(m, P.TF_PRESETS["warm"])
    img = P.render_image(src, P.fibonacci_cameras(8, 203, 157)[3], P.RenderSettings(stepsize=1 / 128))
    assert np.array_equal(frame, img.data)
    assert count == src.last_eval_count


def _fallback_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2112_01579_b200 as P
    from paper_2112_01579_b200 import _lib as L
    from paper_2112_01579_b200.sharding import PeerFrameRenderer, PeerUnavailable

    if rank == 1:   # this rank cannot map rank 0's framebuffer
        L.lib().fvsrn_ipc_open = lambda *a: 3
    m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=16, seed=0))
    src = P.ModelSource(m, P.TF_PRESETS["warm"])
    raised = False
    try:
        PeerFrameRenderer(src)._frame(64, 48)
    except PeerUnavailable:
        raised = True
    q.put((rank, raised))
    dist.barrier()
    dist.destroy_process_group()


def test_peer_frame_failure_is_agreed_by_all_ranks():
    # one rank failing to open the IPC handle must not leave the other hanging in a
    # later collective: every rank raises PeerUnavailable (bench.py then falls back to
    # the NCCL gather path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fallback_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}
