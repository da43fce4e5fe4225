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
    # a live allocation first, so rank 0's frames sit at a non-zero offset inside the
    # caching allocator's segment (IPC maps the segment base; the offset must travel)
    pad = torch.empty(40000, dtype=torch.float32, device="cuda")
    r = PeerFrameRenderer(src)
    cams = P.fibonacci_cameras(8, 203, 157)
    got = []
    for v in (3, 4, 5):     # three frames through the two ping-pong buffers
        out = r.render(cams[v], P.RenderSettings(stepsize=1 / 128), count=True)
        if rank == 0:
            got.append((out.cpu().numpy(), r.last_eval_count))
    if rank == 0:
        q.put(got)
    del pad
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
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=16, seed=0))
    src = P.ModelSource(m, P.TF_PRESETS["warm"])
    cams = P.fibonacci_cameras(8, 203, 157)
    for (frame, count), v in zip(got, (3, 4, 5)):
        img = P.render_image(src, cams[v], P.RenderSettings(stepsize=1 / 128))
        bad = np.argwhere(np.abs(frame - img.data).max(-1) > 0)
        assert len(bad) == 0, (v, len(bad), bad[:8].tolist(), float(np.abs(frame - img.data).max()),
                               src.device_model.info())
        assert count == src.last_eval_count


def test_ipc_export_reports_offset_from_allocation_base():
    import ctypes as C

    import torch

    from paper_2112_01579_b200 import _lib as L

    a = torch.empty(4096, dtype=torch.float32, device="cuda")
    b = torch.empty(4096, dtype=torch.float32, device="cuda")
    offs = []
    for t in (a, b):
        h, off = C.create_string_buffer(64), C.c_uint64()
        L.check(L.lib().fvsrn_ipc_export(C.c_void_p(t.data_ptr()), h, C.byref(off)))
        offs.append(off.value)
    # both live in one caching-allocator segment: offsets differ by their address gap
    assert offs[1] - offs[0] == b.data_ptr() - a.data_ptr()
    assert offs[1] > 0


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
        L.lib().fvsrn_ipc_open = lambda *a: 3   # noqa: E731
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
