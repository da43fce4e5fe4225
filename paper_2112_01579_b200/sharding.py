"""Screen-tile sharding of one DVR frame across GPUs (one process per GPU).

SURVEY 8(e): rays are independent, so a frame splits into 8x8-pixel tiles
assigned round-robin (tile t -> rank t mod world; the projected cube sits in the
frame centre, so contiguous slabs would be imbalanced).  The model, grid and TF
are replicated (each rank uploads its own copy).  Every rank renders its tiles
into a compact slot-ordered buffer with the fused kernel; one NCCL gather moves
the buffers to rank 0, where a permutation kernel writes the row-major frame.
Tiles are rendered by exactly the same per-ray code as the 1-GPU path, so the
gathered frame is bit-identical to a single-GPU render (tested).
"""

from __future__ import annotations

import math

import numpy as np

TILE = 8


def tile_grid(width: int, height: int):
    tx = math.ceil(width / TILE)
    return tx, tx * math.ceil(height / TILE)


def shard_pixel_index(width: int, height: int, rank: int, world: int) -> np.ndarray:
    """Row-major pixel index of each compact slot of ``rank`` (-1 = padding).

    Host mirror of slot_pixel() in fvsrn_kernels.cu; length max_local_tiles*64.
    """
    tx, n_tiles = tile_grid(width, height)
    max_local = math.ceil(n_tiles / world)
    s = np.arange(max_local * TILE * TILE)
    tile = rank + (s >> 6) * world
    e = s & 63
    px = (tile % tx) * TILE + (e & 7)
    py = (tile // tx) * TILE + (e >> 3)
    ok = (tile < n_tiles) & (px < width) & (py < height)
    return np.where(ok, py * width + px, -1)


def reassemble_host(gathered: np.ndarray, width: int, height: int) -> np.ndarray:
    """Host version of tiles_to_frame (used by CPU multi-process tests)."""
    world = gathered.shape[0]
    frame = np.zeros((height * width, 4), dtype=gathered.dtype)
    for r in range(world):
        idx = shard_pixel_index(width, height, r, world)
        ok = idx >= 0
        frame[idx[ok]] = gathered[r][ok]
    return frame.reshape(height, width, 4)


class TileShardRenderer:
    """Renders frames of one ModelSource across the ranks of a torch.distributed group.

    Each rank binds its own GPU (``torch.cuda.current_device()``); call
    ``render(camera, settings)`` on every rank: rank 0 returns the (H,W,4)
    device tensor, other ranks return None.
    """

    def __init__(self, source, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.source = source
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.dm = source.device_model
        self._bufs = {}
        self.last_eval_count = 0

    def _buffers(self, width, height):
        key = (width, height)
        if key not in self._bufs:
            t = self.torch
            _, per_rank = _shard_len(width, height, self.world)
            local = t.empty((per_rank, 4), dtype=t.float32, device="cuda")
            gathered = (t.empty((self.world, per_rank, 4), dtype=t.float32, device="cuda")
                        if self.rank == 0 else None)
            frame = (t.empty((height, width, 4), dtype=t.float32, device="cuda")
                     if self.rank == 0 else None)
            count = t.zeros(1, dtype=t.int64, device="cuda")
            self._bufs[key] = (local, gathered, frame, count)
        return self._bufs[key]

    def render(self, camera, settings, count: bool = False):
        from .device import tiles_to_frame_device

        t = self.torch
        local, gathered, frame, cnt = self._buffers(camera.width, camera.height)
        stream = t.cuda.current_stream().cuda_stream
        if count:
            cnt.zero_()
        self.dm.render_device(self.source.tf, camera, settings, self.source.t, local.data_ptr(),
                              cnt.data_ptr() if count else None, stream, rank=self.rank,
                              world=self.world, compact=True)
        if self.world > 1:
            if self.rank == 0:
                self.dist.gather(local, gather_list=list(gathered.unbind(0)), dst=0,
                                 group=self.group)
            else:
                self.dist.gather(local, gather_list=None, dst=0, group=self.group)
        elif gathered is not None:
            gathered[0].copy_(local)
        if self.rank == 0:
            tiles_to_frame_device(gathered.data_ptr(), camera.width, camera.height, self.world,
                                  frame.data_ptr(), stream)
        if count:
            if self.world > 1:
                self.dist.all_reduce(cnt, group=self.group)
            self.last_eval_count = int(cnt.item())
        return frame if self.rank == 0 else None


def _shard_len(width, height, world):
    _, n_tiles = tile_grid(width, height)
    return n_tiles, math.ceil(n_tiles / world) * TILE * TILE


class PeerUnavailable(RuntimeError):
    """Raised on every rank when any rank cannot map rank 0's framebuffer."""


class PeerFrameRenderer:
    """Screen-tile sharding with the frame assembled in peer memory.

    Rank 0 exports its (H,W,4) device framebuffers (CUDA IPC: handle + offset from the
    allocation base); every other rank opens them and its fused kernel stores each
    finished pixel of its round-robin tiles straight into rank 0's frame over NVLink
    P2P -- the "gather" happens inside the render kernel, tile by tile, overlapped with
    the ray marching; there is no separate collective and no reassembly kernel.  After
    each rank's stream completes, a process-group barrier publishes the frame.  Pixels
    are produced by the same per-ray code as the 1-GPU path, so the frame is
    bit-identical to a single-GPU render.

    Frames alternate between two exported buffers.  The frame ``render`` returns on rank
    0 stays valid until the second following ``render`` call: a peer rank can only start
    writing frame N+2 (the same buffer) after the barrier that ends frame N+1, which rank
    0 reaches after it has finished with frame N.
    """

    NBUF = 2

    def __init__(self, source, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.source = source
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.dm = source.device_model
        self._frames = {}
        self._opened = []
        self._seq = 0
        self.last_eval_count = 0

    def _export(self, frame):
        """rank 0: (handle bytes, offset); others: open it -> peer pointer.  Every rank
        reaches the same collectives and agrees on failure (PeerUnavailable everywhere)."""
        import ctypes as C

        from . import _lib as L

        t = self.torch
        ptr = frame.data_ptr() if frame is not None else None
        obj, err = [None], None
        if self.rank == 0:
            try:
                h = C.create_string_buffer(64)
                off = C.c_uint64()
                L.check(L.lib().fvsrn_ipc_export(C.c_void_p(ptr), h, C.byref(off)))
                obj = [(h.raw, int(off.value))]
            except Exception as e:          # noqa: BLE001 -- reported below
                err = e
        self.dist.broadcast_object_list(obj, src=0, group=self.group)
        if self.rank != 0 and obj[0] is not None:
            try:
                p = C.c_void_p()
                L.check(L.lib().fvsrn_ipc_open(obj[0][0], obj[0][1], t.cuda.current_device(),
                                               C.byref(p)))
                ptr = p.value
                self._opened.append(ptr)
            except Exception as e:          # noqa: BLE001
                err = e
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        ok = t.tensor([0 if (err is not None or obj[0] is None) else 1], device=dev)
        self.dist.all_reduce(ok, op=self.dist.ReduceOp.MIN, group=self.group)
        if not int(ok.item()):
            self.close()
            raise PeerUnavailable(f"peer framebuffer unavailable on some rank ({err})")
        return ptr

    def _frame(self, width, height, slot: int = 0):
        key = (width, height)
        if key not in self._frames:
            t = self.torch
            bufs = []
            for _ in range(self.NBUF):
                frame = (t.empty((height, width, 4), dtype=t.float32, device="cuda")
                         if self.rank == 0 else None)
                ptr = self._export(frame) if self.world > 1 else frame.data_ptr()
                bufs.append((frame, ptr))
            cnt = t.zeros(1, dtype=t.int64, device="cuda")
            self._frames[key] = (bufs, cnt)
        bufs, cnt = self._frames[key]
        frame, ptr = bufs[slot % self.NBUF]
        return frame, ptr, cnt

    def render_async(self, camera, settings, count: bool = False, slot: int | None = None):
        """Launch this rank's share on the current stream (no synchronisation) into buffer
        ``slot`` (default: the next one in the ping-pong)."""
        t = self.torch
        if slot is None:
            slot, self._seq = self._seq, self._seq + 1
        frame, ptr, cnt = self._frame(camera.width, camera.height, slot)
        if count:
            cnt.zero_()
        self.dm.render_device(self.source.tf, camera, settings, self.source.t, ptr,
                              cnt.data_ptr() if count else None, t.cuda.current_stream().cuda_stream,
                              rank=self.rank, world=self.world, compact=False)
        return frame, cnt

    def render(self, camera, settings, count: bool = False):
        frame, cnt = self.render_async(camera, settings, count)
        self.torch.cuda.current_stream().synchronize()      # this rank's stores have landed
        if self.world > 1:
            self.dist.barrier(group=self.group)              # ... and every other rank's
            if count:
                self.dist.all_reduce(cnt, group=self.group)
        if count:
            self.last_eval_count = int(cnt.item())
        return frame if self.rank == 0 else None

    def close(self):
        from . import _lib as L

        for ptr in self._opened:
            L.lib().fvsrn_ipc_close(__import__("ctypes").c_void_p(ptr))
        self._opened.clear()
        self._frames.clear()
