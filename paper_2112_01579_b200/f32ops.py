"""Reference-semantics (f32) evaluation of the model's pieces on the GPU.

``fvsrn_f32_eval`` evaluates, for a batch of samples, the assembled network input
(assemble_input, model.py:248-279), the latent vectors (grid_sample / keyframe_sample,
grid.py:115-121, 222-230), or the MLP (mlp_eval, nn.py:195-204) with the reference's
f32 arithmetic (f64 Fourier phases).  These are the standalone API counterparts of
pieces the render kernels evaluate fused, on chip, in fp16.  Device plumbing via torch.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

_ACT = {"relu": 0, "sigmoid": 1, "softplus": 2, "snake": 3, "snake_alt": 4}
_TIME = {"none": 0, "direct": 1, "fourier": 2, "both": 3}


class NetDesc:
    """fvsrn_train_desc + the flat f32 parameter buffer ([W..] [b..] [grids..]) on a device."""

    def __init__(self, weights, biases, activation, head, d_in, b_matrix=None, grids=(),
                 keyframe_times=None, time_mode="none", time_b=None, time_span=(0.0, 0.0),
                 raw_width=3, fourier_in=3, device=None):
        import torch

        self.torch = torch
        self.dev = torch.device("cuda", L.current_device() if device is None else device)
        arrays = [*weights, *biases, *(np.asarray(g) for g in grids)]
        flat = np.concatenate([np.ascontiguousarray(a, dtype=np.float32).reshape(-1) for a in arrays])
        self.params = torch.from_numpy(flat).to(self.dev)
        m = 0 if b_matrix is None else int(b_matrix.shape[0])
        self.bmat = (torch.from_numpy(np.ascontiguousarray(b_matrix, dtype=np.float32)).to(self.dev)
                     if m else None)
        R = int(np.asarray(grids[0]).shape[0]) if grids else 0
        F = int(np.asarray(grids[0]).shape[3]) if grids else 0
        hidden = int(weights[0].shape[0]) if len(weights) > 1 else 1
        self.desc = L.TrainDesc(len(weights), hidden, d_in, int(weights[-1].shape[0]), _ACT[activation],
                                0 if head == "density" else 1, m,
                                self.bmat.data_ptr() if m else None, R, F)
        self.desc.raw_width, self.desc.fourier_in = raw_width, fourier_in
        if keyframe_times is not None:
            self._kf = np.ascontiguousarray(keyframe_times, dtype=np.float64)
            self.desc.n_keyframes = len(self._kf)
            self.desc.keyframe_times = L.dptr(self._kf)
        mode = _TIME[time_mode]
        self._tb = (np.ascontiguousarray(time_b, dtype=np.float32).reshape(-1)
                    if time_b is not None else np.zeros(1, np.float32))
        self.desc.time_mode = mode
        self.desc.time_fourier_count = int(self._tb.size) if mode & 2 else 0
        self.desc.time_b = L.fptr(self._tb)
        self.desc.time_t0, self.desc.time_t1 = float(time_span[0]), float(time_span[1])
        self.d_in, self.d_out, self.F = d_in, int(weights[-1].shape[0]), F

    @classmethod
    def for_model(cls, model):
        cfg = model.config
        span = (0.0, 0.0)
        if model.is_temporal:
            span = cfg.time_range if cfg.time_range is not None else model.keyframes.span
        enc = model.spatial_encoder
        return cls(model.params.weights, model.params.biases, cfg.activation, cfg.head, cfg.input_width,
                   enc.b_matrix if enc.m > 0 else None, [g.values for g in model.grids],
                   list(model.keyframes.times) if model.is_temporal else None, cfg.time_mode,
                   model.time_encoder.b_matrix if cfg.time_mode in ("fourier", "both") else None, span,
                   raw_width=6 if cfg.direction_mode in ("dirP", "dirF") else 3,
                   fourier_in=6 if cfg.direction_mode == "dirF" else 3)

    def run(self, stage: int, n: int, out_w: int, p=None, d=None, t=None, x=None) -> np.ndarray:
        torch = self.torch
        dev = self.dev

        def dt(a, dtype):
            return None if a is None else torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=dev)

        pd, dd, td, xd = dt(p, torch.float64), dt(d, torch.float64), dt(t, torch.float64), dt(x, torch.float32)
        out = torch.empty((max(n, 1), out_w), dtype=torch.float32, device=dev)
        ptr = lambda a: C.c_void_p(a.data_ptr() if a is not None else None)  # noqa: E731
        stream = torch.cuda.current_stream(dev).cuda_stream
        L.check(L.lib().fvsrn_f32_eval(C.byref(self.desc), ptr(self.params), ptr(pd), ptr(dd), ptr(td),
                                       ptr(xd), n, stage, ptr(out), C.c_void_p(stream)))
        return out[:n].cpu().numpy()
