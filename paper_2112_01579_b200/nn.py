"""Network parameter containers and seeded initialisation (host side).

Mirrors the parameter API of the reference ``fvsrn.nn`` (nn.py:15-168) so a
reference user can build models the same way; evaluation itself runs on the
GPU (``paper_2112_01579_b200.model`` / ``render``).  Initialisation draws from
``numpy.random.default_rng(seed)`` in the reference's order, so a given seed
yields bit-identical weights (pinned by tests/test_host_api.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ACTIVATION_KINDS = ("relu", "sigmoid", "softplus", "snake", "snake_alt")


def nerf_rows(m: int, d_in: int) -> np.ndarray:
    """(m, d_in) f32 frequency matrix: row i has 2*pi*2**(i // d_in) on axis i % d_in."""
    out = np.zeros((m, d_in), dtype=np.float32)
    i = np.arange(m)
    out[i, i % d_in] = (2.0 * np.pi) * np.exp2((i // d_in).astype(np.float64))
    return out


@dataclass(frozen=True)
class FourierEncoder:
    """v -> [v | sin(Bv) | cos(Bv)] with a frozen B (nn.py:60-76)."""

    mode: str
    b_matrix: np.ndarray
    d_in: int
    sigma: float = 1.0
    seed: int = 0

    @property
    def m(self) -> int:
        return int(self.b_matrix.shape[0])

    @property
    def out_width(self) -> int:
        return self.d_in + 2 * self.m


def fourier_make(mode: str, m: int, d_in: int, sigma: float = 1.0, seed: int = 0) -> FourierEncoder:
    """nn.py:79-93 semantics: "off" (or m == 0), "nerf" (m % d_in == 0), "random"."""
    if m < 0:
        raise ValueError("m must be non-negative")
    if mode == "off" or m == 0:
        return FourierEncoder("off", np.zeros((0, d_in), np.float32), d_in)
    if mode == "nerf":
        if m % d_in:
            raise ValueError(f"nerf mode needs m divisible by d_in, got m={m}, d_in={d_in}")
        return FourierEncoder("nerf", nerf_rows(m, d_in), d_in)
    if mode == "random":
        b = np.random.default_rng(seed).normal(0.0, 2.0 * np.pi * sigma, size=(m, d_in))
        return FourierEncoder("random", b.astype(np.float32), d_in, sigma, seed)
    raise ValueError(f"unknown fourier mode {mode!r}")


def fourier_encode(enc: FourierEncoder, v) -> np.ndarray:
    """[v | sin(v B^T) | cos(v B^T)] in v's dtype; mode "off" passes through (nn.py:96-105).
    Host utility on host arrays (the render / training kernels encode on chip)."""
    v = np.atleast_2d(np.asarray(v))
    if v.shape[1] != enc.d_in:
        raise ValueError(f"expected {enc.d_in} input components, got {v.shape[1]}")
    if enc.m == 0:
        return v
    phase = v @ enc.b_matrix.T.astype(v.dtype)
    return np.concatenate([v, np.sin(phase), np.cos(phase)], axis=1)


@dataclass
class MlpParams:
    """(out, in) weight matrices + biases; hidden layers share one activation."""

    weights: list
    biases: list
    activation: str = "snake_alt"

    def __post_init__(self):
        if not self.weights or len(self.weights) != len(self.biases):
            raise ValueError("weights and biases must be non-empty and equal length")
        prev = None
        for i, (w, b) in enumerate(zip(self.weights, self.biases)):
            if w.ndim != 2 or b.shape != (w.shape[0],):
                raise ValueError(f"layer {i} has inconsistent shapes {w.shape} / {b.shape}")
            if prev is not None and w.shape[1] != prev:
                raise ValueError(f"layer {i} input width does not chain")
            prev = w.shape[0]
        if self.activation not in ACTIVATION_KINDS:
            raise ValueError(f"unknown activation kind {self.activation!r}")

    @property
    def layer_count(self) -> int:
        return len(self.weights)

    @property
    def d_in(self) -> int:
        return int(self.weights[0].shape[1])

    @property
    def d_out(self) -> int:
        return int(self.weights[-1].shape[0])

    @property
    def hidden_channels(self) -> int:
        return int(self.weights[0].shape[0])

    @property
    def param_count(self) -> int:
        return int(sum(w.size + b.size for w, b in zip(self.weights, self.biases)))


def init_params(layer_count: int, hidden: int, d_in: int, d_out: int, seed: int = 0,
                activation: str = "snake_alt", dtype=np.float32) -> MlpParams:
    """Xavier-uniform weights (drawn layer by layer from one generator), zero biases."""
    if layer_count < 1:
        raise ValueError("need at least one layer")
    dims = [d_in, *([hidden] * (layer_count - 1)), d_out]
    gen = np.random.default_rng(seed)
    ws, bs = [], []
    for fan_in, fan_out in zip(dims[:-1], dims[1:]):
        lim = np.sqrt(6.0 / (fan_in + fan_out))
        ws.append(gen.uniform(-lim, lim, size=(fan_out, fan_in)).astype(dtype))
        bs.append(np.zeros(fan_out, dtype=dtype))
    return MlpParams(ws, bs, activation)


def act_eval(kind: str, x: np.ndarray) -> np.ndarray:
    """Activation functions (nn.py:18-29); host utility (the kernels evaluate them fused)."""
    if kind == "relu":
        return np.maximum(x, 0.0)
    if kind == "sigmoid":
        return 1.0 / (1.0 + np.exp(-x))
    if kind == "softplus":
        return np.logaddexp(0.0, x)
    if kind == "snake":
        return x + np.sin(x) ** 2
    if kind == "snake_alt":
        return 0.5 * x + np.sin(x) ** 2
    raise ValueError(f"unknown activation kind {kind!r}")


def act_grad(kind: str, x: np.ndarray) -> np.ndarray:
    """Activation derivatives (nn.py:32-44); host utility."""
    if kind == "relu":
        return (x > 0).astype(x.dtype)
    if kind == "sigmoid":
        s = 1.0 / (1.0 + np.exp(-x))
        return s * (1.0 - s)
    if kind == "softplus":
        return 1.0 / (1.0 + np.exp(-x))
    if kind == "snake":
        return 1.0 + np.sin(2.0 * x)
    if kind == "snake_alt":
        return 0.5 + np.sin(2.0 * x)
    raise ValueError(f"unknown activation kind {kind!r}")


def mlp_eval(params: MlpParams, x: np.ndarray) -> np.ndarray:
    """Forward pass of the network (nn.py:195-204) on the GPU, f32 like the reference;
    the last layer stays linear."""
    from .f32ops import NetDesc

    x = np.asarray(x)
    d_in = int(params.weights[0].shape[1])
    if x.ndim != 2 or x.shape[1] != d_in:
        raise ValueError(f"expected input shape (N, {d_in}), got {x.shape}")
    nd = NetDesc(params.weights, params.biases, params.activation, "density", d_in)
    return nd.run(3, x.shape[0], int(params.weights[-1].shape[0]), x=x)


@dataclass
class MlpCache:
    """Per-layer inputs and pre-activations of a forward pass (nn.py:172-176)."""

    inputs: list
    preacts: list


def _mlp_run(params: MlpParams, x: np.ndarray, y_bar=None):
    """One fvsrn_mlp_forward_backward call: outputs, caches and (with y_bar) the weight /
    bias / input adjoints as cuBLAS GEMMs over the cached deltas (nn.py:248-255)."""
    import ctypes as C

    import torch

    from . import _lib as L
    from .f32ops import NetDesc

    n, d_in = x.shape
    Lc = params.layer_count
    d_out = int(params.weights[-1].shape[0])
    H = int(params.weights[0].shape[0]) if Lc > 1 else 1
    nd = NetDesc(params.weights, params.biases, params.activation, "density", d_in)
    dev = nd.dev
    w_in = [d_in] + [H] * (Lc - 1)
    w_out = [H] * (Lc - 1) + [d_out]
    xd = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32), device=dev)
    yd = torch.empty((max(n, 1), d_out), dtype=torch.float32, device=dev)
    inputs = torch.empty(max(1, n * sum(w_in)), dtype=torch.float32, device=dev)
    preacts = torch.empty(max(1, (Lc - 1) * n * H), dtype=torch.float32, device=dev)
    deltas = torch.empty(max(1, n * sum(w_out)), dtype=torch.float32, device=dev)
    yb = (None if y_bar is None else
          torch.as_tensor(np.ascontiguousarray(y_bar, dtype=np.float32), device=dev))
    ptr = lambda a: C.c_void_p(a.data_ptr() if a is not None else None)  # noqa: E731
    xb = torch.empty((max(n, 1), d_in), dtype=torch.float32, device=dev) if y_bar is not None else None
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    L.check(L.lib().fvsrn_mlp_forward_backward(
        C.byref(nd.desc), ptr(nd.params), ptr(xd), ptr(yb), n, ptr(yd), ptr(inputs), ptr(preacts),
        ptr(deltas), ptr(xb), stream))
    y = yd[:n].cpu().numpy()
    ins, pre = [], []
    io = 0
    for l in range(Lc):
        ins.append(inputs[io:io + n * w_in[l]].view(n, w_in[l]).cpu().numpy())
        io += n * w_in[l]
        pre.append(preacts[l * n * H:(l + 1) * n * H].view(n, H).cpu().numpy() if l < Lc - 1 else y.copy())
    if y_bar is None:
        return y, MlpCache(inputs=ins, preacts=pre), None, None
    # nn.py:252-254: weight / bias gradients on the tensor cores (fvsrn_layer_grads), the
    # input adjoint delta_0 @ W_0 per row from the backward kernel
    nw = sum(int(w.size) for w in params.weights)
    flat = torch.zeros(nw + sum(int(b.size) for b in params.biases), dtype=torch.float32, device=dev)
    L.check(L.lib().fvsrn_layer_grads(C.byref(nd.desc), ptr(inputs), ptr(deltas), n, n, ptr(flat), 0,
                                      stream))
    host = flat.cpu().numpy()
    gw, gb, o = [], [], 0
    for w in params.weights:
        gw.append(host[o:o + w.size].reshape(w.shape).copy())
        o += w.size
    for b in params.biases:
        gb.append(host[o:o + b.size].copy())
        o += b.size
    x_bar = xb[:n].cpu().numpy()
    return y, MlpCache(inputs=ins, preacts=pre), gw, (gb, x_bar)


def mlp_forward(params: MlpParams, x: np.ndarray):
    """Evaluate the network keeping the per-layer caches (nn.py:179-193), on the GPU in
    f32; the last layer stays linear.  Returns (y, MlpCache)."""
    x = np.asarray(x)
    d_in = int(params.weights[0].shape[1])
    if x.ndim != 2 or x.shape[1] != d_in:
        raise ValueError(f"expected input shape (N, {d_in}), got {x.shape}")
    y, cache, _, _ = _mlp_run(params, x)
    return y, cache


def mlp_backward(params: MlpParams, cache: MlpCache, y_bar: np.ndarray):
    """Reverse pass for sum(y_bar * y) (nn.py:234-256): returns the input adjoints and a
    GradientBuffer of weight / bias gradients (grids empty).  The deltas come from one
    CUDA kernel (forward recomputed from cache.inputs[0]); the reductions are GEMMs."""
    from .train import GradientBuffer

    if len(cache.inputs) != params.layer_count:
        raise ValueError("cache does not match the parameter set")
    y_bar = np.asarray(y_bar)
    if y_bar.shape != np.shape(cache.preacts[-1]):
        raise ValueError(f"adjoint shape {y_bar.shape} does not match output {np.shape(cache.preacts[-1])}")
    _, _, gw, (gb, x_bar) = _mlp_run(params, np.asarray(cache.inputs[0]), y_bar)
    return x_bar, GradientBuffer(weights=gw, biases=gb, grids=[])


@dataclass
class AdamState:
    """First/second moment accumulators, one per parameter array (nn.py:258-276)."""

    m: list
    v: list
    t: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    @classmethod
    def for_arrays(cls, arrays, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8) -> "AdamState":
        return cls(m=[np.zeros_like(a) for a in arrays], v=[np.zeros_like(a) for a in arrays],
                   beta1=beta1, beta2=beta2, eps=eps)


def adam_step(arrays: list, grads: list, state: AdamState, lr: float) -> None:
    """One bias-corrected Adam update of host arrays, in place (nn.py:279-298), by the
    CUDA Adam kernel (``fvsrn_adam_step``) over one flat device buffer; the arrays and
    the moments are written back.  A non-finite gradient raises FloatingPointError and
    updates nothing (the step counter included)."""
    import ctypes as C

    import torch

    from . import _lib as L

    if len(arrays) != len(state.m) or len(grads) != len(arrays) or len(state.v) != len(arrays):
        raise ValueError("parameter/gradient/state lengths disagree")
    for p, g in zip(arrays, grads):
        if np.shape(p) != np.shape(g):
            raise ValueError(f"gradient shape {np.shape(g)} does not match parameter {np.shape(p)}")
    if not arrays:
        state.t += 1
        return
    dev = torch.device("cuda", L.current_device())

    def flat(xs):
        return torch.from_numpy(np.concatenate([np.asarray(x, dtype=np.float32).reshape(-1) for x in xs])).to(dev)

    P, G, M, V = flat(arrays), flat(grads), flat(state.m), flat(state.v)
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    L.check(L.lib().fvsrn_adam_step(C.c_void_p(P.data_ptr()), C.c_void_p(G.data_ptr()),
                                    C.c_void_p(M.data_ptr()), C.c_void_p(V.data_ptr()), P.numel(),
                                    float(lr), float(state.beta1), float(state.beta2), float(state.eps),
                                    state.t + 1, C.c_void_p(bad.data_ptr()), C.c_void_p(stream)))
    if int(bad.item()):
        raise FloatingPointError("non-finite gradient passed to adam_step")
    state.t += 1
    off = 0
    hp, hm, hv = P.cpu().numpy(), M.cpu().numpy(), V.cpu().numpy()
    for p, m, v in zip(arrays, state.m, state.v):
        k = int(np.size(p))
        p[...] = hp[off:off + k].reshape(np.shape(p))
        m[...] = hm[off:off + k].reshape(np.shape(m))
        v[...] = hv[off:off + k].reshape(np.shape(v))
        off += k
