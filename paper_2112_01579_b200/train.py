"""World- and screen-space training on the GPU (reference train.py:26-262).

Same names and semantics as the reference: ``WorldTrainConfig``, ``WorldTarget``,
``ErrorGrid``, ``TrainingDiverged``, ``sample_world_dataset``, ``build_error_grid``
and ``train_world(model, target, cfg, progress=None) -> (model, trace)`` -- L1 loss,
joint network + latent-grid training with Adam, optional error-grid importance
resampling.  The datasets come from the same numpy RNG draws as the reference;
every batch step runs on the device:

* ``fvsrn_train_world_grads`` (thread per sample, f32): forward with cached layer
  inputs / pre-activations, L1 adjoint (fixed-order loss reduction), head + MLP
  backward, and the latent-grid scatter as a deterministic per-vertex gather in the
  reference's order and arithmetic;
* ``fvsrn_layer_grads``: the weight/bias gradients ``delta_l^T @ inputs_l`` /
  ``sum(delta_l)`` (nn.py:252-253) on the tensor cores (mma.sync TF32, 3xTF32 split),
  fixed chunks summed in order -- no torch or cuBLAS math on the train path, gradients
  bit-identical run to run;
* ``fvsrn_adam_step`` applies adam_step (nn.py:279-298) to one flat parameter buffer
  laid out like ``FvsrnModel.trainable_arrays()``.

Screen space (``train_screen``, ``raymarch_backward``): ``fvsrn_train_screen_forward``
marches each view with f32 model evaluation and f64 compositing keeping the terminal
states, ``fvsrn_train_screen_backward`` walks every ray in reverse with the blend
inversion (constant memory per ray) and writes each sample's cache rows, and
``fvsrn_layer_grads`` reduces the weight gradients over all samples of the view.

Temporal models (``train_temporal``): per-sample timesteps drive the time features and
the keyframe bracket; the latent scatter goes to both bracketing grids.

Scope: position-input models (``train_world`` / ``train_temporal`` targets are positions).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .transfer import TransferFunction, tf_eval
from .volume import ScalarVolume, sample_volume

_ACT = {"relu": 0, "sigmoid": 1, "softplus": 2, "snake": 3, "snake_alt": 4}


class TrainingDiverged(RuntimeError):
    def __init__(self, epoch: int, message: str):
        super().__init__(f"epoch {epoch}: {message}")
        self.epoch = epoch


@dataclass
class WorldTrainConfig:
    sample_count: int = 64**3
    batch_size: int = 16384
    epochs: int = 200
    lr: float = 0.01
    seed: int = 0
    adaptive: bool = False
    resample_interval: int = 50
    error_grid_resolution: int = 32
    samples_per_voxel: int = 8

    def __post_init__(self):
        if min(self.sample_count, self.batch_size, self.epochs + 1, self.resample_interval) < 1:
            raise ValueError("counts must be positive")
        if self.batch_size > self.sample_count:
            raise ValueError("batch size cannot exceed the sample count")


@dataclass
class ErrorGrid:
    """Coarse per-voxel mean absolute prediction error."""

    values: np.ndarray  # (r, r, r)

    @property
    def resolution(self) -> int:
        return self.values.shape[0]


@dataclass
class WorldTarget:
    """Ground truth for world-space training: densities, or TF-mapped colors."""

    volume: ScalarVolume
    tf: TransferFunction | None = None

    def reference(self, p: np.ndarray) -> np.ndarray:
        dens = sample_volume(self.volume, p)
        if self.tf is None:
            return dens.astype(np.float32)
        rgb, sigma = tf_eval(self.tf, dens)
        return np.concatenate([rgb, sigma[:, None]], axis=1)


def sample_world_dataset(target: WorldTarget, count: int, sampler="uniform", seed: int = 0):
    """Draw (positions, reference values) exactly as train.py:118-133 (same RNG calls)."""
    rng = np.random.default_rng(seed)
    if isinstance(sampler, ErrorGrid) and float(sampler.values.sum()) > 0.0:
        r = sampler.resolution
        mass = sampler.values.reshape(-1).astype(np.float64)
        probs = mass / mass.sum()
        voxels = rng.choice(r**3, size=count, p=probs)
        corner = np.stack(np.unravel_index(voxels, (r, r, r)), axis=1)
        p = (corner + rng.uniform(0.0, 1.0, size=(count, 3))) / r
    else:
        p = rng.uniform(0.0, 1.0, size=(count, 3))
    return p, target.reference(p)


def _model_predict(model, p: np.ndarray) -> np.ndarray:
    from .model import eval_color, eval_density

    if model.config.head == "density":
        return eval_density(model, p)
    return eval_color(model, p)


def build_error_grid(model, target: WorldTarget, resolution: int, samples_per_voxel: int = 8,
                     seed: int = 0, t: float | None = None) -> ErrorGrid:
    """Mean absolute prediction error per voxel of an r^3 lattice (train.py:136-155);
    the predictions come from the GPU evaluation path."""
    if t is not None:
        raise ValueError("the GPU world trainer handles static models")
    rng = np.random.default_rng(seed)
    r = resolution
    corners = np.stack(np.meshgrid(*(np.arange(r),) * 3, indexing="ij"), axis=-1).reshape(-1, 3)
    err = np.zeros(r**3, dtype=np.float64)
    chunk = max(1, (1 << 18) // samples_per_voxel)
    for lo in range(0, r**3, chunk):
        c = corners[lo:lo + chunk]
        jitter = rng.uniform(0.0, 1.0, size=(len(c), samples_per_voxel, 3))
        p = ((c[:, None, :] + jitter) / r).reshape(-1, 3)
        pred = _model_predict(model, p)
        ref = target.reference(p)
        diff = np.abs(np.atleast_2d(pred.T).T - np.atleast_2d(ref.T).T)
        err[lo:lo + chunk] = diff.reshape(len(c), samples_per_voxel, -1).mean(axis=(1, 2))
    return ErrorGrid(values=err.reshape(r, r, r).astype(np.float32))


class WorldTrainer:
    """Device-resident trainable state of one model: the flat f32 parameter buffer
    (trainable_arrays order), its gradient buffer and the Adam moments."""

    def __init__(self, model, device: int | None = None):
        import torch

        cfg = model.config
        if cfg.direction_mode != "pos":
            raise ValueError("the GPU world trainer handles position-input models")
        if cfg.fourier_mode not in ("off", "nerf", "random") or (
                model.spatial_encoder.m > 0 and model.spatial_encoder.b_matrix.shape[1] != 3):
            raise ValueError("unsupported spatial encoder")
        self.torch = torch
        self.dev = torch.device("cuda", L.current_device() if device is None else device)
        self.model = model
        arrays = model.trainable_arrays()
        self.shapes = [a.shape for a in arrays]
        self.sizes = [int(a.size) for a in arrays]
        flat = np.concatenate([np.ascontiguousarray(a, dtype=np.float32).reshape(-1) for a in arrays])
        self.params = torch.from_numpy(flat).to(self.dev)
        self.grads = torch.zeros_like(self.params)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.t = 0
        n_layers = model.params.layer_count
        self.n_layers = n_layers
        offs = np.concatenate([[0], np.cumsum(self.sizes)])
        self._views = [(int(offs[i]), int(offs[i + 1])) for i in range(len(arrays))]
        self.grid_off = int(offs[2 * n_layers]) if len(arrays) > 2 * n_layers else 0
        m = model.spatial_encoder.m
        self.bmat = (torch.from_numpy(np.ascontiguousarray(model.spatial_encoder.b_matrix,
                                                           dtype=np.float32)).to(self.dev)
                     if m > 0 else None)
        self.desc = L.TrainDesc(n_layers, cfg.hidden, cfg.input_width, cfg.output_width,
                                _ACT[cfg.activation], 0 if cfg.head == "density" else 1, m,
                                self.bmat.data_ptr() if m > 0 else None,
                                cfg.grid_resolution, cfg.grid_channels if cfg.grid_resolution else 0)
        if model.is_temporal:      # model.py:190-245 (host arrays kept alive with the desc)
            self._kf = np.ascontiguousarray(model.keyframes.times, dtype=np.float64)
            mode = {"none": 0, "direct": 1, "fourier": 2, "both": 3}[cfg.time_mode]
            self._tb = (np.ascontiguousarray(model.time_encoder.b_matrix, dtype=np.float32).reshape(-1)
                        if mode & 2 else np.zeros(1, np.float32))
            t0, t1 = cfg.time_range if cfg.time_range is not None else model.keyframes.span
            self.desc.n_keyframes = len(self._kf)
            self.desc.keyframe_times = L.dptr(self._kf)
            self.desc.time_mode = mode
            self.desc.time_fourier_count = cfg.time_fourier_count
            self.desc.time_b = L.fptr(self._tb)
            self.desc.time_t0, self.desc.time_t1 = float(t0), float(t1)
        self.widths_in = [cfg.input_width] + [cfg.hidden] * (n_layers - 1)
        self.widths_out = [cfg.hidden] * (n_layers - 1) + [cfg.output_width]
        self._scratch_n = -1
        self.loss_sum = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.nonfinite = torch.zeros(1, dtype=torch.int64, device=self.dev)

    def _scratch(self, n: int):
        if n != self._scratch_n:
            t = self.torch
            self.inputs = t.empty(n * sum(self.widths_in), dtype=t.float32, device=self.dev)
            self.deltas = t.empty(n * sum(self.widths_out), dtype=t.float32, device=self.dev)
            self.preacts = t.empty(max(1, (self.n_layers - 1) * n * self.model.config.hidden),
                                   dtype=t.float32, device=self.dev)
            self._scratch_n = n

    def gradients(self, positions, reference, times=None) -> float:
        """Fill self.grads for one batch (device tensors or numpy; ``times`` per sample for
        temporal models); returns the batch L1 loss (mean over samples and channels,
        train.py:158-161)."""
        t = self.torch
        if self.model.is_temporal != (times is not None):
            raise ValueError("temporal models need per-sample times (and only they)")
        tt = (t.as_tensor(times, dtype=t.float64, device=self.dev).reshape(-1).contiguous()
              if times is not None else None)
        pos = t.as_tensor(positions, dtype=t.float64, device=self.dev).contiguous()
        ref = t.as_tensor(reference, dtype=t.float32, device=self.dev).reshape(len(pos), -1).contiguous()
        n = len(pos)
        self._scratch(n)
        self.grads.zero_()
        self.loss_sum.zero_()
        stream = t.cuda.current_stream(self.dev).cuda_stream
        grid_ptr = self.grads.data_ptr() + 4 * self.grid_off if self.model.config.grid_resolution else None
        L.check(L.lib().fvsrn_train_world_grads(
            C.byref(self.desc), C.c_void_p(self.params.data_ptr()), C.c_void_p(pos.data_ptr()),
            C.c_void_p(tt.data_ptr() if tt is not None else None),
            C.c_void_p(ref.data_ptr()), n, C.c_void_p(grid_ptr), C.c_void_p(self.inputs.data_ptr()),
            C.c_void_p(self.preacts.data_ptr()), C.c_void_p(self.deltas.data_ptr()),
            C.c_void_p(self.loss_sum.data_ptr()), C.c_void_p(stream)))
        # delta_l^T @ inputs_l and sum(delta_l) (nn.py:252-253), tensor cores, deterministic
        L.check(L.lib().fvsrn_layer_grads(
            C.byref(self.desc), C.c_void_p(self.inputs.data_ptr()), C.c_void_p(self.deltas.data_ptr()),
            n, n, C.c_void_p(self.grads.data_ptr()), 0, C.c_void_p(stream)))
        return float(self.loss_sum.item()) / (n * ref.shape[1])

    def adam(self, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8) -> None:
        self.nonfinite.zero_()
        stream = self.torch.cuda.current_stream(self.dev).cuda_stream
        L.check(L.lib().fvsrn_adam_step(
            C.c_void_p(self.params.data_ptr()), C.c_void_p(self.grads.data_ptr()),
            C.c_void_p(self.m.data_ptr()), C.c_void_p(self.v.data_ptr()), self.params.numel(),
            lr, beta1, beta2, eps, self.t + 1, C.c_void_p(self.nonfinite.data_ptr()),
            C.c_void_p(stream)))
        if int(self.nonfinite.item()):
            raise FloatingPointError("non-finite gradient passed to adam_step")
        self.t += 1

    def write_back(self) -> None:
        """Copy the trained parameters into the model's arrays (and drop its render copy)."""
        flat = self.params.cpu().numpy()
        for a, (lo, hi), shape in zip(self.model.trainable_arrays(), self._views, self.shapes):
            a[...] = flat[lo:hi].reshape(shape)
        self.model.quantized = None        # the u8 codes no longer describe the grids
        self.model.invalidate_device()


def train_world(model, target: WorldTarget, cfg: WorldTrainConfig, progress=None):
    """L1 world-space training of network and grid jointly with Adam (train.py:165-206).

    Returns (model, per-epoch loss trace); the model's arrays are updated in place."""
    import torch

    if (model.config.head == "color") != (target.tf is not None):
        raise ValueError("model head does not match the training target")
    rng = np.random.default_rng(cfg.seed)
    positions, values = sample_world_dataset(target, cfg.sample_count, "uniform", cfg.seed)
    tr = WorldTrainer(model)
    pos_d = torch.as_tensor(positions, dtype=torch.float64, device=tr.dev)
    val_d = torch.as_tensor(values, dtype=torch.float32, device=tr.dev).reshape(cfg.sample_count, -1)
    trace = []
    for epoch in range(cfg.epochs):
        if cfg.adaptive and epoch > 0 and epoch % cfg.resample_interval == 0:
            tr.write_back()
            egrid = build_error_grid(model, target, cfg.error_grid_resolution,
                                     cfg.samples_per_voxel, seed=cfg.seed + epoch)
            positions, values = sample_world_dataset(target, cfg.sample_count, egrid,
                                                     seed=cfg.seed + epoch)
            pos_d = torch.as_tensor(positions, dtype=torch.float64, device=tr.dev)
            val_d = torch.as_tensor(values, dtype=torch.float32,
                                    device=tr.dev).reshape(cfg.sample_count, -1)
        perm = torch.as_tensor(rng.permutation(cfg.sample_count), device=tr.dev)
        total = 0.0
        for lo in range(0, cfg.sample_count, cfg.batch_size):
            idx = perm[lo:lo + cfg.batch_size]
            loss = tr.gradients(pos_d[idx], val_d[idx])
            if not np.isfinite(loss):
                raise TrainingDiverged(epoch, "non-finite loss")
            tr.adam(cfg.lr)
            total += loss * len(idx)
        trace.append(total / cfg.sample_count)
        if progress is not None:
            tr.write_back()            # the reference updates the model in place every step
            progress(epoch, trace[-1])
    tr.write_back()
    return model, trace


# ------------------------------------------------------------------ temporal
@dataclass
class TemporalTrainConfig:
    keyframe_times: list = field(default_factory=lambda: [1, 11, 21])
    train_times: list = field(default_factory=lambda: [1, 6, 11, 16, 21])
    world: WorldTrainConfig = field(default_factory=WorldTrainConfig)

    def __post_init__(self):
        if not self.train_times:
            raise ValueError("train_times must be non-empty")
        lo, hi = min(self.train_times), max(self.train_times)
        if len(self.keyframe_times) > 1 and (lo < self.keyframe_times[0] or hi > self.keyframe_times[-1]):
            raise ValueError("keyframes must cover the training timestep span")


def train_temporal(model, volume_provider, cfg: TemporalTrainConfig, progress=None):
    """World-space training over (position, timestep) pairs (train.py:265-314): all
    keyframe grids and the network train jointly; the latent vectors interpolate linearly
    between keyframes (the kernel scatters (1-w) z_bar / w z_bar into the bracketing pair)."""
    import torch

    if not model.is_temporal:
        raise ValueError("train_temporal requires a temporal model")
    if list(model.keyframes.times) != list(cfg.keyframe_times):
        raise ValueError("model keyframes do not match the training config")
    wc = cfg.world
    volumes = {t: volume_provider(t) for t in cfg.train_times}
    rng = np.random.default_rng(wc.seed)
    lo_t, hi_t = model.keyframes.span

    def draw(count, seed):       # the reference's draw (train.py:283-293), same RNG calls
        r = np.random.default_rng(seed)
        p = r.uniform(0.0, 1.0, size=(count, 3))
        t = r.choice(cfg.train_times, size=count)
        if len(cfg.keyframe_times) > 1:
            assert t.min() >= lo_t and t.max() <= hi_t
        v = np.empty(count, dtype=np.float32)
        for tt in np.unique(t):
            mask = t == tt
            v[mask] = sample_volume(volumes[int(tt)], p[mask])
        return p, t.astype(np.float64), v

    positions, times, values = draw(wc.sample_count, wc.seed)
    tr = WorldTrainer(model)
    pos_d = torch.as_tensor(positions, device=tr.dev)
    tim_d = torch.as_tensor(times, device=tr.dev)
    val_d = torch.as_tensor(values, device=tr.dev).reshape(-1, 1)
    trace = []
    for epoch in range(wc.epochs):
        perm = torch.as_tensor(rng.permutation(wc.sample_count), device=tr.dev)
        total = 0.0
        for lo in range(0, wc.sample_count, wc.batch_size):
            idx = perm[lo:lo + wc.batch_size]
            loss = tr.gradients(pos_d[idx], val_d[idx], tim_d[idx])
            if not np.isfinite(loss):
                raise TrainingDiverged(epoch, "non-finite loss")
            tr.adam(wc.lr)
            total += loss * len(idx)
        trace.append(total / wc.sample_count)
        if progress is not None:
            tr.write_back()            # the reference updates the model in place every step
            progress(epoch, trace[-1])
    tr.write_back()
    return model, trace


# ------------------------------------------------------------------ screen space
@dataclass
class ScreenTrainConfig:
    views: int = 96
    resolution: int = 256
    stepsize: float = 0.02
    epochs: int = 100
    lr: float = 0.01
    seed: int = 0
    reference_stepsize_voxels: float = 0.1
    camera_radius: float = 2.2

    def __post_init__(self):
        if self.views < 1 or self.stepsize <= 0:
            raise ValueError("need at least one view and a positive stepsize")


@dataclass
class GradientBuffer:
    """Gradients in the reference's GradientBuffer shape (nn.py:207-231)."""

    weights: list
    biases: list
    grids: list = field(default_factory=list)

    @classmethod
    def zeros_like_params(cls, params, grid_shapes=()) -> "GradientBuffer":
        return cls(weights=[np.zeros_like(w) for w in params.weights],
                   biases=[np.zeros_like(b) for b in params.biases],
                   grids=[np.zeros(s, dtype=np.float32) for s in grid_shapes])

    def arrays(self) -> list:
        return [*self.weights, *self.biases, *self.grids]

    def add_scaled(self, other: "GradientBuffer", scale: float = 1.0) -> None:
        for a, b in zip(self.arrays(), other.arrays()):
            a += scale * b

    def all_finite(self) -> bool:
        return all(np.all(np.isfinite(a)) for a in self.arrays())


class ScreenTrainer(WorldTrainer):
    """Adds the screen-space forward (want_states) and constant-memory backward of a
    colour-head model to the world trainer's device state."""

    CAP_ROWS = 1 << 22          # samples per backward chunk (cache rows)

    def __init__(self, model, device: int | None = None):
        if model.config.head != "color":
            raise ValueError("screen-space training requires a color-head model")
        super().__init__(model, device)
        self._cap = -1

    def forward(self, origins, dirs, settings):
        """raymarch_forward(..., want_states=True): (pixels (n,4) f32, state tuple)."""
        from .device import settings_desc

        t = self.torch
        o = t.as_tensor(origins, dtype=t.float64, device=self.dev).reshape(-1, 3).contiguous()
        d = t.as_tensor(dirs, dtype=t.float64, device=self.dev).reshape(-1, 3).contiguous()
        n = len(o)
        px = t.empty((n, 4), dtype=t.float32, device=self.dev)
        col = t.empty((n, 3), dtype=t.float64, device=self.dev)
        alp, tmin, ds = (t.empty(n, dtype=t.float64, device=self.dev) for _ in range(3))
        ns = t.empty(n, dtype=t.int32, device=self.dev)
        stream = t.cuda.current_stream(self.dev).cuda_stream
        ptr = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
        L.check(L.lib().fvsrn_train_screen_forward(
            C.byref(self.desc), ptr(self.params), ptr(o), ptr(d), n, C.byref(settings_desc(settings)),
            ptr(px), ptr(col), ptr(alp), ptr(tmin), ptr(ds), ptr(ns), C.c_void_p(stream)))
        return px, (o, d, col, alp, tmin, ds, ns)

    def _cache(self, rows: int):
        if rows > self._cap:
            t = self.torch
            self.c_inputs = t.empty(rows * sum(self.widths_in), dtype=t.float32, device=self.dev)
            self.c_deltas = t.empty(rows * sum(self.widths_out), dtype=t.float32, device=self.dev)
            self.c_preacts = t.empty(max(1, (self.n_layers - 1) * rows * self.model.config.hidden),
                                     dtype=t.float32, device=self.dev)
            self._cap = rows

    def backward(self, state, settings, image_adjoint) -> None:
        """raymarch_backward (render.py:241-306) into self.grads (zeroed first)."""
        t = self.torch
        o, d, col, alp, tmin, ds, ns = state
        adj = t.as_tensor(image_adjoint, dtype=t.float32, device=self.dev).reshape(-1, 4).contiguous()
        if not bool(t.isfinite(adj).all()):
            raise ValueError("non-finite image adjoint")
        bg = t.tensor(list(settings.background), dtype=t.float64, device=self.dev)
        self.grads.zero_()
        steps = ns.to(t.int64)
        n_host = steps.cpu().numpy()
        stream = t.cuda.current_stream(self.dev).cuda_stream
        ptr = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
        grid_ptr = (C.c_void_p(self.grads.data_ptr() + 4 * self.grid_off)
                    if self.model.config.grid_resolution else None)
        lo, n = 0, len(n_host)
        while lo < n:              # ray chunks whose samples fit the cache
            csum = np.cumsum(n_host[lo:])
            hi = lo + max(1, int(np.searchsorted(csum, self.CAP_ROWS, side="right")))
            rows = int(csum[hi - lo - 1])
            if rows:
                self._cache(rows)
                off = t.cumsum(steps[lo:hi], 0) - steps[lo:hi]
                L.check(L.lib().fvsrn_train_screen_backward(
                    C.byref(self.desc), ptr(self.params), C.c_void_p(o.data_ptr() + 24 * lo),
                    C.c_void_p(d.data_ptr() + 24 * lo), hi - lo, float(settings.eps_blend),
                    C.c_void_p(col.data_ptr() + 24 * lo), C.c_void_p(alp.data_ptr() + 8 * lo),
                    C.c_void_p(tmin.data_ptr() + 8 * lo), C.c_void_p(ds.data_ptr() + 8 * lo),
                    C.c_void_p(ns.data_ptr() + 4 * lo), ptr(off), C.c_void_p(adj.data_ptr() + 16 * lo),
                    ptr(bg), self._cap, ptr(self.c_inputs), ptr(self.c_preacts), ptr(self.c_deltas),
                    grid_ptr, C.c_void_p(stream)))
                # nn.py:252-253 summed over every sample of the chunk, added to self.grads
                L.check(L.lib().fvsrn_layer_grads(
                    C.byref(self.desc), ptr(self.c_inputs), ptr(self.c_deltas), self._cap, rows,
                    ptr(self.grads), 1, C.c_void_p(stream)))
            lo = hi

    def gradient_buffer(self) -> GradientBuffer:
        flat = self.grads.cpu().numpy()
        arrs = [flat[lo:hi].reshape(shape) for (lo, hi), shape in zip(self._views, self.shapes)]
        L_ = self.n_layers
        return GradientBuffer(arrs[:L_], arrs[L_:2 * L_], arrs[2 * L_:])


def raymarch_backward(model, origins, dirs, settings, image_adjoint, terminal_states=None,
                      t=None, grads=None) -> GradientBuffer:
    """Adjoint of raymarch_forward for a colour-head model (render.py:241-306) on the GPU:
    constant memory per ray (blend inversion), f32 model re-evaluation."""
    if t is not None:
        raise ValueError("the GPU trainer handles static models")
    tr = ScreenTrainer(model)
    _, state = tr.forward(origins, dirs, settings)
    tr.backward(state, settings, image_adjoint)
    g = tr.gradient_buffer()
    if grads is not None:
        for acc, x in zip(grads.arrays(), g.arrays()):
            acc += x
        return grads
    return g


def train_screen(model, volume, tf, cfg: ScreenTrainConfig, progress=None):
    """Image-space training: L1 against pre-rendered reference views (train.py:227-262)."""
    import torch

    from .render import RenderSettings, VolumeSource, camera_rays, fibonacci_cameras, raymarch_forward

    if model.config.head != "color":
        raise ValueError("screen-space training requires a color-head model")
    cams = fibonacci_cameras(cfg.views, cfg.resolution, cfg.resolution, radius=cfg.camera_radius)
    ref_settings = RenderSettings.for_voxels(volume.resolution, cfg.reference_stepsize_voxels)
    tr = ScreenTrainer(model)
    vsrc = VolumeSource(volume, tf)
    references = []
    for cam in cams:
        o, d = camera_rays(cam)
        pix, _ = raymarch_forward(vsrc, o, d, ref_settings)
        references.append((o, d, torch.as_tensor(pix, device=tr.dev)))
    settings = RenderSettings(stepsize=cfg.stepsize)
    trace = []
    for epoch in range(cfg.epochs):
        total = 0.0
        for o, d, ref in references:
            pix, state = tr.forward(o, d, settings)
            diff = pix - ref
            loss = float(diff.abs().mean())
            if not np.isfinite(loss):
                raise TrainingDiverged(epoch, "non-finite loss")
            tr.backward(state, settings, torch.sign(diff) / diff.numel())
            tr.adam(cfg.lr)
            total += loss
        trace.append(total / len(references))
        if progress is not None:
            tr.write_back()            # the reference updates the model in place every step
            progress(epoch, trace[-1])
    tr.write_back()
    return model, trace



# ------------------------------------------------------------------ evaluation
def evaluate_views(model, volume, tf, n_views: int = 64, resolution: int = 512,
                   stepsize_voxels: float = 1.0, t: float | None = None, use_fused: bool = True) -> list:
    """Render a deterministic orbit from the model and from the ground-truth volume, both
    on the GPU (ModelSource / VolumeSource), and score each view with PSNR and SSIM
    (train.py:317-341).  One row per view plus a trailing "mean" row."""
    from .imaging import metric_psnr, metric_ssim
    from .render import ModelSource, RenderSettings, VolumeSource, fibonacci_cameras, render_image

    cams = fibonacci_cameras(n_views, resolution, resolution)
    settings = RenderSettings.for_voxels(volume.resolution, stepsize_voxels)
    ref_source = VolumeSource(volume, tf)
    model_source = ModelSource(model, tf=tf if model.config.head == "density" else None, t=t,
                               use_fused=use_fused)
    rows = []
    for i, cam in enumerate(cams):
        ref = render_image(ref_source, cam, settings)
        img = render_image(model_source, cam, settings)
        rows.append({"view": i, "psnr": metric_psnr(img, ref), "ssim": metric_ssim(img, ref)})
    rows.append({"view": "mean", "psnr": float(np.mean([r["psnr"] for r in rows])),
                 "ssim": float(np.mean([r["ssim"] for r in rows]))})
    return rows


def metrics_csv(rows: list) -> str:
    lines = ["view,psnr,ssim"]
    for r in rows:
        lines.append(f"{r['view']},{r['psnr']:.4f},{r['ssim']:.6f}")
    return "\n".join(lines) + "\n"


def loss_csv(trace: list) -> str:
    lines = ["epoch,loss"]
    for i, v in enumerate(trace):
        lines.append(f"{i},{v:.8f}")
    return "\n".join(lines) + "\n"
