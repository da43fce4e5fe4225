"""The fused-evaluator operator: capacity plan + ``fused_eval`` on the GPU.

``plan_build`` restates the paper's 48 KB tensor-core capacity model exactly as
the reference does (fused.py:62-101, Table 1) so existing callers keep
their plans and CapacityErrors.  ``fused_eval`` keeps the signature of
fused.py:281-301 but runs head(mlp(x)) on the B200 tensor cores
(fvsrn_fused_eval, fp16 operands / fp32 accumulate).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import CapacityError

DEFAULT_BUDGET = 48 * 1024
TILE_SAMPLES = 32
BLOCK = 16


def _pad16(n: int) -> int:
    return max(BLOCK, -(-n // BLOCK) * BLOCK)


@dataclass(frozen=True)
class FusedPlan:
    layers: int
    hidden: int
    d_in: int
    d_out: int
    padded_widths: tuple
    budget_bytes: int
    m_w: int
    m_s: int
    w: int
    resident_weight_bytes: int
    resident_scratch_bytes: int
    max_resident_tiles: int
    scratch_bytes_f32: int


def plan_build(layers: int, hidden: int, d_in: int, d_out: int,
               budget_bytes: int = DEFAULT_BUDGET) -> FusedPlan:
    """Paper accounting (2 B/entry): m_w, m_s, w; padded-shape capacity check."""
    if min(layers, hidden, d_in, d_out) < 1:
        raise ValueError("layer shape components must be positive")
    widths = (_pad16(d_in),) + (_pad16(hidden),) * (layers - 1) + (_pad16(d_out),)
    m_w = layers * 2 * hidden * (hidden + 1)
    m_s = 2 * TILE_SAMPLES * hidden
    w_entries = sum(a * b for a, b in zip(widths[:-1], widths[1:]))
    resident_w = 2 * (w_entries + sum(widths[1:]))
    resident_s = 2 * TILE_SAMPLES * max(widths)
    if resident_w + resident_s > budget_bytes:
        raise CapacityError(
            f"network does not fit the fast-memory budget: weights+biases {resident_w} bytes "
            f"plus per-tile activations {resident_s} bytes exceed {budget_bytes} bytes")
    return FusedPlan(layers, hidden, d_in, d_out, widths, budget_bytes, m_w, m_s,
                     (budget_bytes - m_w) // m_s, resident_w, resident_s,
                     (budget_bytes - resident_w) // resident_s,
                     2 * TILE_SAMPLES * max(widths) * 4)


def plan_for_model(model, budget_bytes: int = DEFAULT_BUDGET) -> FusedPlan:
    c = model.config
    return plan_build(c.layers, c.hidden, c.input_width, c.output_width, budget_bytes)


def fused_eval(plan: FusedPlan, model, x: np.ndarray, python_tiles: bool = False) -> np.ndarray:
    """head(mlp(x)) for assembled inputs x (N, d_in): (N,) density or (N, 4) colour."""
    from .device import device_model

    x = np.asarray(x, dtype=np.float32)
    if x.ndim != 2 or x.shape[1] != plan.d_in:
        raise ValueError(f"expected assembled inputs (N, {plan.d_in}), got {x.shape}")
    c = model.config
    if (plan.layers, plan.d_in, plan.d_out) != (c.layers, c.input_width, c.output_width):
        raise ValueError("model parameters do not match the plan shape")
    return device_model(model).fused_eval(x)


def warmup(plan: FusedPlan, model) -> None:
    fused_eval(plan, model, np.zeros((TILE_SAMPLES, plan.d_in), dtype=np.float32))


def naive_eval_model(model, x: np.ndarray) -> np.ndarray:
    """Layer-by-layer evaluator (fused.py:304-312): head(mlp_eval(x)) with the reference's
    f32 arithmetic on the GPU f32 evaluator (the fused path is ``fused_eval``)."""
    from .model import apply_color_head, apply_density_head
    from .nn import mlp_eval

    raw = mlp_eval(model.params, np.asarray(x, dtype=np.float32))
    return apply_density_head(raw) if model.config.head == "density" else apply_color_head(raw)


def bench_compare(model, batch_sizes: list, runs: int = 5, seed: int = 0) -> list:
    """Median throughput of the naive (f32) and fused (fp16 tensor-core) evaluators per
    batch size (fused.py:320-343); host-synchronous calls including transfers."""
    import time

    plan = plan_for_model(model)
    warmup(plan, model)
    rng = np.random.default_rng(seed)
    rows = []
    for batch in batch_sizes:
        x = rng.uniform(-1.0, 1.0, size=(batch, plan.d_in)).astype(np.float32)
        naive_eval_model(model, x)
        for name, fn in (("naive", lambda: naive_eval_model(model, x)),
                         ("fused", lambda: fused_eval(plan, model, x))):
            times = []
            for _ in range(max(runs, 5)):
                t0 = time.perf_counter()
                fn()
                times.append(time.perf_counter() - t0)
            rows.append({"batch": batch, "evaluator": name,
                         "samples_per_sec": batch / sorted(times)[len(times) // 2]})
    return rows


def bench_csv(rows: list) -> str:
    lines = ["batch,evaluator,samples_per_sec"]
    for r in rows:
        lines.append(f"{r['batch']},{r['evaluator']},{r['samples_per_sec']:.1f}")
    return "\n".join(lines) + "\n"
