"""Parity margins at the BASELINE shapes and on the trained checkpoints (GPU box).

Prints, per model x latent-grid sampler: density max-abs / mean-abs error vs the pinned
oracle at 2^20 uniform positions (and its argmax position), and the PSNR of every
shape-exact reference render (tests/golden/golden_shapes.*).  Output goes to stdout;
profiles/r2/precision_shapes.txt keeps the committed copy.

    python tools/precision_shapes.py [--renders]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2112_01579_b200 as P  # noqa: E402
from oracle import fvsrn_oracle as O  # noqa: E402

G = ROOT / "tests" / "golden"


def models():
    meta = json.load(open(G / "golden_shapes.json"))
    out = {}
    for name in ("cfg2", "cfg3", "cfg5"):
        cfg = meta["models"][name]
        out[name] = (P.model_init(P.ModelConfig(**cfg)), O.model_init(O.OConfig(**cfg)))
    out["trained"] = (P.checkpoint_load(G / "trained_cfg2.fvsrn"), O.checkpoint_load(G / "trained_cfg2.fvsrn"))
    out["trained3"] = (P.checkpoint_load(G / "trained_cfg3.fvsrn"), O.checkpoint_load(G / "trained_cfg3.fvsrn"))
    return meta, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--renders", action="store_true")
    args = ap.parse_args()
    meta, ms = models()
    p = np.random.default_rng(31).uniform(0.0, 1.0, size=(1 << 20, 3))
    print("density vs pinned oracle, 2^20 uniform positions (tolerance 1e-2)")
    for name, (m, om) in ms.items():
        t = 6.5 if name == "cfg5" else None
        want = O.eval_density(om, p, t=t)
        info = P.device.device_model(m).info()
        print(f"  {name:9s} upload probe: max|tex-ldg| {info['texture_probe_err']:.3e} -> auto uses "
              f"{'tex' if info['texture_sampler_ok'] else 'ldg'}")
        for sampler in ("tex", "ldg", "auto"):
            prev = P.set_grid_sampler(sampler)
            try:
                got = P.eval_density(m, p, t=t)
            finally:
                P.set_grid_sampler(prev)
            e = np.abs(got - want)
            k = int(e.argmax())
            print(f"  {name:9s} {sampler}: max {e.max():.3e} mean {e.mean():.3e} p99.99 "
                  f"{np.quantile(e, 0.9999):.3e} at p={np.round(p[k], 4).tolist()} "
                  f"(ref {want[k]:.4f})", flush=True)
    print("decode_volume (64^3 lattice) vs pinned oracle (tolerance 1e-2)")
    axis = np.linspace(0.0, 1.0, 64)
    gx, gy, gz = np.meshgrid(axis, axis, axis, indexing="ij")
    lat = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], -1)
    for name, (m, om) in ms.items():
        t = 6.5 if name == "cfg5" else None
        want = O.eval_density(om, lat, t=t).reshape(64, 64, 64)
        P.device.kernel_timer(True)
        got = P.decode_volume(m, 64, t=t).values
        P.device.kernel_timer_read()
        kname = P.device.kernel_timer_info().split(" ")[0]
        P.device.kernel_timer(False)
        e = np.abs(got - want)
        print(f"  {name:9s} {kname}: max {e.max():.3e} mean {e.mean():.3e}", flush=True)
    if not args.renders:
        return
    a = np.load(G / "golden_shapes.npz")
    print("shape-exact renders: PSNR over the reference rows (tolerance 40 dB)")
    for tag, r in meta["renders"].items():
        mname = r["model"]
        m = ms[mname][0]
        c = r["camera"]
        cam = P.Camera(eye=c["eye"], target=c["target"], up=c["up"], fov_y=c["fov_y"],
                       width=c["width"], height=c["height"])
        src = P.ModelSource(m, P.TF_PRESETS[r["tf"]], t=r["t"])
        img = P.render_image(src, cam, P.RenderSettings(stepsize=r["stepsize"]))
        rows = a[f"rows_{tag}"]
        psnr = P.metric_psnr(img.data[rows].reshape(-1, 4), a[f"px_{tag}"])
        print(f"  {tag:16s} {psnr:6.2f} dB  ({len(rows)} rows of {c['width']}x{c['height']})", flush=True)


if __name__ == "__main__":
    main()
