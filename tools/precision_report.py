"""Parity margins per DVR kernel x grid sampler vs the reference goldens (GPU box).

    python tools/precision_report.py > profiles/r1/precision.txt
"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np

import paper_2112_01579_b200 as P
from paper_2112_01579_b200 import device as D
from tests.golden_util import arrays, meta

A, M = arrays(), meta()


def model(name):
    return P.model_init(P.ModelConfig(**M["models"][name]["config"]))


def cam(c):
    return P.Camera(eye=c["eye"], target=c["target"], up=c["up"], fov_y=c["fov_y"],
                    width=c["width"], height=c["height"])


RENDERS = {"cfg1_v1_peaks_bg": "cfg1", "cfg2_v2_gray": "cfg2", "cfg3_v0_gray_48": "cfg3",
           "inside_gray": "cfg1", "temporal_t6.5": "temporal"}
for sampler in ("tex", "ldg"):
    D.set_grid_sampler(sampler)
    errs = {n: float(np.abs(P.eval_density(model(n), A["eval_p"]) - A[f"density_{n}"]).max())
            for n in ("cfg1", "cfg2", "cfg3")}
    errs["temporal_t6.5"] = float(np.abs(P.eval_density(model("temporal"), A["eval_p"], t=6.5)
                                         - A["density_temporal_t6.5"]).max())
    print(f"sampler={sampler} density max-abs vs reference: " +
          ", ".join(f"{k} {v:.2e}" for k, v in errs.items()))
    for kernel in ("warp", "tc"):
        D.set_dvr_kernel(kernel)
        out = []
        for tag, mn in RENDERS.items():
            r = M["renders"][tag]
            src = P.ModelSource(model(mn), P.TF_PRESETS[r["tf"]], t=r["t"])
            s = P.RenderSettings(stepsize=r["stepsize"], max_steps=r["max_steps"],
                                 background=tuple(r["background"]), early_term_alpha=r["et"])
            img = P.render_image(src, cam(r["camera"]), s)
            out.append(f"{tag} {P.metric_psnr(img, A[f'render_{tag}']):.1f} dB "
                       f"(evals {src.last_eval_count - r['count']:+d})")
        print(f"  kernel={kernel}: " + "; ".join(out))
D.set_dvr_kernel("auto")
D.set_grid_sampler("auto")
