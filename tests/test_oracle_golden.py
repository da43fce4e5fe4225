"""Pin the CPU oracle against golden vectors produced by the reference itself.

If these pass, the oracle is a faithful restatement of the reference path and
can serve as the checker for the CUDA kernels (tests/test_gpu_parity.py).
"""

import hashlib

import numpy as np
import pytest

from oracle import fvsrn_oracle as O
from tests.golden_util import arrays, meta


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _model(name):
    return O.model_init(O.OConfig(**meta()["models"][name]["config"]))


def _cam(c):
    return O.OCamera(np.array(c["eye"]), np.array(c["target"]), np.array(c["up"]),
                     c["fov_y"], c["width"], c["height"])


@pytest.mark.parametrize("name", sorted(meta()["models"]))
def test_model_init_bit_exact(name):
    m = _model(name)
    h = meta()["models"][name]["hashes"]
    assert [_sha(w) for w in m.weights] == h["weights"]
    assert [_sha(b) for b in m.biases] == h["biases"]
    assert [_sha(g) for g in m.grids] == h["grids"]
    assert _sha(m.b_matrix) == h["b_matrix"]
    assert m.config.input_width == meta()["models"][name]["input_width"]


@pytest.mark.parametrize("cam", ["fib0", "fib5", "center", "inside"])
def test_rays_and_geometry_bit_exact(cam):
    a = arrays()
    o, d = O.camera_rays(_cam(meta()["cameras"][cam]))
    assert np.array_equal(o, a[f"rays_{cam}_o"])
    assert np.array_equal(d, a[f"rays_{cam}_d"])
    tmin, ds, n = O.march_geometry(o, d, 1 / 128, 4096)
    assert np.array_equal(tmin, a[f"rays_{cam}_tmin"])
    assert np.array_equal(ds, a[f"rays_{cam}_ds"])
    assert np.array_equal(n, a[f"rays_{cam}_n"])


@pytest.mark.parametrize("name", sorted(meta()["models"]))
def test_assemble_input(name):
    a = arrays()
    m = _model(name)
    p, d = a["eval_p"][:257], a["eval_d"][:257]
    t = 6.5 if m.keyframe_times is not None else None
    x = O.assemble_input(m, p, d if m.config.direction_mode != "pos" else None, t)
    np.testing.assert_allclose(x, a[f"assemble_{name}"], atol=2e-6, rtol=0)


@pytest.mark.parametrize("name", sorted(meta()["models"]))
def test_eval(name):
    a = arrays()
    m = _model(name)
    p, d = a["eval_p"], a["eval_d"]
    if m.config.head == "density":
        if m.keyframe_times is not None:
            for tt in (1.0, 6.5, 11.0, 16.25, 21.0, 0.0, 30.0):
                np.testing.assert_allclose(O.eval_density(m, p, t=tt),
                                           a[f"density_{name}_t{tt}"], atol=2e-6)
        else:
            np.testing.assert_allclose(O.eval_density(m, p), a[f"density_{name}"], atol=2e-6)
    else:
        dd = d if m.config.direction_mode != "pos" else None
        np.testing.assert_allclose(O.eval_color(m, p, dd), a[f"color_{name}"], atol=2e-6)


@pytest.mark.parametrize("tf", ["grayscale", "warm", "two_peaks"])
def test_tf_eval(tf):
    a = arrays()
    rgb, sig = O.tf_eval(O.TF_PRESETS[tf], a["tf_density"])
    assert np.array_equal(rgb, a[f"tf_{tf}_rgb"])
    assert np.array_equal(sig, a[f"tf_{tf}_sigma"])


SMALL_RENDERS = ["cfg1_v6_warm", "cfg1_v1_peaks_bg", "tiny_center_gray", "temporal_both_t3",
                 "color_dirf", "color_pos_et", "inside_gray"]


@pytest.mark.parametrize("tag", SMALL_RENDERS)
def test_render_matches_reference(tag):
    r = meta()["renders"][tag]
    name = {"cfg1": "cfg1", "tiny": "tiny", "temporal": "temporal_both", "color": None,
            "inside": "cfg1"}[tag.split("_")[0]]
    if name is None:
        name = "color_dirf" if "dirf" in tag else "color_pos"
    if tag.startswith("temporal_both"):
        name = "temporal_both"
    m = _model(name)
    tf = O.TF_PRESETS[r["tf"]] if r["tf"] else None
    cnt = [0]
    img = O.render_image(m, tf, _cam(r["camera"]), r["stepsize"], r["max_steps"],
                         tuple(r["background"]), r["et"], t=r["t"], counter=cnt)
    ref = arrays()[f"render_{tag}"]
    assert O.metric_psnr(img, ref) > 80.0
    assert abs(cnt[0] - r["count"]) <= max(2, r["count"] // 100000)


def test_decode_matches_reference():
    a = arrays()
    np.testing.assert_allclose(O.decode_volume(_model("tiny"), 9), a["decode_tiny_9"], atol=2e-6)
    np.testing.assert_allclose(O.decode_volume(_model("cfg1"), 17), a["decode_cfg1_17"], atol=2e-6)
    np.testing.assert_allclose(O.decode_volume(_model("temporal"), 12, t=16.25),
                               a["decode_temporal_12_t16.25"], atol=2e-6)


def test_psnr_known_answers():
    x = np.zeros((4, 4, 4))
    assert O.metric_psnr(x, x) == 99.0
    assert O.metric_psnr(x, x + 1.0) == pytest.approx(0.0)
    assert O.metric_psnr(x, x + 0.1) == pytest.approx(20.0)


@pytest.mark.parametrize("tag", ["vol_sphere32_grayscale", "vol_gauss48_warm",
                                 "vol_random975_two_peaks"])
def test_volume_source_render_matches_reference(tag):
    r = meta()["renders"][tag]
    vol = O.OVolume(arrays()[f"volume_{r['volume']}"])
    img = O.render_image(vol, O.TF_PRESETS[r["tf"]], _cam(r["camera"]), r["stepsize"],
                         r["max_steps"], tuple(r["background"]), r["et"])
    assert O.metric_psnr(img, arrays()[f"render_{tag}"]) > 90.0


# ---- shape-exact fixtures (tests/golden/make_golden_shapes.py) -----------------------
def _shapes():
    import json

    from tests.golden_util import GOLDEN

    with np.load(GOLDEN / "golden_shapes.npz") as z:
        a = {k: z[k] for k in z.files}
    with open(GOLDEN / "golden_shapes.json") as f:
        return GOLDEN, a, json.load(f)


@pytest.mark.parametrize("ckpt,key,n", [("trained_cfg2.fvsrn", "trained_density", 8192),
                                        ("trained_cfg3.fvsrn", "trained3_density", 2048)])
def test_oracle_trained_checkpoint_density(ckpt, key, n):
    # the oracle's checkpoint reader + evaluator vs the reference on the trained weights
    g, a, _ = _shapes()
    om = O.checkpoint_load(g / ckpt)
    np.testing.assert_allclose(O.eval_density(om, a["trained_p"][:n]), a[key][:n], atol=2e-6)


@pytest.mark.parametrize("tag", ["cfg2_v3", "trained_v5", "cfg5_t16.25"])
def test_oracle_shape_rows(tag):
    # one row of a full-size reference frame through the oracle's raymarch (same rays)
    g, a, m = _shapes()
    r = m["renders"][tag]
    if r["model"] == "trained":
        om = O.checkpoint_load(g / "trained_cfg2.fvsrn")
    else:
        om = O.model_init(O.OConfig(**m["models"][r["model"]]))
    c = r["camera"]
    cam = O.OCamera(np.array(c["eye"]), np.array(c["target"]), np.array(c["up"]), c["fov_y"],
                    c["width"], c["height"])
    rows = a[f"rows_{tag}"]
    k = len(rows) // 2
    cnt = [0]
    img = O.render_image(om, O.TF_PRESETS[r["tf"]], cam, r["stepsize"], t=r["t"], counter=cnt,
                         rows=rows[k:k + 1])
    want = a[f"px_{tag}"].reshape(len(rows), c["width"], 4)[k]
    assert O.metric_psnr(img[rows[k]], want) > 80.0
