"""CPU tests of the host-side mirror of the reference API and of the C-ABI library
(no compute calls: this container has no GPU)."""

import ctypes
import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2112_01579_b200 as P
from paper_2112_01579_b200 import _lib
from tests.golden_util import GOLDEN, arrays, meta

ROOT = Path(__file__).resolve().parents[1]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(meta()["models"]))
def test_model_init_bit_exact_vs_reference(name):
    m = P.model_init(P.ModelConfig(**meta()["models"][name]["config"]))
    h = meta()["models"][name]["hashes"]
    assert [_sha(w) for w in m.params.weights] == h["weights"]
    assert [_sha(b) for b in m.params.biases] == h["biases"]
    assert [_sha(g.values) for g in m.grids] == h["grids"]
    assert _sha(m.spatial_encoder.b_matrix) == h["b_matrix"]
    assert m.config.input_width == meta()["models"][name]["input_width"]


def test_config_validation_matches_reference():
    with pytest.raises(ValueError):
        P.ModelConfig(head="rgb")
    with pytest.raises(ValueError):
        P.ModelConfig(direction_mode="dirP")          # needs the colour head
    with pytest.raises(ValueError):
        P.ModelConfig(time_mode="direct")             # needs keyframes
    with pytest.raises(ValueError):
        P.ModelConfig(keyframe_times=[1, 2], grid_resolution=0)
    assert P.ModelConfig().input_width == 47
    assert P.ModelConfig(layers=6, hidden=64, fourier_m=30).input_width == 79


@pytest.mark.parametrize("name", ["tiny_f32", "tiny_f16_u8", "temporal_both_f32"])
def test_checkpoint_load_reference_files(name, tmp_path):
    m = P.checkpoint_load(GOLDEN / f"{name}.fvsrn")
    cfg_name = "temporal_both" if "temporal" in name else "tiny"
    ref = P.model_init(P.ModelConfig(**meta()["models"][cfg_name]["config"]))
    if name.endswith("f32"):
        for a, b in zip(m.params.weights, ref.params.weights):
            assert np.array_equal(a, b)
        for a, b in zip(m.grids, ref.grids):
            assert np.array_equal(a.values, b.values)
    else:
        assert m.quantized is not None and len(m.quantized) == 1
        q = P.grid_quantize(ref.grid)
        assert np.array_equal(m.quantized[0].codes, q.codes)
    # round trip through our writer
    out = tmp_path / "rt.fvsrn"
    P.checkpoint_save(m, out)
    back = P.checkpoint_load(out)
    for a, b in zip(back.params.weights, m.params.weights):
        assert np.array_equal(a, b)


def test_checkpoint_errors(tmp_path):
    m = P.model_init(P.ModelConfig(layers=2, hidden=16, fourier_m=6, grid_resolution=4,
                                   grid_channels=4, seed=7))
    p = tmp_path / "x.fvsrn"
    P.checkpoint_save(m, p)
    raw = p.read_bytes()
    (tmp_path / "bad.fvsrn").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(P.CheckpointError):
        P.checkpoint_load(tmp_path / "bad.fvsrn")
    (tmp_path / "trunc.fvsrn").write_bytes(raw[:-64])
    with pytest.raises(P.CheckpointError):
        P.checkpoint_load(tmp_path / "trunc.fvsrn")


def test_quantize_known_answers():
    v = np.zeros((2, 2, 2, 1), np.float32)
    v[0, 0, 0, 0], v[1, 1, 1, 0] = -1.0, 1.0
    assert P.grid_quantize(P.LatentGrid(v)).codes[0, 1, 0, 0] == 128
    g = P.LatentGrid(np.full((3, 3, 3, 2), 0.42, np.float32))
    q = P.grid_quantize(g)
    assert np.all(q.codes == 0)
    assert np.array_equal(P.grid_dequantize(q).values, g.values)


CAPACITY_FRONTIER = {32: 22, 48: 10, 64: 6, 96: 3, 128: 2}   # PAPER.md Table 1


@pytest.mark.parametrize("c,l", CAPACITY_FRONTIER.items())
def test_plan_build_table1_frontier(c, l):
    plan = P.plan_build(l, c, c - 1, 1)
    assert plan.resident_weight_bytes + plan.resident_scratch_bytes <= plan.budget_bytes
    with pytest.raises(P.CapacityError):
        P.plan_build(l + 1, c, c - 1, 1)


def test_plan_build_worked_example():
    plan = P.plan_build(4, 48, 47, 1)
    assert (plan.m_w, plan.m_s, plan.w) == (18816, 3072, 9)
    assert P.plan_build(4, 32, 47, 1).padded_widths == (48, 32, 32, 32, 16)


def test_transfer_function_validation():
    tf = P.TF_PRESETS["warm"]
    assert tf.max_sigma == 10.0
    with pytest.raises(ValueError):
        P.TransferFunction.from_points([(0.0, (0, 0, 0), 0.0)])
    with pytest.raises(ValueError):
        P.TransferFunction.from_points([(0.0, (0, 0, 0), 0.0), (0.5, (1, 1, 1), 1.0)])
    with pytest.raises(ValueError):
        P.TransferFunction.from_points([(0.0, (0, 0, 0), -1.0), (1.0, (1, 1, 1), 1.0)])
    back = P.tf_from_json([{"x": x, "rgb": list(r), "sigma": s}
                           for x, r, s in zip(tf.xs, tf.rgbs, tf.sigmas)])
    assert np.array_equal(back.xs, tf.xs)


def test_camera_and_settings_validation():
    with pytest.raises(ValueError):
        P.Camera(eye=(0, 0, 0), target=(0, 0, 0), up=(0, 1, 0), fov_y=1.0, width=4, height=4)
    with pytest.raises(ValueError):
        P.Camera(eye=(0, 0, 1), target=(0, 0, 0), up=(0, 0, 1), fov_y=1.0, width=4, height=4)
    with pytest.raises(ValueError):
        P.RenderSettings(stepsize=0.0)
    with pytest.raises(ValueError):
        P.RenderSettings(early_term_alpha=1.5)
    assert P.RenderSettings.for_voxels(256, 1.0).stepsize == 1.0 / 256


@pytest.mark.parametrize("cam", ["fib0", "fib5", "center", "inside"])
def test_camera_rays_bit_exact(cam):
    c = meta()["cameras"][cam]
    o, d = P.camera_rays(P.Camera(eye=c["eye"], target=c["target"], up=c["up"],
                                  fov_y=c["fov_y"], width=c["width"], height=c["height"]))
    assert np.array_equal(o, arrays()[f"rays_{cam}_o"])
    assert np.array_equal(d, arrays()[f"rays_{cam}_d"])


def test_fibonacci_cameras_match_reference_views():
    r = meta()["renders"]["cfg1_v0_gray"]["camera"]
    cam = P.fibonacci_cameras(8, 128, 128)[0]
    assert np.array_equal(cam.eye, np.array(r["eye"]))
    assert np.array_equal(cam.up, np.array(r["up"]))


def test_psnr_known_answers():
    x = np.zeros((2, 2, 4), np.float32)
    assert P.metric_psnr(x, x) == 99.0
    assert P.metric_psnr(x, x + 1) == pytest.approx(0.0)
    with pytest.raises(ValueError):
        P.metric_psnr(x, np.zeros((2, 3, 4)))


# ------------------------------------------------------------------ C ABI library
def _header_symbols():
    text = (ROOT / "include" / "fvsrn_b200.h").read_text()
    return sorted(set(re.findall(r"FVSRN_API\s+[\w\s\*]+?\b(fvsrn_\w+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.lib()
    syms = _header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS), "ctypes table and header disagree"
    assert b"sm_100a" in lib.fvsrn_version()


def test_library_reports_errors_without_gpu():
    lib = _lib.lib()
    # a null descriptor is a contract violation, reported as ValueError
    h = ctypes.c_void_p()
    rc = lib.fvsrn_model_create(None, 0, ctypes.byref(h))
    assert rc == _lib.FVSRN_EINVAL
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_library_is_sm100a_cubin():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name,cfg_name", [("cfg1_f16_u8", "cfg1"), ("temporal_f16_u8", "temporal")])
def test_checkpoint_u8_codes_match_reference_quantizer(name, cfg_name):
    """The reference-written u8 checkpoints of the default shapes carry exactly the codes
    and (min, max) of grid_quantize on the seeded grids (grid.py:157-166) -- the data the
    GPU texture path samples directly."""
    m = P.checkpoint_load(GOLDEN / f"{name}.fvsrn")
    ref = P.model_init(P.ModelConfig(**meta()["models"][cfg_name]["config"]))
    assert m.quantized is not None and len(m.quantized) == len(ref.grids)
    for q, g in zip(m.quantized, ref.grids):
        rq = P.grid_quantize(g)
        assert np.array_equal(q.codes, rq.codes)
        assert np.array_equal(q.mins, rq.mins) and np.array_equal(q.maxs, rq.maxs)


def test_host_geometry_and_compositing_utilities():
    """ray_box_intersect / composite_step / composite_invert (render.py:97-129): host
    utilities mirroring the reference on host arrays."""
    from tests.golden_util import arrays as garr

    a = garr()
    o, d = a["rays_fib0_o"], a["rays_fib0_d"]
    tmin, tmax, valid = P.ray_box_intersect(o, d)
    assert valid.sum() == (a["rays_fib0_n"] > 0).sum()
    rng = np.random.default_rng(0)
    c = rng.uniform(size=(64, 3)) * 0.3
    al = rng.uniform(size=64) * 0.5
    rgb, sig = rng.uniform(size=(64, 3)), rng.uniform(size=64) * 5
    c2, a2 = P.composite_step(c, al, rgb, sig, 0.01)
    c3, a3 = P.composite_invert(c2, a2, rgb, sig, 0.01)
    np.testing.assert_allclose(c3, c, atol=1e-12)
    np.testing.assert_allclose(a3, al, atol=1e-12)


def test_metric_ssim_vs_reference():
    # imaging.py:156-177 restated on the host (luminance, Gaussian window, K1/K2)
    a, g = arrays(), meta()["ssim"]
    assert P.metric_ssim(P.Image(a["ssim_a"]), P.Image(a["ssim_b"])) == pytest.approx(g["rgb"], abs=1e-12)
    assert P.metric_ssim(a["ssim_g1"], a["ssim_g2"]) == pytest.approx(g["gray"], abs=1e-12)
    assert P.metric_ssim(P.Image(a["ssim_a"]), P.Image(a["ssim_a"])) == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(ValueError):
        P.metric_ssim(a["ssim_g1"], a["ssim_g1"][:, :20])
    with pytest.raises(ValueError):
        P.metric_ssim(np.zeros((10, 40)), np.zeros((10, 40)))


def test_metrics_and_loss_csv_format():
    rows = meta()["evaluate_views"]["rows"]
    assert P.metrics_csv(rows) == meta()["evaluate_views"]["csv"]
    assert P.loss_csv([0.5, 0.25]) == "epoch,loss\n0,0.50000000\n1,0.25000000\n"


def test_fourier_encode_vs_reference():
    a = arrays()
    for mode, mm in (("nerf", 12), ("random", 7)):
        enc = P.fourier_make(mode, mm, 3, sigma=2.0, seed=5)
        got64 = P.fourier_encode(enc, a["fenc_v"])
        got32 = P.fourier_encode(enc, a["fenc_v"].astype(np.float32))
        assert got64.dtype == np.float64 and got32.dtype == np.float32
        np.testing.assert_array_equal(got64, a[f"fenc_{mode}_f64"])
        np.testing.assert_array_equal(got32, a[f"fenc_{mode}_f32"])
    with pytest.raises(ValueError):
        P.fourier_encode(P.fourier_make("nerf", 12, 3), np.zeros((2, 4)))


def test_gradient_buffer_helpers():
    from paper_2112_01579_b200.train import GradientBuffer

    m = P.model_init(P.ModelConfig(layers=3, hidden=16, grid_resolution=4, grid_channels=4, seed=1))
    g = m.grad_buffer()
    assert [x.shape for x in g.arrays()] == [x.shape for x in m.trainable_arrays()]
    assert g.all_finite()
    h = GradientBuffer.zeros_like_params(m.params, [x.values.shape for x in m.grids])
    for x in h.arrays():
        x += 1.0
    g.add_scaled(h, 0.5)
    assert all(np.all(x == 0.5) for x in g.arrays())
    g.weights[0][0, 0] = np.nan
    assert not g.all_finite()


# ---- the duck-typed source protocol (render.py:226): any object with sample(p, d) ----
class _HostVolume:
    """A caller-defined source: trilinear volume through a TF on host arrays."""

    def __init__(self, values, tf):
        self.vol = P.ScalarVolume(values=values)
        self.tf = tf
        self.calls = 0

    def sample(self, p, d):
        self.calls += 1
        return P.tf_eval(self.tf, P.sample_volume(self.vol, p))


@pytest.mark.parametrize("tag", ["vol_sphere32_grayscale", "vol_gauss48_warm"])
def test_duck_typed_source_matches_reference(tag):
    from tests.golden_util import arrays, meta

    r = meta()["renders"][tag]
    c = r["camera"]
    cam = P.Camera(eye=c["eye"], target=c["target"], up=c["up"], fov_y=c["fov_y"],
                   width=c["width"], height=c["height"])
    src = _HostVolume(arrays()[f"volume_{r['volume']}"], P.TF_PRESETS[r["tf"]])
    st = P.RenderSettings(stepsize=r["stepsize"], max_steps=r["max_steps"],
                          background=tuple(r["background"]), early_term_alpha=r["et"])
    img = P.render_image(src, cam, st)
    assert src.calls > 0
    assert P.metric_psnr(img, arrays()[f"render_{tag}"]) > 90.0
    o, d = P.camera_rays(cam)
    px, states = P.raymarch_forward(src, o, d, st, want_states=True)
    assert states is not None and states.alpha.shape == (len(o),)


def test_source_without_sample_is_rejected():
    cam = P.Camera(eye=(0.5, 0.5, 3.0), target=(0.5, 0.5, 0.5), up=(0, 1, 0), fov_y=0.8,
                   width=4, height=4)
    with pytest.raises(TypeError, match="sample"):
        P.render_image(object(), cam, P.RenderSettings())


def test_mode_setters_fail_without_changing_the_mode():
    # host-only entry points (no GPU needed): failures are negative status codes, so a
    # rejected selection can never be mistaken for a previous mode
    from paper_2112_01579_b200 import device as D

    before = D.set_dvr_kernel("auto")
    try:
        with pytest.raises(ValueError, match="not in this build"):
            D.set_dvr_kernel("ws")
        assert D.set_dvr_kernel("auto") == "auto"
        assert _lib.lib().fvsrn_set_grid_sampler(7) < 0
        assert _lib.lib().fvsrn_set_dvr_kernel(-3) < 0
    finally:
        D.set_dvr_kernel(before)


def test_bench_kernel_key_and_mufu_counts():
    """bench.py's ncu-capture matching and per-kernel MUFU counts (roofline.xu_pipe)."""
    import bench
    ncu_name = ("void fvsrn::dvr_tc_kernel<(int)32, (int)14, (int)4, (int)1>(fvsrn::TcNetDev, "
                "fvsrn::FeatDev, const fvsrn::TFDev *)")
    lib_name = "dvr_tc_kernel<32,14,4,1> (tcgen05.mma kind::f16, TMEM accumulators); grid: texture units"
    assert bench._kernel_key(ncu_name) == bench._kernel_key(lib_name) == "dvr_tc_kernel<32,14,4,1>"
    assert bench._kernel_key("void dvr_tc_kernel<64, 30, 6, 1>(TcNetDev)") != bench._kernel_key(lib_name)
    m32, m64 = {"layers": 4, "hidden": 32}, {"layers": 6, "hidden": 64}
    # 32-wide tcgen05: 10 of 32 cosines per row on the FMA pipe (every 3rd packed word, HFMA2),
    # + 6 NeRF sin/cos + tanh + ex2
    assert bench.mufu_per_eval_of(m32, lib_name) == 3 * 22 + 2 + 6
    # 64-wide: 10 per 32-column half (every 3rd word); the f32 dot-product row: 5 per half (every 6th)
    assert bench.mufu_per_eval_of(m64, "dvr_tc_kernel<64,30,6,1>") == 4 * 44 + 54 + 2 + 6
    # mma.sync kernels: 3 of 4 n8 column tiles' cosines on MUFU, NeRF base angles on the FMA pipe
    assert bench.mufu_per_eval_of(m32, "dvr_pair_kernel<32,4,14,4,1,8>") == 3 * 24 + 2
    # the decode: last hidden row is the f32 dot product (every 5th column), no alpha ex2
    assert bench.mufu_per_eval_of(m32, "decode_tc_kernel<32,14,4,1>") == 2 * 22 + 26 + 1 + 6
