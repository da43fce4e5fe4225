"""GPU parity: the CUDA path (through the C ABI) vs reference goldens and the oracle.

Tolerances (north star): per-sample density max-abs <= 1e-2 (fp16 operands vs
the fp32 reference), rendered images PSNR >= 40 dB.  Ray geometry is
bit-exact (the evaluated-sample count with early termination disabled equals
the reference's sum of per-ray step counts exactly).
"""

import numpy as np
import pytest

import paper_2112_01579_b200 as P
from oracle import fvsrn_oracle as O
from tests.golden_util import GOLDEN, arrays, meta

pytestmark = pytest.mark.gpu

DENS_TOL = 1e-2


def _model(name):
    return P.model_init(P.ModelConfig(**meta()["models"][name]["config"]))


def _omodel(name):
    return O.model_init(O.OConfig(**meta()["models"][name]["config"]))


def _cam(c):
    return P.Camera(eye=c["eye"], target=c["target"], up=c["up"], fov_y=c["fov_y"],
                    width=c["width"], height=c["height"])


DENSITY_MODELS = ["cfg1", "cfg2", "cfg3", "tiny", "random_fourier", "relu_nogrid", "snake_f12"]


@pytest.mark.parametrize("name", DENSITY_MODELS)
def test_eval_density_vs_reference(name):
    got = P.eval_density(_model(name), arrays()["eval_p"])
    want = arrays()[f"density_{name}"]
    err = np.abs(got - want).max()
    assert err <= DENS_TOL, f"{name}: max abs density error {err:.3e}"


@pytest.mark.parametrize("tt", [1.0, 6.5, 11.0, 16.25, 21.0, 0.0, 30.0])
def test_eval_density_temporal(tt):
    got = P.eval_density(_model("temporal"), arrays()["eval_p"], t=tt)
    assert np.abs(got - arrays()[f"density_temporal_t{tt}"]).max() <= DENS_TOL
    got = P.eval_density(_model("temporal_both"), arrays()["eval_p"], t=tt)
    assert np.abs(got - arrays()[f"density_temporal_both_t{tt}"]).max() <= DENS_TOL


@pytest.mark.parametrize("name", ["color_dirf", "color_pos"])
def test_eval_color_vs_reference(name):
    m = _model(name)
    d = arrays()["eval_d"] if m.config.direction_mode != "pos" else None
    got = P.eval_color(m, arrays()["eval_p"], d)
    want = arrays()[f"color_{name}"]
    assert np.abs(got - want).max() <= DENS_TOL


@pytest.mark.parametrize("name", ["cfg1", "color_pos", "random_fourier"])
def test_fused_eval_operator(name):
    m = _model(name)
    got = P.fused_eval(P.plan_build(m.config.layers, m.config.hidden, m.config.input_width,
                                    m.config.output_width, budget_bytes=1 << 30), m,
                       arrays()[f"fused_x_{name}"])
    assert np.abs(got - arrays()[f"fused_y_{name}"]).max() <= DENS_TOL


def test_fused_eval_interleaved_shapes():
    # launches of one kernel with different shared-memory sizes, in both orders (the
    # per-kernel smem attribute must cover every cached configuration), and a failed
    # call must not poison the next one
    ms = {n: _model(n) for n in ("cfg1", "color_pos", "random_fourier")}
    for name in ["random_fourier", "cfg1", "color_pos", "random_fourier", "cfg1"]:
        m = ms[name]
        got = P.fused_eval(P.plan_build(m.config.layers, m.config.hidden, m.config.input_width,
                                        m.config.output_width, budget_bytes=1 << 30), m,
                           arrays()[f"fused_x_{name}"])
        assert np.abs(got - arrays()[f"fused_y_{name}"]).max() <= DENS_TOL, name
    P.bench_compare(ms["cfg1"], [1024], runs=1)


def test_decode_vs_reference():
    a = arrays()
    v = P.decode_volume(_model("tiny"), 9).values
    assert np.abs(v - a["decode_tiny_9"]).max() <= DENS_TOL
    v = P.decode_volume(_model("cfg1"), 17).values
    assert np.abs(v - a["decode_cfg1_17"]).max() <= DENS_TOL
    v = P.decode_volume(_model("temporal"), 12, t=16.25).values
    assert np.abs(v - a["decode_temporal_12_t16.25"]).max() <= DENS_TOL


@pytest.mark.parametrize("kernel", ["tc", "warp"])
def test_decode_kernels_vs_oracle(kernel):
    """The tcgen05 lattice decode (default for the default shapes) and the mma.sync one,
    each against the oracle on a whole 48^3 lattice, and launched as named."""
    from paper_2112_01579_b200 import device as D

    m, om = _model("cfg2"), _omodel("cfg2")
    prev = D.set_dvr_kernel(kernel)
    try:
        D.kernel_timer(True)
        vol = P.decode_volume(m, 48).values
        D.kernel_timer_read()
        name = D.kernel_timer_info()
        D.kernel_timer(False)
    finally:
        D.set_dvr_kernel(prev)
    assert ("decode_tc_kernel" in name) == (kernel == "tc"), name
    axis = np.linspace(0.0, 1.0, 48)
    gx, gy, gz = np.meshgrid(axis, axis, axis, indexing="ij")
    want = O.eval_density(om, np.stack([gx.ravel(), gy.ravel(), gz.ravel()], -1)).reshape(48, 48, 48)
    assert np.abs(vol - want).max() <= DENS_TOL


def test_decode_full_256_vs_oracle_slices():
    # config 4: full 256^3 decode on the GPU; oracle on two lattice slabs
    m, om = _model("cfg2"), _omodel("cfg2")
    vol = P.decode_volume(m, 256).values
    assert vol.shape == (256, 256, 256)
    axis = np.linspace(0.0, 1.0, 256)
    for ix in (0, 137, 255):
        gy, gz = np.meshgrid(axis, axis, indexing="ij")
        pts = np.stack([np.full(gy.size, axis[ix]), gy.ravel(), gz.ravel()], -1)
        want = O.eval_density(om, pts).reshape(256, 256)
        assert np.abs(vol[ix] - want).max() <= DENS_TOL


RENDER_MODEL = {"cfg1_v0_gray": "cfg1", "cfg1_v3_gray": "cfg1", "cfg1_v6_warm": "cfg1",
                "cfg1_v1_peaks_bg": "cfg1", "cfg2_v2_gray": "cfg2", "tiny_center_gray": "tiny",
                "temporal_t6.5": "temporal", "temporal_both_t3": "temporal_both",
                "color_dirf": "color_dirf", "color_pos_et": "color_pos", "inside_gray": "cfg1",
                "cfg3_v0_gray_48": "cfg3", "cfg2_ragged_cap": "cfg2"}


@pytest.mark.parametrize("tag", sorted(RENDER_MODEL))
def test_render_vs_reference(tag):
    r = meta()["renders"][tag]
    m = _model(RENDER_MODEL[tag])
    tf = P.TF_PRESETS[r["tf"]] if r["tf"] else None
    src = P.ModelSource(m, tf, t=r["t"], use_fused=True)
    s = P.RenderSettings(stepsize=r["stepsize"], max_steps=r["max_steps"],
                         background=tuple(r["background"]), early_term_alpha=r["et"])
    img = P.render_image(src, _cam(r["camera"]), s)
    psnr = P.metric_psnr(img, arrays()[f"render_{tag}"])
    assert psnr >= 40.0, f"{tag}: PSNR {psnr:.2f} dB"
    # evaluated-sample count: identical up to early-termination threshold crossings
    # (a ray whose opacity lands within fp16 noise of 0.999 may stop one step
    # later, or run on through a transparent TF gap); <= 0.1%.  The exact-count
    # gate is test_ray_geometry_bit_exact_count (ET disabled).
    assert abs(src.last_eval_count - r["count"]) <= max(4, r["count"] // 1000), \
        (src.last_eval_count, r["count"])
    if r["et"] >= 1.0:   # ET off: the count is the bit-exact geometry's sum of n
        assert src.last_eval_count == r["count"]


@pytest.mark.parametrize("cam", ["fib0", "fib5", "center", "inside"])
def test_ray_geometry_bit_exact_count(cam):
    # ET disabled -> the count is exactly sum_n of render.py:189-200 (bit-exact f64 geometry)
    c = _cam(meta()["cameras"][cam])
    src = P.ModelSource(_model("tiny"), P.TF_PRESETS["grayscale"])
    P.render_image(src, c, P.RenderSettings(stepsize=1 / 128, early_term_alpha=1.0))
    assert src.last_eval_count == int(arrays()[f"rays_{cam}_n"].sum())


def test_camera_rays_host_bit_exact():
    for cam in ("fib0", "fib5", "center", "inside"):
        o, d = P.camera_rays(_cam(meta()["cameras"][cam]))
        assert np.array_equal(o, arrays()[f"rays_{cam}_o"])
        assert np.array_equal(d, arrays()[f"rays_{cam}_d"])


def test_raymarch_forward_explicit_rays():
    a = arrays()
    src = P.ModelSource(_model("cfg1"), P.TF_PRESETS["warm"])
    px, st = P.raymarch_forward(src, a["rays_explicit_o"], a["rays_explicit_d"],
                                P.RenderSettings(stepsize=1 / 300, max_steps=200))
    assert st is None
    assert O.metric_psnr(px, a["rays_explicit_px"]) >= 40.0
    px2, st2 = P.raymarch_forward(src, a["rays_explicit_o"], a["rays_explicit_d"],
                                  P.RenderSettings(stepsize=1 / 300, max_steps=200),
                                  want_states=True)
    assert st2.alpha.shape == (64,) and np.all(st2.alpha < 1.0)


def test_render_deterministic_and_background():
    m = _model("cfg1")
    src = P.ModelSource(m, P.TF_PRESETS["warm"])
    cam = P.fibonacci_cameras(8, 96, 80)[2]
    s = P.RenderSettings(stepsize=1 / 128, background=(0.2, 0.3, 0.4))
    a = P.render_image(src, cam, s).data
    b = P.render_image(src, cam, s).data
    assert np.array_equal(a, b)
    miss = a[..., 3] == 0
    assert miss.any()
    np.testing.assert_array_equal(a[miss][:, :3],
                                  np.broadcast_to(np.float32([0.2, 0.3, 0.4]), (miss.sum(), 3)))


def test_render_cfg2_1024_rows_vs_oracle():
    # BASELINE config 2 at full size on the GPU; oracle on every 64th row
    m, om = _model("cfg2"), _omodel("cfg2")
    cam = P.fibonacci_cameras(8, 1024, 1024)[1]
    src = P.ModelSource(m, P.TF_PRESETS["grayscale"])
    img = P.render_image(src, cam, P.RenderSettings(stepsize=1 / 256)).data
    rows = np.arange(0, 1024, 64)
    ocam = O.OCamera(cam.eye, cam.target, cam.up, cam.fov_y, 1024, 1024)
    ref = O.render_image(om, O.TF_PRESETS["grayscale"], ocam, 1 / 256, rows=rows)
    assert O.metric_psnr(img[rows], ref[rows]) >= 40.0
    assert 70e6 < src.last_eval_count < 110e6


def test_shards_reassemble_bit_identical():
    torch = pytest.importorskip("torch")
    from paper_2112_01579_b200 import device as D

    m = _model("cfg1")
    src = P.ModelSource(m, P.TF_PRESETS["grayscale"])
    cam = P.fibonacci_cameras(8, 123, 77)[4]
    s = P.RenderSettings(stepsize=1 / 128)
    full = P.render_image(src, cam, s).data
    for world in (2, 3, 8):
        _, per_rank = D.shard_slots(cam.width, cam.height, world)
        gathered = torch.zeros((world, per_rank, 4), dtype=torch.float32, device="cuda")
        stream = torch.cuda.current_stream().cuda_stream
        for r in range(world):
            src.device_model.render_device(src.tf, cam, s, None, gathered[r].data_ptr(), None,
                                           stream, rank=r, world=world, compact=True)
        frame = torch.zeros((cam.height, cam.width, 4), dtype=torch.float32, device="cuda")
        D.tiles_to_frame_device(gathered.data_ptr(), cam.width, cam.height, world,
                                frame.data_ptr(), stream)
        torch.cuda.synchronize()
        assert np.array_equal(frame.cpu().numpy(), full), world


@pytest.mark.parametrize("name", ["tiny_f32", "tiny_f16_u8", "temporal_both_f32"])
def test_reference_checkpoints(name):
    m = P.checkpoint_load(GOLDEN / f"{name}.fvsrn")
    t = 3.0 if m.is_temporal else None
    got = P.eval_density(m, arrays()["eval_p"][:512], t=t)
    assert np.abs(got - arrays()[f"ckpt_{name}_density"]).max() <= DENS_TOL


def test_contract_errors():
    m = _model("tiny")
    with pytest.raises(ValueError):
        P.ModelSource(m)                                  # density head needs a TF
    with pytest.raises(ValueError):
        P.ModelSource(m, P.TF_PRESETS["grayscale"], t=1.0)
    with pytest.raises(ValueError):
        P.eval_density(_model("color_pos"), np.zeros((4, 3)))
    with pytest.raises(ValueError):
        P.eval_density(_model("temporal"), np.zeros((4, 3)))   # missing t
    with pytest.raises(TypeError):
        P.render_image(object(), P.fibonacci_cameras(1, 8, 8)[0])


def test_empty_and_single_ray():
    src = P.ModelSource(_model("tiny"), P.TF_PRESETS["grayscale"])
    px, _ = P.raymarch_forward(src, np.zeros((0, 3)), np.zeros((0, 3)), P.RenderSettings())
    assert px.shape == (0, 4)
    img = P.render_image(src, P.fibonacci_cameras(1, 1, 1)[0], P.RenderSettings())
    assert img.data.shape == (1, 1, 4)
    assert P.eval_density(_model("tiny"), np.zeros((0, 3))).shape == (0,)


# ------------------------------------------------------------------ VolumeSource
@pytest.mark.parametrize("tag", ["vol_sphere32_grayscale", "vol_gauss48_warm",
                                 "vol_random975_two_peaks"])
def test_volume_source_vs_reference(tag):
    r = meta()["renders"][tag]
    vol = P.ScalarVolume(arrays()[f"volume_{r['volume']}"])
    src = P.VolumeSource(vol, P.TF_PRESETS[r["tf"]])
    s = P.RenderSettings(stepsize=r["stepsize"], max_steps=r["max_steps"],
                         background=tuple(r["background"]), early_term_alpha=r["et"])
    img = P.render_image(src, _cam(r["camera"]), s)
    assert P.metric_psnr(img, arrays()[f"render_{tag}"]) >= 60.0


def test_volume_source_empty_and_beer_lambert():
    # tests/test_render.py:208-226 of the reference, on the GPU path
    empty = P.ScalarVolume(np.zeros((8, 8, 8), np.float32))
    cam = P.Camera(eye=(0.5, 0.5, 3.5), target=(0.5, 0.5, 0.5), up=(0, 1, 0), fov_y=np.pi / 5,
                   width=9, height=9)
    img = P.render_image(P.VolumeSource(empty, P.TF_PRESETS["grayscale"]), cam,
                         P.RenderSettings(stepsize=0.05, background=(0.2, 0.3, 0.4)))
    np.testing.assert_allclose(img.data[:, :, :3], np.broadcast_to([0.2, 0.3, 0.4], (9, 9, 3)),
                               atol=1e-6)
    ones = P.ScalarVolume(np.ones((4, 4, 4), np.float32))
    tf = P.TransferFunction.from_points([(0.0, (1, 1, 1), 8.0), (1.0, (1, 1, 1), 8.0)])
    px, _ = P.raymarch_forward(P.VolumeSource(ones, tf), np.array([[0.5, 0.5, -1.0]]),
                               np.array([[0.0, 0.0, 1.0]]), P.RenderSettings(stepsize=1.0 / 1000))
    assert px[0, 3] == pytest.approx(1 - np.exp(-8.0), rel=0.01)


def test_model_vs_dense_decode_on_gpu():
    # tests/test_render.py:236-243: render the model and its 64^3 decode, PSNR > 40 dB
    m = _model("tiny")
    s = P.RenderSettings.for_voxels(64, 1.0)
    cam = P.Camera(eye=(0.5, 0.5, 2.5), target=(0.5, 0.5, 0.5), up=(0, 1, 0), fov_y=np.pi / 5,
                   width=48, height=48)
    img_model = P.render_image(P.ModelSource(m, P.TF_PRESETS["grayscale"]), cam, s)
    img_dec = P.render_image(P.VolumeSource(P.decode_volume(m, 64), P.TF_PRESETS["grayscale"]),
                             cam, s)
    assert P.metric_psnr(img_model, img_dec) > 40.0


@pytest.mark.parametrize("sampler", ["tex", "ldg"])
@pytest.mark.parametrize("kernel", ["tc", "ws", "warp", "pipe", "dual"])
@pytest.mark.parametrize("tag", ["cfg1_v1_peaks_bg", "cfg2_v2_gray", "cfg3_v0_gray_48", "inside_gray",
                                 "temporal_t6.5"])
def test_dvr_kernel_variants(kernel, tag, sampler):
    """Every DVR kernel (tcgen05/TMEM, warp-specialised and single-role mma.sync) with
    either latent-grid sampler (texture units / LDG + HFMA2) renders the reference image
    (PSNR >= 40 dB) with the reference's evaluated-sample count."""
    from paper_2112_01579_b200 import device as D

    try:
        prev = D.set_dvr_kernel(kernel)
    except ValueError:
        pytest.skip(f"{kernel}: measured-slower A/B variant, not in the default build")
    prev_s = D.set_grid_sampler(sampler)
    try:
        r = meta()["renders"][tag]
        src = P.ModelSource(_model(RENDER_MODEL[tag]), P.TF_PRESETS[r["tf"]], t=r["t"])
        s = P.RenderSettings(stepsize=r["stepsize"], max_steps=r["max_steps"],
                             background=tuple(r["background"]), early_term_alpha=r["et"])
        img = P.render_image(src, _cam(r["camera"]), s)
        assert P.metric_psnr(img, arrays()[f"render_{tag}"]) >= 40.0
        assert abs(src.last_eval_count - r["count"]) <= max(4, r["count"] // 1000)
        # ET disabled: exact reference step count through this kernel too
        c = _cam(meta()["cameras"]["fib0"])
        src2 = P.ModelSource(_model("cfg1"), P.TF_PRESETS["grayscale"])
        P.render_image(src2, c, P.RenderSettings(stepsize=1 / 128, early_term_alpha=1.0))
        assert src2.last_eval_count == int(arrays()["rays_fib0_n"].sum())
    finally:
        D.set_dvr_kernel(prev)
        D.set_grid_sampler(prev_s)


@pytest.mark.parametrize("sampler", ["tex", "ldg"])
def test_grid_sampler_density_and_decode(sampler):
    """Per-sample densities (static and temporal) and the lattice decode through each
    latent-grid sampler stay within the north-star tolerance of the reference."""
    from paper_2112_01579_b200 import device as D

    prev = D.set_grid_sampler(sampler)
    try:
        for name in ("cfg1", "cfg2", "cfg3"):
            got = P.eval_density(_model(name), arrays()["eval_p"])
            assert np.abs(got - arrays()[f"density_{name}"]).max() <= DENS_TOL, name
        for tt in (1.0, 6.5, 16.25, 30.0):
            got = P.eval_density(_model("temporal"), arrays()["eval_p"], t=tt)
            assert np.abs(got - arrays()[f"density_temporal_t{tt}"]).max() <= DENS_TOL, tt
        v = P.decode_volume(_model("cfg1"), 17).values
        assert np.abs(v - arrays()["decode_cfg1_17"]).max() <= DENS_TOL
    finally:
        D.set_grid_sampler(prev)


@pytest.mark.parametrize("kernel", ["tc", "warp", "pipe", "dual"])
def test_dvr_kernel_cfg2_full_frame_and_shards(kernel):
    """Full 1024^2 config-2 frame per kernel vs the oracle on sampled rows, explicit-ray
    marching, and shard reassembly bit-identical to the 1-GPU frame."""
    torch = pytest.importorskip("torch")
    from paper_2112_01579_b200 import device as D

    try:
        prev = D.set_dvr_kernel(kernel)
    except ValueError:
        pytest.skip(f"{kernel}: measured-slower A/B variant, not in the default build")
    try:
        m, om = _model("cfg2"), _omodel("cfg2")
        cam = P.fibonacci_cameras(8, 1024, 1024)[3]
        src = P.ModelSource(m, P.TF_PRESETS["grayscale"])
        s = P.RenderSettings(stepsize=1 / 256)
        img = P.render_image(src, cam, s).data
        rows = np.arange(5, 1024, 97)
        ocam = O.OCamera(cam.eye, cam.target, cam.up, cam.fov_y, 1024, 1024)
        ref = O.render_image(om, O.TF_PRESETS["grayscale"], ocam, 1 / 256, rows=rows)
        assert O.metric_psnr(img[rows], ref[rows]) >= 40.0
        # explicit rays = the same rays: identical pixels
        o, d = P.camera_rays(cam)
        sel = np.arange(0, o.shape[0], 173)
        px, _ = P.raymarch_forward(src, o[sel], d[sel], s)
        np.testing.assert_array_equal(px, img.reshape(-1, 4)[sel])
        world = 3
        _, per_rank = D.shard_slots(cam.width, cam.height, world)
        gathered = torch.zeros((world, per_rank, 4), dtype=torch.float32, device="cuda")
        stream = torch.cuda.current_stream().cuda_stream
        for r in range(world):
            src.device_model.render_device(src.tf, cam, s, None, gathered[r].data_ptr(), None,
                                           stream, rank=r, world=world, compact=True)
        frame = torch.zeros((cam.height, cam.width, 4), dtype=torch.float32, device="cuda")
        D.tiles_to_frame_device(gathered.data_ptr(), cam.width, cam.height, world,
                                frame.data_ptr(), stream)
        torch.cuda.synchronize()
        assert np.array_equal(frame.cpu().numpy(), img)
    finally:
        D.set_dvr_kernel(prev)


@pytest.mark.parametrize("sampler", ["tex", "ldg"])
@pytest.mark.parametrize("name,t", [("cfg1_f16_u8", None), ("temporal_f16_u8", 6.5)])
def test_u8_checkpoint_sampled_directly(name, t, sampler):
    """a reference-written checkpoint with a u8-quantised latent grid.  The
    texture sampler reads the 8-bit codes (RGBA8 textures, dequantised in the kernel);
    the LDG sampler reads the grid dequantised on upload.  Both match the reference's
    densities and render."""
    from paper_2112_01579_b200 import device as D

    prev = D.set_grid_sampler(sampler)
    try:
        m = P.checkpoint_load(GOLDEN / f"{name}.fvsrn")
        assert m.config.grid_resolution > 0
        got = P.eval_density(m, arrays()["eval_p"][:4096], t=t)
        assert np.abs(got - arrays()[f"ckpt_{name}_density"]).max() <= DENS_TOL
        r = meta()["renders"][f"ckpt_{name}"]
        src = P.ModelSource(m, P.TF_PRESETS[r["tf"]], t=r["t"])
        img = P.render_image(src, _cam(r["camera"]), P.RenderSettings(stepsize=r["stepsize"]))
        assert P.metric_psnr(img, arrays()[f"render_ckpt_{name}"]) >= 40.0
        assert abs(src.last_eval_count - r["count"]) <= max(4, r["count"] // 1000)
    finally:
        D.set_grid_sampler(prev)


# ------------------------------------------------------------------ standalone pieces
ALL_MODELS = ["cfg1", "cfg2", "cfg3", "tiny", "temporal", "temporal_both", "color_dirf", "color_pos",
              "random_fourier", "relu_nogrid", "snake_f12"]


@pytest.mark.parametrize("name", ALL_MODELS)
def test_assemble_input_and_pieces_vs_reference(name):
    """assemble_input (model.py:248-279), grid_sample / keyframe_sample (grid.py:115-121,
    222-230) and mlp_eval + heads (nn.py:195-204, model.py:342-357) through the GPU f32
    evaluator, against the reference's own outputs."""
    a = arrays()
    m = _model(name)
    p = a["eval_p"][:257]
    d = a["eval_d"][:257] if m.config.direction_mode != "pos" else None
    t = 6.5 if m.is_temporal else None
    x = P.assemble_input(m, p, d, t)
    want = a[f"assemble_{name}"]
    assert x.shape == want.shape and x.dtype == np.float32
    np.testing.assert_allclose(x, want, rtol=0, atol=2e-6)
    F = m.config.grid_channels if m.config.grid_resolution else 0
    if F:
        z = P.keyframe_sample(m.keyframes, p, t) if m.is_temporal else P.grid_sample(m.grid, p)
        np.testing.assert_allclose(z, want[:, -F:], rtol=0, atol=2e-6)
    raw = P.mlp_eval(m.params, want)
    if m.config.head == "density" and not m.is_temporal:
        np.testing.assert_allclose(P.apply_density_head(raw), a[f"density_{name}"][:257], rtol=0, atol=2e-6)
    elif m.config.head == "color":
        np.testing.assert_allclose(P.apply_color_head(raw), a[f"color_{name}"][:257], rtol=0, atol=2e-6)


@pytest.mark.parametrize("name", ["cfg1", "color_pos", "random_fourier"])
def test_naive_vs_fused_eval(name):
    """naive_eval_model (f32, fused.py:304-312) vs fused_eval (fp16 tensor cores) vs the
    reference's fused outputs; bench_compare rows are well formed."""
    m = _model(name)
    x = arrays()[f"fused_x_{name}"]
    naive = P.naive_eval_model(m, x)
    assert np.abs(naive - arrays()[f"fused_y_{name}"]).max() <= 1e-4      # fused.py tolerance
    rows = P.bench_compare(m, [1024], runs=2)
    assert {r["evaluator"] for r in rows} == {"naive", "fused"} and all(r["samples_per_sec"] > 0 for r in rows)
    assert P.bench_csv(rows).startswith("batch,evaluator,samples_per_sec")


def test_mapped_framebuffer_tile_order_bit_identical():
    # a mapped page-locked frame uses the filler/zigzag tile order (fvsrn_capi.cu
    # render_impl), a pageable one pure LPT: the pixels must not depend on the order
    m = _model("cfg1")
    src = P.ModelSource(m, P.TF_PRESETS["warm"])
    cam = P.fibonacci_cameras(8, 1024, 1024)[5]
    s = P.RenderSettings(stepsize=1 / 128)
    fb = P.pinned_empty((1024, 1024, 4))
    a = P.render_image(src, cam, s, out=fb).data.copy()
    na = src.last_eval_count
    b = P.render_image(src, cam, s).data
    assert np.array_equal(a, b) and na == src.last_eval_count


def test_decode_into_pinned_volume_matches():
    # a page-locked output volume takes the chunked decode + overlapped copy path
    m = _model("cfg1")
    vb = P.pinned_empty((128, 128, 128))
    a = P.decode_volume(m, 128, out=vb).values.copy()
    b = P.decode_volume(m, 128).values
    assert np.array_equal(a, b)
