"""World-space training on the GPU vs the reference's train.py.

Goldens (tests/golden/make_golden.py, produced by the reference): one-batch L1
gradients through model_backward for four model shapes, and 4-epoch train_world loss
traces.  The host parts (targets, datasets) are compared exactly on the CPU."""

import numpy as np
import pytest

import paper_2112_01579_b200 as P
from tests.golden_util import arrays, meta

NAMES = ["cfg1", "color_pos", "relu_nogrid", "tiny"]


def _model(name):
    return P.model_init(P.ModelConfig(**meta()["models"][name]["config"]))


def _target(name):
    tfname = meta()["train"][name]["tf"]
    return P.WorldTarget(P.ScalarVolume(arrays()["train_volume"]),
                         P.TF_PRESETS[tfname] if tfname else None)


@pytest.mark.parametrize("name", NAMES)
def test_training_targets_bit_exact(name):
    # sample_volume / tf_eval restated on the host (volume.py:213-255, transfer.py:57-65)
    got = _target(name).reference(arrays()[f"train_pos_{name}"])
    np.testing.assert_array_equal(np.asarray(got, np.float32), arrays()[f"train_ref_{name}"])


def test_sample_world_dataset_same_draws():
    t = P.WorldTarget(P.ScalarVolume(arrays()["train_volume"]))
    p, v = P.sample_world_dataset(t, 1000, "uniform", seed=3)
    np.testing.assert_array_equal(p, np.random.default_rng(3).uniform(0.0, 1.0, size=(1000, 3)))
    eg = P.ErrorGrid(values=np.random.default_rng(1).uniform(size=(4, 4, 4)).astype(np.float32))
    p2, _ = P.sample_world_dataset(t, 500, eg, seed=5)
    assert p2.shape == (500, 3) and p2.min() >= 0.0 and p2.max() <= 1.0


def test_config_validation():
    with pytest.raises(ValueError):
        P.WorldTrainConfig(sample_count=10, batch_size=20)
    with pytest.raises(ValueError):
        P.WorldTrainConfig(epochs=-2)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_batch_gradients_vs_reference(name):
    from paper_2112_01579_b200.train import WorldTrainer

    m = _model(name)
    tr = WorldTrainer(m)
    loss = tr.gradients(arrays()[f"train_pos_{name}"], arrays()[f"train_ref_{name}"])
    assert abs(loss - meta()["train"][name]["loss"]) <= 1e-6 * max(1.0, abs(loss))
    got = tr.grads.cpu().numpy()
    want = arrays()[f"train_grads_{name}"]
    assert got.shape == want.shape
    off = 0
    for a in m.trainable_arrays():       # per parameter array, relative to its scale
        g, w = got[off:off + a.size], want[off:off + a.size]
        scale = float(np.abs(w).max()) or 1.0
        assert np.abs(g - w).max() <= 1e-4 * scale, (name, a.shape, np.abs(g - w).max(), scale)
        off += a.size


@pytest.mark.gpu
def test_adam_step_matches_numpy_restatement():
    from paper_2112_01579_b200.train import WorldTrainer

    m = _model("tiny")
    tr = WorldTrainer(m)
    rng = np.random.default_rng(0)
    p0 = tr.params.cpu().numpy().copy()
    mm = np.zeros_like(p0)
    vv = np.zeros_like(p0)
    for t in range(1, 4):             # adam_step, nn.py:287-298, in float32
        g = (rng.standard_normal(p0.shape) * 1e-2).astype(np.float32)
        tr.grads.copy_(__import__("torch").from_numpy(g))
        tr.adam(0.01)
        bc1, bc2 = 1.0 - 0.9 ** t, 1.0 - 0.999 ** t
        mm *= np.float32(0.9)
        mm += np.float32(1.0 - 0.9) * g
        vv *= np.float32(0.999)
        vv += np.float32(1.0 - 0.999) * g * g
        p0 -= np.float32(0.01) * (mm / np.float32(bc1)) / (np.sqrt(vv / np.float32(bc2)) + np.float32(1e-8))
        np.testing.assert_allclose(tr.params.cpu().numpy(), p0, rtol=0, atol=2e-7)
    # a non-finite gradient raises and leaves every parameter untouched
    before = tr.params.cpu().numpy().copy()
    bad = np.zeros_like(p0)
    bad[5] = np.nan
    tr.grads.copy_(__import__("torch").from_numpy(bad))
    with pytest.raises(FloatingPointError):
        tr.adam(0.01)
    np.testing.assert_array_equal(tr.params.cpu().numpy(), before)
    assert tr.t == 3


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tiny", "cfg1"])
def test_train_world_trace_vs_reference(name):
    m = _model(name)
    vol = P.ScalarVolume(arrays()["train_volume"])
    cfg = P.WorldTrainConfig(sample_count=4096, batch_size=1024, epochs=4, lr=0.01, seed=0)
    before = P.eval_density(m, arrays()["train_pos_cfg1"][:64])   # device copy of the init
    _, trace = P.train_world(m, P.WorldTarget(vol), cfg)
    want = arrays()[f"train_trace_{name}"]
    # epoch 0 is the same data, order and initial parameters: tight; later epochs follow
    # Adam trajectories that start from f32-rounding-level gradient differences
    assert abs(trace[0] - want[0]) <= 1e-4 * want[0]
    np.testing.assert_allclose(trace, want, rtol=3e-2)
    assert trace[-1] < trace[0]
    final = np.concatenate([a.reshape(-1) for a in m.trainable_arrays()])
    ref_final = arrays()[f"train_final_{name}"]
    assert np.abs(final - ref_final).max() <= 0.05 * np.abs(ref_final).max()
    # the trained parameters reached the model and its render copy was refreshed
    after = P.eval_density(m, arrays()["train_pos_cfg1"][:64])
    assert not np.allclose(before, after)


# ------------------------------------------------------------------ screen space
@pytest.mark.gpu
def test_screen_forward_states_and_backward_vs_reference():
    from paper_2112_01579_b200.train import ScreenTrainer

    a = arrays()
    m = _model("color_pos")
    st = P.RenderSettings(stepsize=meta()["screen"]["stepsize"])
    tr = ScreenTrainer(m)
    px, state = tr.forward(a["screen_o"], a["screen_d"], st)
    # raymarch_forward(want_states=True): f32 model, f64 compositing, no ET
    np.testing.assert_allclose(px.cpu().numpy(), a["screen_px"], rtol=0, atol=2e-6)
    np.testing.assert_allclose(state[2].cpu().numpy(), a["screen_state_c"], rtol=0, atol=2e-6)
    np.testing.assert_allclose(state[3].cpu().numpy(), a["screen_state_a"], rtol=0, atol=2e-6)
    tr.backward(state, st, a["screen_adj"])
    got, want = tr.grads.cpu().numpy(), a["screen_grads"]
    off = 0
    for arr in m.trainable_arrays():
        g, w = got[off:off + arr.size], want[off:off + arr.size]
        scale = float(np.abs(w).max()) or 1.0
        assert np.abs(g - w).max() <= 1e-4 * scale, (arr.shape, np.abs(g - w).max(), scale)
        off += arr.size
    # the functional API returns the reference's GradientBuffer shape
    gb = P.raymarch_backward(m, a["screen_o"], a["screen_d"], st, a["screen_adj"])
    assert [g.shape for g in gb.arrays()] == [x.shape for x in m.trainable_arrays()]


@pytest.mark.gpu
def test_train_screen_trace_vs_reference():
    m = _model("color_pos")
    vol = P.ScalarVolume(arrays()["train_volume"])
    cfg = P.ScreenTrainConfig(views=2, resolution=12, stepsize=0.05, epochs=3,
                              reference_stepsize_voxels=0.5)
    _, trace = P.train_screen(m, vol, P.TF_PRESETS["warm"], cfg)
    want = arrays()["screen_trace"]
    assert abs(trace[0] - want[0]) <= 1e-4 * want[0]
    np.testing.assert_allclose(trace, want, rtol=3e-2)
    assert trace[-1] < trace[0]
    with pytest.raises(ValueError):
        P.train_screen(_model("cfg1"), vol, P.TF_PRESETS["warm"], cfg)


# ------------------------------------------------------------------ temporal
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["temporal", "temporal_both"])
def test_temporal_batch_gradients_vs_reference(name):
    """Per-sample timesteps (between and exactly on keyframes): time features, keyframe
    brackets and the two-grid latent scatter (model.py:190-245, 318-333)."""
    from paper_2112_01579_b200.train import WorldTrainer

    a = arrays()
    m = _model(name)
    tr = WorldTrainer(m)
    loss = tr.gradients(a[f"ttrain_pos_{name}"], a[f"ttrain_ref_{name}"], a[f"ttrain_t_{name}"])
    assert abs(loss - meta()["train"][f"t_{name}"]["loss"]) <= 1e-6 * max(1.0, abs(loss))
    got, want = tr.grads.cpu().numpy(), a[f"ttrain_grads_{name}"]
    off = 0
    for arr in m.trainable_arrays():
        g, w = got[off:off + arr.size], want[off:off + arr.size]
        scale = float(np.abs(w).max()) or 1.0
        assert np.abs(g - w).max() <= 1e-4 * scale, (name, arr.shape, np.abs(g - w).max(), scale)
        off += arr.size
    with pytest.raises(ValueError):
        tr.gradients(a[f"ttrain_pos_{name}"], a[f"ttrain_ref_{name}"])      # times required


@pytest.mark.gpu
def test_train_temporal_trace_vs_reference():
    a = arrays()
    m = _model("temporal")
    cfg = P.TemporalTrainConfig(keyframe_times=[1, 11, 21], train_times=[1, 6, 11, 16, 21],
                                world=P.WorldTrainConfig(sample_count=4096, batch_size=1024, epochs=3,
                                                         lr=0.01, seed=0))
    _, trace = P.train_temporal(m, lambda t: P.ScalarVolume(a[f"ttrain_vol_{t}"]), cfg)
    want = a["ttrain_trace"]
    assert abs(trace[0] - want[0]) <= 1e-4 * want[0]
    np.testing.assert_allclose(trace, want, rtol=3e-2)
    with pytest.raises(ValueError):
        P.train_temporal(_model("cfg1"), lambda t: None, cfg)


def test_temporal_config_validation():
    with pytest.raises(ValueError):
        P.TemporalTrainConfig(train_times=[])
    with pytest.raises(ValueError):
        P.TemporalTrainConfig(keyframe_times=[5, 10], train_times=[1, 10])


@pytest.mark.gpu
def test_evaluate_views_vs_reference():
    # train.py:317-341: GPU renders of model (ModelSource) and ground truth (VolumeSource)
    g = meta()["evaluate_views"]
    m = _model(g["model"])
    rows = P.evaluate_views(m, P.ScalarVolume(arrays()["train_volume"]), P.TF_PRESETS[g["tf"]],
                            n_views=g["n_views"], resolution=g["resolution"])
    assert [r["view"] for r in rows] == [r["view"] for r in g["rows"]]
    for got, ref in zip(rows, g["rows"]):
        # fp16 network in the kernel vs f32 reference evaluation: metric-level tolerance
        assert got["psnr"] == pytest.approx(ref["psnr"], abs=0.05)
        assert got["ssim"] == pytest.approx(ref["ssim"], abs=5e-3)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES + ["t_temporal", "t_temporal_both"])
def test_model_forward_backward_vs_reference(name):
    # model_forward / model_backward (model.py:290-335) with the reference's L1 adjoint
    # through the head backward (train.py:158-162, model.py:346-365)
    a = arrays()
    if name.startswith("t_"):
        key = name[2:]
        m = P.model_init(P.ModelConfig(**meta()["models"][key]["config"]))
        pb, tb, ref = a[f"ttrain_pos_{key}"], a[f"ttrain_t_{key}"], a[f"ttrain_ref_{key}"]
        want = a[f"ttrain_grads_{key}"]
    else:
        m, pb, tb, ref = _model(name), a[f"train_pos_{name}"], None, a[f"train_ref_{name}"]
        want = a[f"train_grads_{name}"]
    raw, ctx = P.model_forward(m, pb, t=tb)
    assert ctx.inputs.shape == (len(pb), m.config.input_width)
    dens = m.config.head == "density"
    pred = P.apply_density_head(raw) if dens else P.apply_color_head(raw)
    diff = pred - np.asarray(ref).reshape(pred.shape)
    adj = (np.sign(diff) / diff.size).astype(np.float32)
    raw_bar = P.density_head_backward(raw, adj) if dens else P.color_head_backward(raw, adj)
    g = P.model_backward(m, ctx, raw_bar)
    got = np.concatenate([x.reshape(-1) for x in g.arrays()])
    assert got.shape == want.shape
    off = 0
    for arr in m.trainable_arrays():
        gg, ww = got[off:off + arr.size], want[off:off + arr.size]
        scale = float(np.abs(ww).max()) or 1.0
        assert np.abs(gg - ww).max() <= 1e-4 * scale, (name, arr.shape, np.abs(gg - ww).max(), scale)
        off += arr.size
    # accumulation into an existing buffer doubles it
    g2 = P.model_backward(m, ctx, raw_bar, grads=P.model_backward(m, ctx, raw_bar))
    np.testing.assert_allclose(np.concatenate([x.reshape(-1) for x in g2.arrays()]), 2 * got,
                               rtol=1e-5, atol=1e-9)


def test_head_backward_host_utilities():
    raw = np.random.default_rng(0).normal(size=(7, 4)).astype(np.float32)
    yb = np.random.default_rng(1).normal(size=(7, 4)).astype(np.float32)
    s = 1 / (1 + np.exp(-raw))
    d = P.density_head_backward(raw, yb[:, 0])
    np.testing.assert_allclose(d[:, 0], yb[:, 0] * s[:, 0] * (1 - s[:, 0]), rtol=1e-6)
    assert np.all(d[:, 1:] == 0)
    c = P.color_head_backward(raw, yb)
    np.testing.assert_allclose(c[:, :3], yb[:, :3] * s[:, :3] * (1 - s[:, :3]), rtol=1e-6)
    np.testing.assert_allclose(c[:, 3], yb[:, 3] * s[:, 3], rtol=1e-6)


@pytest.mark.gpu
def test_adam_step_host_api_matches_reference_semantics():
    # adam_step / AdamState (nn.py:258-298) on host arrays through the CUDA Adam kernel
    rng = np.random.default_rng(4)
    arrays = [rng.normal(size=(3, 5)).astype(np.float32), rng.normal(size=(5,)).astype(np.float32)]
    ref = [a.copy() for a in arrays]
    st = P.AdamState.for_arrays(arrays)
    m = [np.zeros_like(a) for a in arrays]
    v = [np.zeros_like(a) for a in arrays]
    for t in range(1, 4):
        grads = [(rng.normal(size=a.shape) * 1e-2).astype(np.float32) for a in arrays]
        P.adam_step(arrays, grads, st, 0.01)
        bc1, bc2 = 1 - 0.9 ** t, 1 - 0.999 ** t
        for p, g, mm, vv in zip(ref, grads, m, v):
            mm *= np.float32(0.9); mm += np.float32(0.1) * g
            vv *= np.float32(0.999); vv += np.float32(0.001) * g * g
            p -= np.float32(0.01) * (mm / np.float32(bc1)) / (np.sqrt(vv / np.float32(bc2)) + np.float32(1e-8))
        for a, r in zip(arrays, ref):
            np.testing.assert_allclose(a, r, rtol=0, atol=2e-7)
    assert st.t == 3
    before = [a.copy() for a in arrays]
    bad = [np.zeros_like(a) for a in arrays]
    bad[1][2] = np.inf
    with pytest.raises(FloatingPointError):
        P.adam_step(arrays, bad, st, 0.01)
    assert st.t == 3 and all(np.array_equal(a, b) for a, b in zip(arrays, before))
    with pytest.raises(ValueError):
        P.adam_step(arrays, bad[:1], st, 0.01)


@pytest.mark.gpu
def test_grid_sample_backward_vs_reference():
    # grid.py:123-137 scatter-add, incl. clamped positions outside the cube: the
    # deterministic gather sums every vertex in the reference's sequential order and
    # arithmetic (f64 weights x f32 adjoint into the f32 gradient) -> bit-identical
    a = arrays()
    m = _model("cfg1")
    g = np.zeros_like(m.grid.values)
    P.grid_sample_backward(m.grid, a["gsb_pos"], a["gsb_zbar"], g)
    want = a["gsb_grad"]
    assert np.array_equal(g, want), np.abs(g - want).max()
    # accumulates in place
    P.grid_sample_backward(m.grid, a["gsb_pos"], a["gsb_zbar"], g)
    assert np.abs(g - 2 * want).max() <= 2e-5 * float(np.abs(want).max())
    with pytest.raises(ValueError):
        P.grid_sample_backward(m.grid, a["gsb_pos"], a["gsb_zbar"][:, :3], g)
    with pytest.raises(ValueError):
        P.grid_sample_backward(m.grid, a["gsb_pos"], a["gsb_zbar"], g[:2])


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["snake4", "relu1", "snake2", "softplus3"])
def test_mlp_forward_backward_vs_reference(tag):
    # nn.py:179-193, 234-256 on the GPU (f32 FMA order vs numpy matmul: tolerance)
    a = arrays()
    lc, hid, din, dout, act = meta()["mlp"][tag]
    prm = P.init_params(lc, hid, din, dout, seed=3, activation=act)
    off = 0
    bias = a[f"mlp_{tag}_biases"]
    for b in prm.biases:
        b[...] = bias[off:off + b.size]
        off += b.size
    y, cache = P.mlp_forward(prm, a[f"mlp_{tag}_x"])
    want = a[f"mlp_{tag}_y"]
    assert np.abs(y - want).max() <= 2e-5 * max(1.0, float(np.abs(want).max()))
    assert len(cache.inputs) == lc and len(cache.preacts) == lc
    np.testing.assert_allclose(cache.preacts[0], a[f"mlp_{tag}_pre0"], rtol=0, atol=2e-5)
    x_bar, g = P.mlp_backward(prm, cache, a[f"mlp_{tag}_ybar"])
    wx = a[f"mlp_{tag}_xbar"]
    assert np.abs(x_bar - wx).max() <= 1e-4 * max(1.0, float(np.abs(wx).max()))
    got = np.concatenate([x.reshape(-1) for x in g.arrays()])
    wg = a[f"mlp_{tag}_grads"]
    assert got.shape == wg.shape and g.grids == []
    assert np.abs(got - wg).max() <= 1e-4 * float(np.abs(wg).max())
    with pytest.raises(ValueError):
        P.mlp_backward(prm, cache, a[f"mlp_{tag}_ybar"][:, :1].repeat(dout + 1, axis=1))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg1", "tiny", "temporal"])
def test_gradients_bit_identical_across_runs(name):
    """No atomics on any gradient: the latent-grid scatter is a fixed-order gather, the
    weight / bias reductions are fixed chunks summed in order, the loss a fixed-order sum."""
    from paper_2112_01579_b200.train import WorldTrainer

    m = _model(name)
    pos = np.random.default_rng(4).uniform(0.0, 1.0, size=(3000, 3))
    ref = np.random.default_rng(5).uniform(0.0, 1.0, size=(3000, 1)).astype(np.float32)
    times = (np.random.default_rng(6).uniform(1.0, 21.0, size=3000) if m.is_temporal else None)
    runs = []
    for _ in range(3):
        tr = WorldTrainer(m)
        loss = tr.gradients(pos, ref, times)
        runs.append((loss, tr.grads.cpu().numpy().copy()))
    for loss, g in runs[1:]:
        assert loss == runs[0][0]
        assert np.array_equal(g, runs[0][1])


@pytest.mark.gpu
def test_train_world_bit_identical_across_runs():
    vol = P.ScalarVolume(values=arrays()["train_volume"])
    out = []
    for _ in range(2):
        m = _model("cfg1")
        _, trace = P.train_world(m, P.WorldTarget(vol), P.WorldTrainConfig(
            sample_count=4096, batch_size=1024, epochs=3, lr=0.01, seed=0))
        out.append((trace, np.concatenate([a.reshape(-1) for a in m.trainable_arrays()])))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])


@pytest.mark.gpu
def test_screen_gradients_bit_identical_across_runs():
    a = arrays()
    st = P.RenderSettings(stepsize=meta()["screen"]["stepsize"])
    gs = []
    for _ in range(2):
        m = _model("color_pos")
        g = P.raymarch_backward(m, a["screen_o"], a["screen_d"], st, a["screen_adj"])
        gs.append(np.concatenate([x.reshape(-1) for x in g.arrays()]))
    assert np.array_equal(gs[0], gs[1])
