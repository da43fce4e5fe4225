"""Single-process multi-device entries (fvsrn_render(..., device_ids[], n_devices),
fvsrn_decode_density(..., n_devices)) through the C ABI.

The GPU box has one B200, so the replicas here share device 0: that exercises the tile
split, the per-device workers, both frame-assembly paths (mapped host frame; shared
device frame + one copy) and the slab split of the decode.  The frame and the volume
must be bit-identical to the single-device call, and the evaluated-sample count equal.
"""

import ctypes as C

import numpy as np
import pytest

import paper_2112_01579_b200 as P
from paper_2112_01579_b200 import _lib as L
from paper_2112_01579_b200 import device as D

pytestmark = pytest.mark.gpu

CFG2 = dict(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0)


@pytest.fixture(scope="module")
def model():
    return P.model_init(P.ModelConfig(**CFG2))


@pytest.mark.parametrize("n", [2, 3, 8])
@pytest.mark.parametrize("pinned", [False, True])
def test_render_multi_bit_identical(model, n, pinned):
    src = P.ModelSource(model, P.TF_PRESETS["warm"])
    cam = P.fibonacci_cameras(8, 200, 136)[3]          # ragged: 25 x 17 tiles
    st = P.RenderSettings(stepsize=1 / 256, background=(0.1, 0.2, 0.3))
    one = P.render_image(src, cam, st).data.copy()
    n1 = src.last_eval_count
    out = P.pinned_empty((136, 200, 4)) if pinned else None
    img = P.render_image(src, cam, st, out=out, devices=[0] * n)
    assert np.array_equal(img.data, one)
    assert src.last_eval_count == n1


def test_render_multi_default_devices(model):
    src = P.ModelSource(model, P.TF_PRESETS["grayscale"])
    cam = P.fibonacci_cameras(8, 256, 256)[1]
    st = P.RenderSettings(stepsize=1 / 128)
    one = P.render_image(src, cam, st).data.copy()
    prev = P.set_devices([0, 0, 0, 0])
    try:
        assert np.array_equal(P.render_image(src, cam, st).data, one)
    finally:
        P.set_devices(prev)


def test_render_multi_temporal():
    m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=8, grid_channels=16,
                                   keyframe_times=[1, 11, 21], seed=0))
    src = P.ModelSource(m, P.TF_PRESETS["grayscale"], t=6.5)
    cam = P.fibonacci_cameras(8, 96, 96)[4]
    st = P.RenderSettings(stepsize=1 / 128)
    one = P.render_image(src, cam, st).data.copy()
    assert np.array_equal(P.render_image(src, cam, st, devices=[0, 0]).data, one)


@pytest.mark.parametrize("n", [2, 5])
def test_decode_multi_bit_identical(model, n):
    one = P.decode_volume(model, 33).values.copy()
    assert np.array_equal(P.decode_volume(model, 33, devices=[0] * n).values, one)


def test_decode_multi_pinned_chunked(model):
    # >= 2^20 lattice points per slab into page-locked memory: the chunked copy pipeline
    one = P.decode_volume(model, 160).values.copy()
    out = P.pinned_empty((160, 160, 160))
    got = P.decode_volume(model, 160, out=out, devices=[0, 0])
    assert np.array_equal(got.values, one)


def test_c_abi_render_multi_direct(model):
    # the entry point as a C caller binds it: replica handles, host frame, status + count
    dm = D.device_model(model, 0)
    cam = P.fibonacci_cameras(8, 64, 48)[0]
    st = P.RenderSettings(stepsize=1 / 64)
    tfd = D.tf_desc(P.TF_PRESETS["grayscale"])
    frame = np.zeros((48, 64, 4), np.float32)
    reps = (C.c_void_p * 3)(dm.handle.value, dm.handle.value, dm.handle.value)
    cnt = C.c_uint64(0)
    rc = L.lib().fvsrn_render_multi(reps, 3, C.byref(tfd.desc), C.byref(D.camera_desc(cam)),
                                    C.byref(D.settings_desc(st)), float("nan"), L.fptr(frame),
                                    C.byref(cnt))
    assert rc == L.FVSRN_OK
    ref, n1 = dm.render(P.TF_PRESETS["grayscale"], cam, st)
    assert np.array_equal(frame, ref) and cnt.value == n1


def test_render_multi_contract_errors(model):
    other = P.model_init(P.ModelConfig(layers=3, hidden=32, grid_resolution=8, seed=1))
    cam = P.fibonacci_cameras(8, 32, 32)[0]
    st = P.RenderSettings()
    dms = [D.device_model(model, 0), D.device_model(other, 0)]
    with pytest.raises(ValueError, match="replicas differ"):
        D.render_multi(dms, P.TF_PRESETS["grayscale"], cam, st)
    with pytest.raises(ValueError):
        D.render_multi([D.device_model(model, 0)] * 2, None, cam, st)   # density head needs a TF
    reps = (C.c_void_p * 1)()
    assert L.lib().fvsrn_render_multi(reps, 0, None, None, None, 0.0, None, None) == L.FVSRN_EINVAL


@pytest.mark.parametrize("res,tf,et", [(256, "grayscale", 0.999), (97, "warm", 0.5), (180, "two_peaks", 1.0)])
def test_small_frame_pair_kernel_bit_identical(model, res, tf, et):
    """Small camera frames march two or four lanes per ray (dvr_pair_kernel); the same rays
    through raymarch_forward take the one-lane kernel.  Pixels and evaluated-sample counts must be
    identical (early termination on, loose and off)."""
    src = P.ModelSource(model, P.TF_PRESETS[tf])
    cam = P.fibonacci_cameras(8, res, res)[2]
    st = P.RenderSettings(stepsize=1 / 128, early_term_alpha=et, background=(0.05, 0.1, 0.2))
    prev = D.set_dvr_kernel("warp")     # explicit rays through the one-lane mma.sync kernel
    try:
        D.kernel_timer(True)
        img = P.render_image(src, cam, st).data.copy()
        D.kernel_timer_read()
        name = D.kernel_timer_info()
        D.kernel_timer(False)
        n_img = src.last_eval_count
        o, d = P.camera_rays(cam)
        px, _ = P.raymarch_forward(src, o, d, st)
    finally:
        D.set_dvr_kernel(prev)
    assert "dvr_pair_kernel" in name, name
    assert np.array_equal(px.reshape(res, res, 4), img)
    assert src.last_eval_count == n_img


_QUAD_SCRIPT = r"""
import json, sys
import numpy as np
import paper_2112_01579_b200 as P
from paper_2112_01579_b200 import device as D
m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=32, grid_channels=16, seed=0))
out = []
for res, tf, et in ((256, "grayscale", 0.999), (97, "warm", 0.5), (180, "two_peaks", 1.0), (8, "grayscale", 0.999)):
    src = P.ModelSource(m, P.TF_PRESETS[tf])
    cam = P.fibonacci_cameras(8, res, res)[2]
    st = P.RenderSettings(stepsize=1 / 128, early_term_alpha=et, background=(0.05, 0.1, 0.2))
    prev = D.set_dvr_kernel("warp")
    try:
        D.kernel_timer(True)
        img = P.render_image(src, cam, st).data.copy()
        D.kernel_timer_read()
        name = D.kernel_timer_info()
        D.kernel_timer(False)
        n_img = src.last_eval_count
        o, d = P.camera_rays(cam)
        px, _ = P.raymarch_forward(src, o, d, st)
    finally:
        D.set_dvr_kernel(prev)
    out.append({"res": res, "kernel": name, "equal": bool(np.array_equal(px.reshape(res, res, 4), img)),
                "count_equal": src.last_eval_count == n_img})
print(json.dumps(out))
"""


@pytest.mark.parametrize("octo_frac,quad_frac,lanes", [("100", "0", "eight lanes per ray"),
                                                        ("0", "100", "four lanes per ray"),
                                                        ("0", "0", "two lanes per ray")])
def test_small_frame_lane_group_kernels_bit_identical(octo_frac, quad_frac, lanes):
    """Eight / four / two lanes per ray (FVSRN_OCTO_FRAC / FVSRN_QUAD_FRAC admit the frame):
    pixels and counts identical to the one-lane march, ET on / loose / off, and a frame
    smaller than one warp's rays."""
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ, FVSRN_OCTO_FRAC=octo_frac, FVSRN_QUAD_FRAC=quad_frac)
    r = subprocess.run([sys.executable, "-c", _QUAD_SCRIPT], env=env, capture_output=True, text=True,
                       timeout=300, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    for case in json.loads(r.stdout.strip().splitlines()[-1]):
        assert lanes in case["kernel"], case
        assert case["equal"] and case["count_equal"], case
