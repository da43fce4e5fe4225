"""The HTTP service on the GPU path, mirroring the reference's
tests/test_service.py: request validation and /model/info run on the CPU; every
test that renders is marked gpu."""

import io

import numpy as np
import pytest
from fastapi.testclient import TestClient

import paper_2112_01579_b200 as P
from paper_2112_01579_b200.service import SessionState, create_app


def make_client(model=None, **state_kw):
    if model is None:
        model = P.model_init(P.ModelConfig(seed=3))
    state = SessionState(model=model, default_tf=P.TF_PRESETS["grayscale"],
                         native_resolution=32, **state_kw)
    return TestClient(create_app(state))


def default_request(**overrides):
    body = {"camera": {"eye": [0.5, 0.5, 2.5], "target": [0.5, 0.5, 0.5],
                       "up": [0, 1, 0], "fov_y_deg": 45.0},
            "width": 32, "height": 32, "stepsize_voxels": 1.0}
    body.update(overrides)
    return body


def temporal_model():
    return P.model_init(P.ModelConfig(layers=2, hidden=16, fourier_m=6, grid_resolution=4,
                                      grid_channels=4, keyframe_times=[1, 11], time_mode="direct"))


# ------------------------------------------------------------------ CPU (no render)
def test_model_info_reports_default_memory():
    info = make_client().get("/model/info").json()
    assert info["memory"]["grid"] == 2097152
    assert info["temporal_span"] is None
    assert "two_peaks" in info["tf_presets"]


def test_model_info_idempotent_and_temporal_span():
    c = make_client()
    assert c.get("/model/info").json() == c.get("/model/info").json()
    assert make_client(temporal_model()).get("/model/info").json()["temporal_span"] == [1, 11]


def test_503_before_load():
    c = TestClient(create_app(None))
    assert c.get("/model/info").status_code == 503
    assert c.post("/render", json=default_request()).status_code == 503


def test_request_validation_422_409():
    c = make_client()
    assert c.post("/render", json=default_request(width=0)).status_code == 422
    body = default_request()
    body["camera"]["target"] = body["camera"]["eye"]
    assert c.post("/render", json=body).status_code == 422
    assert c.post("/render", json=default_request(t=3.0)).status_code == 422
    bad = [{"x": 0.5, "rgb": [0, 0, 0], "sigma": 0.0}, {"x": 1.0, "rgb": [1, 1, 1], "sigma": 5.0}]
    assert c.post("/render", json=default_request(tf=bad)).status_code == 422
    tc = make_client(temporal_model())
    assert tc.post("/render", json=default_request()).status_code == 422
    assert tc.post("/render", json=default_request(t=99.0)).status_code == 422
    color = P.model_init(P.ModelConfig(head="color", layers=2, hidden=16, fourier_m=6,
                                       grid_resolution=4, grid_channels=4))
    tf = [{"x": 0.0, "rgb": [0, 0, 0], "sigma": 0.0}, {"x": 1.0, "rgb": [1, 1, 1], "sigma": 5.0}]
    assert make_client(color).post("/render", json=default_request(tf=tf)).status_code == 409


# ------------------------------------------------------------------ GPU (renders)
@pytest.mark.gpu
def test_render_png_pixels_equal_quantised_render_image():
    from PIL import Image as PILImage

    model = P.model_init(P.ModelConfig(seed=3))
    r = make_client(model).post("/render", json=default_request(width=48, height=40))
    assert r.status_code == 200
    assert r.headers["content-type"] == "image/png"
    assert r.content[:8] == b"\x89PNG\r\n\x1a\n"
    assert float(r.headers["X-Render-Millis"]) > 0
    px = np.asarray(PILImage.open(io.BytesIO(r.content)).convert("RGBA"))
    cam = P.Camera(eye=np.array([0.5, 0.5, 2.5]), target=np.array([0.5, 0.5, 0.5]),
                   up=np.array([0.0, 1.0, 0.0]), fov_y=np.deg2rad(45.0), width=48, height=40)
    img = P.render_image(P.ModelSource(model, P.TF_PRESETS["grayscale"]), cam,
                         P.RenderSettings.for_voxels(32, 1.0))
    want = np.floor(np.clip(img.data, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)   # imaging.py:74-80
    np.testing.assert_array_equal(px, want)
    # the device quantisation itself, into a mapped page-locked buffer
    fb = P.pinned_empty((40, 48, 4), np.uint8)
    got = P.render_image_rgba8(P.ModelSource(model, P.TF_PRESETS["grayscale"]), cam,
                               P.RenderSettings.for_voxels(32, 1.0), out=fb)
    np.testing.assert_array_equal(got, want)


@pytest.mark.gpu
def test_render_deterministic_tf_swap_temporal_and_concurrent():
    c = make_client()
    a = c.post("/render", json=default_request()).content
    assert a == c.post("/render", json=default_request()).content
    warm = [{"x": 0.0, "rgb": [0, 0, 0], "sigma": 0.0}, {"x": 0.5, "rgb": [1, 0.2, 0.1], "sigma": 8.0},
            {"x": 1.0, "rgb": [1, 1, 1], "sigma": 2.0}]
    assert c.post("/render", json=default_request(tf=warm)).content != a
    assert make_client(temporal_model()).post("/render", json=default_request(t=6.0)).status_code == 200
    model = P.model_init(P.ModelConfig(seed=5))
    assert (make_client(model).post("/render", json=default_request()).content ==
            make_client(model).post("/render", json=default_request()).content)
    # concurrent requests on the server's thread pool match serial execution
    from concurrent.futures import ThreadPoolExecutor

    c2 = make_client(model)
    bodies = [default_request(width=32 + 8 * (i % 3)) for i in range(12)]
    serial = [c2.post("/render", json=b).content for b in bodies]
    with ThreadPoolExecutor(4) as ex:
        par = list(ex.map(lambda b: c2.post("/render", json=b).content, bodies))
    assert par == serial
