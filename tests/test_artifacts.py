"""Experiment artefacts: image I/O byte-identical to the
reference's image.cpp, the x5 difference image and the viridis heatmap
(SPEC.md:463-476 examples, acceptance criterion 10)."""
import ctypes as C
import json

import numpy as np
import pytest

from paper_2305_07238_b200 import (FrameBuffers, ImageIoError, RenderStats, artifacts,
                                   image_error, parse_stats_json, stats_to_json)


def _img(seed, h=7, w=11, lo=-0.3, hi=1.4):
    r = np.random.default_rng(seed)
    a = r.uniform(lo, hi, (h, w, 3)).astype(np.float32)
    a[0, 0] = [0.0, 1.0, 0.5]
    a[0, 1] = [np.float32(127.5 / 255), np.float32(0.5 / 255), np.float32(254.5 / 255)]
    return a


@pytest.mark.parametrize("gamma", [False, True])
def test_ppm_bytes_match_reference(ref, tmp_path, gamma):
    for seed in range(4):
        a = _img(seed)
        ours, theirs = tmp_path / "ours.ppm", tmp_path / "ref.ppm"
        artifacts.write_ppm(str(ours), a, gamma)
        assert ref.L.ref_write_ppm(str(theirs).encode(), a.shape[1], a.shape[0],
                                   a.ctypes.data_as(C.c_void_p), int(gamma)) == 0
        assert ours.read_bytes() == theirs.read_bytes()
        back = artifacts.read_ppm(str(theirs))
        assert back.shape == a.shape and back.dtype == np.float32


def test_pfm_bytes_and_round_trip_match_reference(ref, tmp_path):
    a = _img(9, 5, 6, -1e3, 1e3)
    a[1, 1] = [np.inf, -0.0, 1e-40]
    ours, theirs = tmp_path / "ours.pfm", tmp_path / "ref.pfm"
    artifacts.write_pfm(str(ours), a)
    assert ref.L.ref_write_pfm(str(theirs).encode(), a.shape[1], a.shape[0],
                               a.ctypes.data_as(C.c_void_p)) == 0
    assert ours.read_bytes() == theirs.read_bytes()
    back = artifacts.read_pfm(str(ours))
    np.testing.assert_array_equal(back.view(np.uint32), a.view(np.uint32))
    w, h = C.c_int(), C.c_int()
    out = np.zeros_like(a)
    assert ref.L.ref_read_pfm(str(ours).encode(), C.byref(w), C.byref(h), out.ctypes.data_as(C.c_void_p)) == 0
    np.testing.assert_array_equal(out.view(np.uint32), a.view(np.uint32))


def test_image_io_errors(tmp_path):
    bad = tmp_path / "bad.pfm"
    bad.write_bytes(b"P6\n2 2\n255\n" + bytes(12))
    with pytest.raises(ImageIoError, match="not a color PFM"):
        artifacts.read_pfm(str(bad))
    short = tmp_path / "short.pfm"
    short.write_bytes(b"PF\n4 4\n-1.0\n" + bytes(10))
    with pytest.raises(ImageIoError, match="short read"):
        artifacts.read_pfm(str(short))
    big = tmp_path / "big.pfm"
    big.write_bytes(b"PF\n2 2\n1.0\n" + bytes(48))
    with pytest.raises(ImageIoError, match="big-endian"):
        artifacts.read_pfm(str(big))
    with pytest.raises(ImageIoError, match="dimensions"):
        artifacts.write_ppm(str(tmp_path / "z.ppm"), np.zeros((0, 3, 3), np.float32), False)
    with pytest.raises(ImageIoError, match="cannot open"):
        artifacts.read_ppm(str(tmp_path / "missing.ppm"))


def test_viridis_endpoints_and_midpoint():
    t = artifacts.VIRIDIS
    assert t.shape == (256, 3)
    np.testing.assert_array_equal(artifacts.viridis(0.0), t[0])
    np.testing.assert_array_equal(artifacts.viridis(1.0), t[255])
    np.testing.assert_array_equal(artifacts.viridis(-3.0), t[0])
    np.testing.assert_array_equal(artifacts.viridis(7.0), t[255])
    np.testing.assert_allclose(artifacts.viridis(0.5), 0.5 * (t[127] + t[128]), rtol=0, atol=1e-7)
    # canonical endpoints: dark purple (68, 1, 84) and yellow (253, 231, 37)
    assert (np.rint(t[0] * 255) == [68, 1, 84]).all()
    assert (np.rint(t[255] * 255) == [253, 231, 37]).all()


def test_heatmap_domain_0_to_20(tmp_path):
    v = np.array([[0.0, 10.0, 20.0, 35.0]], np.float32)
    img = artifacts.heatmap(v)
    np.testing.assert_array_equal(img[0, 0], artifacts.viridis(0.0))
    np.testing.assert_array_equal(img[0, 1], artifacts.viridis(0.5))
    np.testing.assert_array_equal(img[0, 2], artifacts.viridis(1.0))
    np.testing.assert_array_equal(img[0, 3], artifacts.viridis(1.0))


def test_heatmap_from_stats_json(tmp_path):
    fb = FrameBuffers(3, 2)
    fb.samples[:] = 2
    fb.nodes_found[:] = np.array([[0, 20, 40], [10, 2, 80]], np.float64)
    st = RenderStats(0.5, 10, 5, 0.5, 3, 0, 4, 100, [1, 2])
    text = stats_to_json(st, fb)
    out = tmp_path / "heat.ppm"
    img = artifacts.write_heatmap(text, str(out))
    np.testing.assert_array_equal(img, artifacts.heatmap(parse_stats_json(text).per_pixel_nodes_found))
    back = artifacts.read_ppm(str(out))
    assert back.shape == (2, 3, 3)
    # all-zero stats -> every pixel viridis(0)
    fb.nodes_found[:] = 0
    img0 = artifacts.write_heatmap(stats_to_json(st, fb), str(out))
    assert (img0 == artifacts.viridis(0.0)).all()
    doc = json.loads(text)
    del doc["per_pixel_nodes_found"]
    with pytest.raises(ValueError):
        artifacts.write_heatmap(json.dumps(doc), str(out))


def test_diff_image_is_clamped_times_five(tmp_path):
    a = _img(3, lo=0.0, hi=1.0)
    d = artifacts.write_diff(a, a, str(tmp_path / "d0.ppm"))
    assert d.mean_abs == 0.0 and d.max_abs == 0.0 and (d.diff == 0).all()
    assert (artifacts.read_ppm(str(tmp_path / "d0.ppm")) == 0).all()
    b = (a + np.float32(0.1)).astype(np.float32)
    d = artifacts.write_diff(a, b, str(tmp_path / "d1.ppm"))
    np.testing.assert_allclose(d.diff, 0.5, atol=1e-5)
    # 5 * (0.1 +- rounding) = 0.5 gray: byte 127 or 128 (lround(0.5 * 255) = 128)
    px = np.frombuffer((tmp_path / "d1.ppm").read_bytes()[-a.size:], np.uint8)
    assert set(np.unique(px)) <= {127, 128}
    q = np.zeros_like(a)
    artifacts.write_diff(q, q + np.float32(0.125), str(tmp_path / "d2.ppm"), scale=4.0)
    assert (np.frombuffer((tmp_path / "d2.ppm").read_bytes()[-a.size:], np.uint8) == 128).all()
    np.testing.assert_array_equal(d.diff, image_error(a, b).diff)
    big = a + np.float32(0.9)
    assert (image_error(a, big).diff == 1.0).all()
