"""The C++ drop-in (integration/matcache_render_b200.cpp) linked with the
reference's own sources: a reference caller's load_scene + render() now run
on the B200 path and produce the same frame as the Python mirror."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from paper_2305_07238_b200 import RenderConfig, load_scene, render, scenes

import _oracle

DROPIN = os.path.join(_oracle.ROOT, "oracle", "_ref", "libmcdropin.so")


@pytest.fixture(scope="module")
def dropin(built):
    if os.path.isdir("/root/reference"):
        subprocess.run(["make", "-C", os.path.join(_oracle.ROOT, "oracle"), "dropin"], check=True,
                       stdout=subprocess.DEVNULL)
    if not os.path.exists(DROPIN):
        pytest.skip("drop-in not built (needs /root/reference at build time)")
    L = C.CDLL(DROPIN)
    L.dropin_render.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_char_p, C.c_size_t]
    return L


def test_dropin_library_links(dropin):
    assert hasattr(dropin, "dropin_render")


@pytest.mark.gpu
@pytest.mark.parametrize("cache_on", [0, 1])
def test_dropin_render_matches_python_api(ctx, dropin, scene_dir, cache_on):
    w, h, spp = 40, 30, 3
    path = scenes.build_scene(scenes.SceneSpec("junkshop", w, h, tris_per_side=4), f"{scene_dir}/dropin")
    rad = np.zeros((h, w, 3), np.float64)
    nodes = np.zeros((h, w), np.float64)
    samples = np.zeros((h, w), np.uint32)
    st = np.zeros(8, np.uint64)
    err = C.create_string_buffer(512)
    rc = dropin.dropin_render(path.encode(), w, h, spp, cache_on, 4099, 4,
                              rad.ctypes.data_as(C.c_void_p), nodes.ctypes.data_as(C.c_void_p),
                              samples.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.c_void_p),
                              err, 512)
    assert rc == 0, err.value.decode()
    assert samples.min() == spp and st[5] == 1 and st[6] == w * h
    s = load_scene(path)
    res = render(s, RenderConfig(width=w, height=h, spp=spp, cache_enabled=bool(cache_on),
                                 n_cells=4099, n_entries=4), ctx=ctx)
    if not cache_on:
        # the drop-in flattens the reference's CompiledProgram itself: same frame, bit for bit
        np.testing.assert_array_equal(rad.view(np.uint64), res.frame.radiance.view(np.uint64))
        assert st[4] == res.stats.instructions_executed
    else:
        # concurrent inserts: which sample wins a texel is a race, so each
        # cached frame is compared with the cache-off frame: both must be the
        # same approximation of it (the cache's texels are coarse at this size)
        assert st[1] > 0 and abs(int(st[0]) - res.stats.lookups) <= res.stats.lookups * 0.01
        off = render(s, RenderConfig(width=w, height=h, spp=spp), ctx=ctx).frame.radiance
        scale = max(1e-9, off.mean())
        e_dropin = np.abs(rad - off).mean() / scale
        e_python = np.abs(res.frame.radiance - off).mean() / scale
        assert e_dropin < 0.25 and e_python < 0.25
        assert abs(e_dropin - e_python) < 0.1
