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


@pytest.mark.gpu
def test_dropin_two_scenes_same_stack_frame(ctx, dropin, scene_dir):
    """the drop-in keys its device upload on the scene's
    content, not its address. Three different scenes loaded one after the
    other into the same stack slot (oracle/dropin_harness.cpp
    dropin_render_scenes), plus the first again: each frame equals the
    Python API's render of that scene, bit for bit (cache off)."""
    w, h, spp = 32, 24, 2
    paths = [scenes.build_scene(scenes.SceneSpec(k, w, h, tris_per_side=4), f"{scene_dir}/two_{k}")
             for k in ("junkshop", "cornell", "italianflat")]
    paths.append(paths[0])
    rad = np.zeros((len(paths), h, w, 3), np.float64)
    err = C.create_string_buffer(512)
    arr = (C.c_char_p * len(paths))(*[p.encode() for p in paths])
    dropin.dropin_render_scenes.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                            C.c_char_p, C.c_size_t]
    rc = dropin.dropin_render_scenes(C.cast(arr, C.c_void_p), len(paths), w, h, spp,
                                     rad.ctypes.data_as(C.c_void_p), err, 512)
    assert rc == 0, err.value.decode()
    for i, p in enumerate(paths):
        want = render(load_scene(p), RenderConfig(width=w, height=h, spp=spp), ctx=ctx).frame.radiance
        np.testing.assert_array_equal(rad[i].view(np.uint64), want.view(np.uint64), err_msg=p)
    assert not np.array_equal(rad[0], rad[1])


@pytest.mark.gpu
def test_dropin_external_cache_follows_the_device(ctx, dropin, scene_dir, tmp_path):
    """an external MaterialCache passed to the drop-in's
    render() is the truth. Each call seeds the device table from its slot
    words and replays the won inserts back through update(), so after every
    render the host table's occupied_slots() and inserts_won counter equal
    the inserts the render reports (accumulating over progressive renders),
    its dump passes the reference's audit, and a progressive second render
    hits more. A fresh cache allocated where a deleted one lived, and a
    cache of another shape, start empty (no stale device table)."""
    w, h, spp, nc, ne, n = 40, 30, 2, 4099, 4, 2
    path = scenes.build_scene(scenes.SceneSpec("junkshop", w, h, tris_per_side=4), f"{scene_dir}/ext")
    out = np.zeros(6 * (n + 2) + 2, np.uint64)
    err = C.create_string_buffer(512)
    dropin.dropin_render_external.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint32,
                                              C.c_int, C.c_char_p, C.c_void_p, C.c_char_p, C.c_size_t]
    rc = dropin.dropin_render_external(path.encode(), w, h, spp, nc, ne, n, str(tmp_path / "d.bin").encode(),
                                       out.ctypes.data_as(C.c_void_p), err, 512)
    assert rc == 0, err.value.decode()
    rows = out[:6 * (n + 2)].reshape(-1, 6).astype(np.int64)
    won_total = 0
    for i, (look, hits, won, occ, cwon, clean) in enumerate(rows):
        won_total = won_total + won if i < n else won
        assert look > 0 and clean == 1, (i, rows)
        assert occ == won_total and cwon == won_total, (i, rows)
    assert rows[1, 1] > rows[0, 1]          # the progressive render hits what the first stored
    assert rows[n, 2] > 0 and rows[n, 3] == rows[n, 2]     # fresh cache (same shape): starts empty
    assert rows[n + 1, 3] == rows[n + 1, 2] > 0            # another shape


_MULTI_SCRIPT = r"""
import ctypes as C, sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render
L = C.CDLL(sys.argv[2])
L.dropin_render_scenes.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_char_p, C.c_size_t]
w, h, spp = 40, 30, 3
rad = np.zeros((1, h, w, 3))
err = C.create_string_buffer(512)
arr = (C.c_char_p * 1)(sys.argv[3].encode())
assert L.dropin_render_scenes(C.cast(arr, C.c_void_p), 1, w, h, spp, rad.ctypes.data_as(C.c_void_p), err, 512) == 0, err.value
want = render(load_scene(sys.argv[3]), RenderConfig(width=w, height=h, spp=spp), ctx=Context(0)).frame.radiance
assert np.array_equal(rad[0].view(np.uint64), want.view(np.uint64))
print("multi ok")
"""


@pytest.mark.gpu
def test_dropin_render_uses_every_listed_device(ctx, dropin, scene_dir):
    """The drop-in's render() without an external cache runs on a context
    over every GPU (MATCACHE_B200_DEVICES, default all visible): tiles dealt
    to the devices, frames gathered. On this one-GPU box device 0 is listed
    twice (device-copy gather instead of NCCL); the frame equals the
    one-device render bit for bit. Own process: the drop-in's contexts are
    created once per process."""
    import sys
    path = scenes.build_scene(scenes.SceneSpec("junkshop", 40, 30, tris_per_side=4), f"{scene_dir}/dropin_multi")
    env = dict(os.environ, MATCACHE_B200_DEVICES="0,0")
    r = subprocess.run([sys.executable, "-c", _MULTI_SCRIPT, _oracle.ROOT, DROPIN, path], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "multi ok" in r.stdout, r.stderr[-2000:]
