"""Pins the C oracle (oracle/mc_oracle.c) to the reference's own compiled code
(oracle/_ref/libmcref.so): every stage of the path, bit for bit."""
import os

import ctypes

import numpy as np
import pytest

from paper_2305_07238_b200 import descriptors, load_scene, scenes

import _oracle
from _oracle import RenderParamsC


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view({4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


def test_descriptor_pipeline_bit_exact(oracle, ref):
    r = np.random.default_rng(11)
    n = 200_000
    d = descriptors(r.integers(0, 1 << 32, n, dtype=np.uint64), r.integers(0, 1 << 32, n, dtype=np.uint64),
                    r.integers(0, 256, n), r.integers(0, 1 << 32, n, dtype=np.uint64),
                    r.integers(0, 1 << 32, n, dtype=np.uint64))
    for a, b in zip(oracle.hash(d), ref.hash(d)):
        np.testing.assert_array_equal(a, b)
    rgb = (r.standard_normal((n, 3)) * np.exp(r.uniform(-100, 100, (n, 1)))).astype(np.float32)
    rgb[::37] = np.inf
    rgb[::41, 2] = np.nan
    rgb[::43] = np.float32(3.4e38)
    rgb[::47] = np.float32(1e-45)
    np.testing.assert_array_equal(oracle.encode(rgb), ref.encode(rgb))
    words = r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    np.testing.assert_array_equal(bits(oracle.decode(words)), bits(ref.decode(words)))
    uv = r.uniform(-1e4, 1e4, (n, 2)).astype(np.float32)
    uv[::13] = np.float32(np.nan)
    g1 = (np.exp(r.uniform(-104, 88, (n, 2))) * r.choice([-1, 1], (n, 2))).astype(np.float32)
    g2 = (np.exp(r.uniform(-104, 88, (n, 2))) * r.choice([-1, 1], (n, 2))).astype(np.float32)
    g1[::17] = 0
    g2[::19] = np.float32(np.inf)
    for off in (-30, -1, 0, 3, 30):
        m1, t1 = oracle.mip_texel(uv, g1, g2, off)
        m2, t2 = ref.mip_texel(uv, g1, g2, off)
        np.testing.assert_array_equal(m1, m2)
        np.testing.assert_array_equal(t1, t2)


def test_eq1_exact_floor_semantics(oracle, ref):
    """SPEC.md:506 #4: Eq. 1 over a grid of gradient pairs including exact
    powers of two and their neighbours (where floor(-log2) flips)."""
    e = np.arange(-30, 4, dtype=np.float32)
    base = np.float32(2.0) ** e
    vals = np.concatenate([base, np.nextafter(base, np.float32(0)), np.nextafter(base, np.float32(10))])
    g1 = np.stack([vals, np.zeros_like(vals)], 1).astype(np.float32)
    g2 = np.stack([np.zeros_like(vals), vals[::-1]], 1).astype(np.float32)
    uv = np.zeros_like(g1)
    for off in range(-2, 3):
        np.testing.assert_array_equal(oracle.mip_texel(uv, g1, g2, off)[0], ref.mip_texel(uv, g1, g2, off)[0])


def test_footprint_fbm_rng_bit_exact(oracle, ref):
    import make_golden
    R = make_golden.random_inputs(seed=99, n=50_000)
    np.testing.assert_array_equal(bits(oracle.footprint(R["fp_in"])), bits(ref.footprint(R["fp_in"])))
    np.testing.assert_array_equal(bits(oracle.fbm(R["octaves"], R["fbm_p"], R["fbm_uv"])),
                                  bits(ref.fbm(R["octaves"], R["fbm_p"], R["fbm_uv"])))
    got = np.array([oracle.L.mco_rng(5, int(p), int(s), int(d))
                    for p, s, d in zip(R["rng_px"][:2000], R["rng_s"][:2000], R["rng_d"][:2000])], np.float32)
    np.testing.assert_array_equal(got, ref.rng(5, R["rng_px"][:2000], R["rng_s"][:2000], R["rng_d"][:2000]))


def test_libm_differences_are_one_ulp(oracle, ref):
    r = np.random.default_rng(3)
    x = r.uniform(-200, 200, 1_000_000).astype(np.float32)
    a, b = oracle.sin_wave(x), ref.sin_wave(x)
    assert np.abs(a.astype(np.float64) - b).max() <= 2.0 ** -24
    xs = r.uniform(0, 8, 1_000_000).astype(np.float32)
    ys = r.uniform(-6, 6, 1_000_000).astype(np.float32)
    a, b = oracle.power(xs, ys), ref.power(xs, ys)
    assert np.abs(a.view(np.int32).astype(np.int64) - b.view(np.int32)).max() <= 1
    # special cases of ops::power (value.hpp:132-137) are exact
    sx = np.array([0, 0, 0, 1, 2, -1, np.inf, 0.5, np.nan, 2], np.float32)
    sy = np.array([0, 1, -1, np.nan, 0, 2, 1, np.inf, 1, -np.inf], np.float32)
    np.testing.assert_array_equal(bits(oracle.power(sx, sy)), bits(ref.power(sx, sy)))


def test_table_operations_bit_exact(oracle, ref):
    r = np.random.default_rng(9)
    for nc, ne in ((1, 1), (7, 3), (1000, 10), (4096, 2)):
        n = 30_000
        k = r.integers(0, 5000, n)
        d = descriptors(k % 8, k // 8, k % 25, k * 31, k * 17)
        rgb = r.uniform(-1, 5, (n, 3)).astype(np.float32)
        oc, rc = oracle.cache_new(nc, ne), ref.cache_new(nc, ne)
        for x, y in zip(oracle.cache_update(oc, d, rgb), ref.cache_update(rc, d, rgb)):
            np.testing.assert_array_equal(x, y)
        h1, v1 = oracle.cache_lookup(oc, d)
        h2, v2 = ref.cache_lookup(rc, d)
        np.testing.assert_array_equal(h1, h2)
        np.testing.assert_array_equal(bits(v1), bits(v2))
        np.testing.assert_array_equal(oracle.cache_slots(oc, nc, ne), ref.cache_slots(rc, nc * ne))
        np.testing.assert_array_equal(oracle.cache_counters(oc), ref.cache_counters(rc))
        oracle.cache_free(oc)
        ref.cache_free(rc)


def test_cache_size_errors(ref):
    with pytest.raises(ValueError):
        ref.cache_new(0, 4)
    from paper_2305_07238_b200 import memory_bytes
    with pytest.raises(OverflowError):
        memory_bytes(1 << 62, 8)
    assert memory_bytes(0, 5) == 0


@pytest.mark.parametrize("libm", [False, True])
def test_vm_matches_reference_execute(oracle, ref, scene_dir, libm):
    path = scenes.materials_only_scene(f"{scene_dir}/vm_{int(libm)}", 50, seed=21 + libm, libm_ops=libm)
    s = load_scene(path)
    rs = ref.scene_load(path)
    sp = scenes.random_shading_points(400, 5)
    mism = 0
    for slot in range(s.n_materials):
        a = oracle.execute(s.flat, slot, sp)
        b = ref.execute(rs, slot, sp)
        e = ref.eval_reference(rs, slot, sp)
        np.testing.assert_array_equal(bits(b[0]), bits(e))   # reference: VM == recursive evaluator
        np.testing.assert_array_equal(a[2], b[2])             # instructions executed
        same = (bits(a[0]) == bits(b[0])).all(axis=1)
        if not libm:
            assert same.all(), f"slot {slot}"
        mism += int((~same).sum())
    if libm:
        assert mism < 0.02 * s.n_materials * len(sp)
    ref.L.ref_scene_free(rs)


def test_vm_with_cache_matches_reference(oracle, ref, scene_dir):
    path = scenes.materials_only_scene(f"{scene_dir}/vm_cache", 20, seed=31, libm_ops=False)
    s = load_scene(path)
    rs = ref.scene_load(path)
    sp = scenes.random_shading_points(2000, 8, uv_range=1.0)
    sp[:, 11:15] = np.float32(0.02)
    for slot in range(s.n_materials):
        oc, rc = oracle.cache_new(509, 4), ref.cache_new(509, 4)
        for _ in range(2):
            for mip in (0, 2):
                a = oracle.execute(s.flat, slot, sp, cache=oc, mip_offset=mip)
                b = ref.execute(rs, slot, sp, cache=rc, mip_offset=mip)
                np.testing.assert_array_equal(bits(a[0]), bits(b[0]))
                np.testing.assert_array_equal(a[1], b[1])
                np.testing.assert_array_equal(a[2], b[2])
        np.testing.assert_array_equal(oracle.cache_slots(oc, 509, 4), ref.cache_slots(rc, 509 * 4))
        oracle.cache_free(oc)
        ref.cache_free(rc)


@pytest.mark.parametrize("kind,spheres", [("cornell", 0), ("classroom", 0), ("cornell", 24)])
def test_bvh_queries_bit_exact(oracle, ref, scene_dir, kind, spheres):
    """Closest / any hit vs Scene::intersect / occluded: bit-exact, except a
    sphere hit's uv (atan2f/acosf, scene.cpp:234-235), which the oracle and
    the device take from the deterministic routines: within 1 ulp of glibc's."""
    path = scenes.build_scene(scenes.SceneSpec(kind, 16, 16, tris_per_side=8, spheres=spheres),
                              f"{scene_dir}/bvh_{kind}_{spheres}")
    s = load_scene(path)
    rs = ref.scene_load(path)
    r = np.random.default_rng(4)
    n = 100_000
    o = r.uniform([-7.9, 0.01, -9.9], [7.9, 4.99, 9.9], (n, 3))
    d = r.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d[:200] = [0, -1, 0]   # axis-aligned rays (infinite reciprocals)
    d[200:400] = [1, 0, 0]
    rays = np.concatenate([o, d], 1).astype(np.float32)
    A, B = oracle.intersect(s.flat, rays), ref.intersect(rs, rays)
    if spheres:
        # u = 0.5 + atan2f/(2 pi), v = acosf/pi: one ulp of atan2f/acosf
        # (<= 2^-22 on [0, pi]) moves u or v by at most 2^-23 + a rounding.
        du = np.abs(A[:, 8:10].astype(np.float64) - B[:, 8:10])
        assert du.max() <= 2.0 ** -22
        assert 0 < (du.sum(1) > 0).mean() < 0.05
        A, B = np.delete(A, [8, 9], 1), np.delete(B, [8, 9], 1)
    np.testing.assert_array_equal(bits(A), bits(B))
    tm = r.uniform(0.01, 20, n).astype(np.float32)
    np.testing.assert_array_equal(oracle.occluded(s.flat, rays, 1e-4, tm), ref.occluded(rs, rays, 1e-4, tm))
    ref.L.ref_scene_free(rs)


@pytest.mark.parametrize("tps,spheres", [(6, 8), (80, 40)])
def test_bvh_nodes_identical_to_reference(ref, scene_dir, tps, spheres):
    """libmcg's BVH build (precomputed centroids; subtrees on parallel threads
    above 65 536 primitives) == Scene::prepare's tree node for node: bounds,
    children, leaf ranges (scene.cpp:154-194)."""
    path = scenes.build_scene(scenes.SceneSpec("classroom", 16, 16, tris_per_side=tps, spheres=spheres),
                              f"{scene_dir}/bvhn_{tps}")
    s = load_scene(path)
    rs = ref.scene_load(path)
    want = ref.bvh(rs)
    ref.L.ref_scene_free(rs)
    f = s.flat
    got = np.ctypeslib.as_array(ctypes.cast(f.nodes, ctypes.POINTER(ctypes.c_uint32)), (f.n_nodes * 8,))
    got = got.reshape(-1, 8)
    assert got.shape[0] == want.shape[0]
    if tps == 80:
        assert f.n_prims >= 65536
    np.testing.assert_array_equal(got[:, 0:3], want[:, 0:3])
    np.testing.assert_array_equal(got[:, 4:7], want[:, 3:6])
    a, b = got[:, 3].view(np.int32), got[:, 7].view(np.int32)
    left, right = want[:, 6].view(np.int32), want[:, 7].view(np.int32)
    leaf = left < 0
    np.testing.assert_array_equal(a < 0, leaf)
    np.testing.assert_array_equal(a[~leaf], left[~leaf])
    np.testing.assert_array_equal(b[~leaf], right[~leaf])
    np.testing.assert_array_equal(~a[leaf], want[leaf, 8].view(np.int32))
    np.testing.assert_array_equal(b[leaf], want[leaf, 9].view(np.int32))


def test_camera_setup_matches(oracle, scene_dir):
    path = scenes.build_scene(scenes.SceneSpec("cornell", 64, 48, tris_per_side=2), f"{scene_dir}/cam")
    s = load_scene(path)
    for w, h in ((64, 48), (1920, 1080), (7, 3)):
        np.testing.assert_array_equal(bits(s.camera_setup(w, h)), bits(oracle.camera(s.flat, w, h)))


@pytest.mark.parametrize("kind,libm,mode,k", [("cornell", False, 0, 1), ("cornell", False, 1, 1),
                                              ("italianflat", False, 1, 2), ("junkshop", False, 1, 3),
                                              ("classroom", True, 0, 1), ("classroom", True, 1, 2)])
def test_render_matches_reference_backed_render(oracle, ref, scene_dir, kind, libm, mode, k):
    """render() restated over the reference's own intersect/footprint/execute/
    MaterialCache (oracle/ref_harness.cpp) vs the C oracle: cache off and the
    epoch-sequential cached order."""
    w, h, spp = 40, 28, 4
    path = scenes.build_scene(scenes.SceneSpec(kind, w, h, tris_per_side=5, libm_ops=libm),
                              f"{scene_dir}/rr_{kind}_{int(libm)}")
    s = load_scene(path)
    rs = ref.scene_load(path)
    P = RenderParamsC(w, h, spp, 4, mode, 0, 1021, 4, 0, 1, 0.2, 16, 0, 1, 0, 0, k)
    A = oracle.render(s.flat, P)
    B = ref.render(rs, P, w, h)
    np.testing.assert_array_equal(A[2], B[2])
    np.testing.assert_array_equal(A[1], B[1])     # per-pixel hit counts
    np.testing.assert_array_equal(A[3], B[3])     # hits per sample
    if libm:
        assert np.abs(A[0] - B[0]).max() <= 1e-5 * np.abs(B[0]).max()
    else:
        np.testing.assert_array_equal(bits(A[0]), bits(B[0]))
    for f in ("lookups", "hits", "inserts_won", "inserts_lost_full", "instructions_executed", "shading_points"):
        assert getattr(A[4], f) == getattr(B[4], f), f
    ref.L.ref_scene_free(rs)


@pytest.mark.parametrize("kind,libm,k,nc,ne", [("cornell", False, 1, 1021, 4), ("junkshop", False, 2, 1021, 4),
                                               ("italianflat", False, 3, 61, 3), ("monster", False, 2, 4099, 10),
                                               ("classroom", True, 2, 1021, 4)])
def test_deterministic_render_matches_reference_deferred_render(oracle, ref, scene_dir, kind, libm, k, nc, ne):
    """Deterministic-insert mode pinned to reference-compiled code: the
    reference-backed render in mode 3 (ref_harness.cpp class Deferred: the
    reference's execute() against the epoch-start table, its inserts taken
    back and re-applied at the epoch's end, sorted by (sample-in-pass,
    pixel, store ordinal), through MaterialCache::update, cache.cpp:94-119)
    vs mc_oracle.c mode 3 -- the rule the GPU's k_shade<true> +
    k_apply_ordered follow. Per-pixel hit counts, hits per sample, counters
    and every table word bit-exact; radiance bit-exact without libm ops and
    within 1e-5 relative with them (sin/pow: glibc vs the correctly rounded
    routine, <= 1 ulp). A 61 x 3 table exercises CellFull."""
    w, h, spp = 40, 28, 6
    path = scenes.build_scene(scenes.SceneSpec(kind, w, h, tris_per_side=5, libm_ops=libm),
                              f"{scene_dir}/det_{kind}_{int(libm)}")
    s = load_scene(path)
    rs = ref.scene_load(path)
    P = RenderParamsC(w, h, spp, 4, 3, 0, nc, ne, 0, 1, 0.2, 16, 0, 1, 0, 0, k)
    oc = oracle.cache_new(nc, ne)
    rc = ref.cache_new(nc, ne)
    A = oracle.render(s.flat, P, cache=oc)
    B = ref.render(rs, P, w, h, cache=rc)
    np.testing.assert_array_equal(A[2], B[2])
    np.testing.assert_array_equal(A[1], B[1])     # per-pixel hit counts
    np.testing.assert_array_equal(A[3], B[3])     # hits per sample
    np.testing.assert_array_equal(oracle.cache_slots(oc, nc, ne), ref.cache_slots(rc, nc * ne))
    if libm:
        assert np.abs(A[0] - B[0]).max() <= 1e-5 * np.abs(B[0]).max()
    else:
        np.testing.assert_array_equal(bits(A[0]), bits(B[0]))
    for f in ("lookups", "hits", "inserts_won", "inserts_lost_full", "stores_attempted", "stores_won",
              "instructions_executed", "shading_points"):
        assert getattr(A[4], f) == getattr(B[4], f), f
    assert B[4].hits > 0 and B[4].inserts_won > 0
    if nc == 61:
        assert B[4].inserts_lost_full > 0
    # and it is not the immediate-insert order (mode 1) under another name:
    # there, later paths of an epoch already hit what earlier ones stored
    P.mode = 1
    rc1 = ref.cache_new(nc, ne)
    B1 = ref.render(rs, P, w, h, cache=rc1)
    assert B1[4].hits > B[4].hits
    oracle.cache_free(oc)
    ref.cache_free(rc)
    ref.cache_free(rc1)
    ref.L.ref_scene_free(rs)


def test_render_with_spheres_matches_reference_backed_render(oracle, ref, scene_dir):
    """Cache off, a scene with analytic spheres: sphere uv differs from
    glibc's by <= 1 ulp of atan2f/acosf, so radiance is compared at the
    north-star 1e-5 relative bound; everything else exactly."""
    w, h, spp = 40, 28, 4
    path = scenes.build_scene(scenes.SceneSpec("junkshop", w, h, tris_per_side=5, spheres=16),
                              f"{scene_dir}/rr_spheres")
    s = load_scene(path)
    rs = ref.scene_load(path)
    P = RenderParamsC(w, h, spp, 4, 0, 0, 1021, 4, 0, 1, 0.2, 16, 0, 1, 0, 0, 1)
    A = oracle.render(s.flat, P)
    B = ref.render(rs, P, w, h)
    np.testing.assert_array_equal(A[2], B[2])
    assert np.abs(A[0] - B[0]).max() <= 1e-5 * np.abs(B[0]).max()
    for f in ("instructions_executed", "shading_points"):
        assert getattr(A[4], f) == getattr(B[4], f), f
    ref.L.ref_scene_free(rs)


def test_sharded_oracle_renders_partition_the_image(oracle, scene_dir):
    """Tile sharding (tracer.hpp:19): the shards' renders (cache off) sum to
    the full render exactly -- every pixel belongs to exactly one rank."""
    w, h, spp = 50, 37, 2
    path = scenes.build_scene(scenes.SceneSpec("cornell", w, h, tris_per_side=3), f"{scene_dir}/shard")
    s = load_scene(path)
    full = oracle.render(s.flat, RenderParamsC(w, h, spp, 4, 0, 0, 97, 4, 0, 1, 0.2, 16, 0, 1, 0, 0, 1))
    for mode in (0, 1):
        for G in (2, 3, 8):
            acc = np.zeros_like(full[0])
            cnt = np.zeros_like(full[2])
            for r in range(G):
                part = oracle.render(s.flat, RenderParamsC(w, h, spp, 4, 0, 0, 97, 4, 0, 1, 0.2, 16, r, G, mode, 0, 1))
                assert not ((cnt > 0) & (part[2] > 0)).any()
                acc += part[0]
                cnt += part[2]
            np.testing.assert_array_equal(bits(acc), bits(full[0]))
            np.testing.assert_array_equal(cnt, full[2])


def test_reference_probe_bench_threads_agree(ref):
    """The CPU leg of the probe microbenchmark (ref_probe_bench): lookups are
    read-only, so 1 and 4 threads find the same hits after one insert-all."""
    nc, ne, n = 20011, 4, 1 << 16
    c = ref.cache_new(nc, ne)
    ref.probe_bench(c, n, 7, 0, 1)
    words = ref.cache_slots(c, nc * ne)
    base = ref.cache_counters(c)
    ref.probe_bench(c, n, 7, 1, 1)
    one = ref.cache_counters(c) - base
    ref.probe_bench(c, n, 7, 1, 4)
    four = ref.cache_counters(c) - base - one
    assert one[0] == four[0] == n and one[1] == four[1] > 0
    np.testing.assert_array_equal(ref.cache_slots(c, nc * ne), words)
    ref.cache_free(c)
