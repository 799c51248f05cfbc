"""Parity at BASELINE.json's configurations and on the exact path bench.py
times ("pin parity on the exact timed path and on the BASELINE
configs").

* C1 (configs[0]: 256x256, 4 spp, one depth-8 material graph, cache 1e5 x 10):
  the GPU render bit-exact against the C oracle and against the reference's
  own compiled code (oracle/_ref), cache off and in deterministic mode;
* a deterministic render through the paper's 1e7 x 10 table (800 MB), every
  table word compared;
* concurrent mode as bench.py runs it (two pass lanes, several passes): the
  north-star RMSE bound against the reference's own threaded render, and
  SPEC.md's render invariants (pixels without a cache hit bit-identical to
  the cache-off render; hits == sum of nodes_found).
"""
import numpy as np
import pytest

from paper_2305_07238_b200 import MaterialCache, RenderConfig, load_scene, render, scenes

import _oracle

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view({4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


def P(w, h, spp, mode, k, nc, ne, mip=0, threads=0):
    return _oracle.RenderParamsC(w, h, spp, 4, mode, mip, nc, ne, 0, 1, 0.2, 16, 0, 1, 0, threads, k)


@pytest.fixture(scope="module")
def c1_scene(scene_dir):
    # configs[0]: the cornell analogue is one depth-8 uv expression per wall
    # material (scenes.material_depth8); libm-free so that the reference's
    # glibc sin/pow do not enter and every comparison is bit for bit
    path = scenes.build_scene(scenes.SceneSpec("cornell", 256, 256, tris_per_side=8, libm_ops=False),
                              f"{scene_dir}/c1")
    return path, load_scene(path)


def test_c1_cache_off_bit_exact(ctx, oracle, ref, c1_scene):
    path, s = c1_scene
    w = h = 256
    res = render(s, RenderConfig(width=w, height=h, spp=4), ctx=ctx)
    rad, nodes, samples, hps, st = oracle.render(s.flat, P(w, h, 4, 0, 1, 1, 1))
    np.testing.assert_array_equal(bits(res.frame.radiance), bits(rad))
    np.testing.assert_array_equal(res.frame.samples, samples)
    rs = ref.scene_load(path)
    rrad, *_ = ref.render(rs, P(w, h, 4, 0, 1, 1, 1), w, h)
    ref.L.ref_scene_free(rs)
    np.testing.assert_array_equal(bits(res.frame.radiance), bits(rrad))


@pytest.mark.parametrize("k", [1, 4])
def test_c1_deterministic_bit_exact_vs_oracle_and_reference(ctx, oracle, ref, c1_scene, k):
    """Deterministic-insert mode at C1 (1e5 x 10 table): per-pixel hit counts,
    hits per sample, counters, every table word and the radiance bit-exact
    against mc_oracle.c mode 3 and against the reference-backed deferred
    render (ref_harness.cpp class Deferred: the reference's execute() and
    MaterialCache::update)."""
    path, s = c1_scene
    w = h = 256
    nc, ne = 100_000, 10
    cache = MaterialCache(nc, ne, ctx)
    res = render(s, RenderConfig(width=w, height=h, spp=4, cache_enabled=True, deterministic=True,
                                 n_cells=nc, n_entries=ne, samples_per_pass=k), external_cache=cache, ctx=ctx)
    words = cache.slot_words()
    oc = oracle.cache_new(nc, ne)
    rad, nodes, samples, hps, st = oracle.render(s.flat, P(w, h, 4, 3, k, nc, ne), cache=oc)
    np.testing.assert_array_equal(res.frame.nodes_found, nodes)
    assert res.stats.hits_per_sample == [int(x) for x in hps]
    np.testing.assert_array_equal(words, oracle.cache_slots(oc, nc, ne))
    np.testing.assert_array_equal(bits(res.frame.radiance), bits(rad))
    assert (res.stats.lookups, res.stats.hits, res.stats.inserts_won) == (st.lookups, st.hits, st.stores_won)
    oracle.cache_free(oc)
    rs = ref.scene_load(path)
    rc = ref.cache_new(nc, ne)
    rrad, rnodes, _, rhps, rst = ref.render(rs, P(w, h, 4, 3, k, nc, ne), w, h, cache=rc)
    np.testing.assert_array_equal(res.frame.nodes_found, rnodes)
    np.testing.assert_array_equal(words, ref.cache_slots(rc, nc * ne))
    np.testing.assert_array_equal(bits(res.frame.radiance), bits(rrad))
    assert (res.stats.lookups, res.stats.hits, res.stats.inserts_won) == (rst.lookups, rst.hits, rst.inserts_won)
    assert res.stats.hits > 0 and res.stats.inserts_won > 0
    ref.cache_free(rc)
    ref.L.ref_scene_free(rs)


def test_deterministic_through_the_1e7_x_10_table(ctx, oracle, scene_dir):
    """The paper's table size (800 MB, ~1/8 of it ever touched here): the
    device's head/tail split layout and fast-mod cell index against the
    oracle's flat table, every one of the 10^8 words compared."""
    w, h, spp, nc, ne = 96, 64, 4, 10_000_000, 10
    path = scenes.build_scene(scenes.SceneSpec("junkshop", w, h, tris_per_side=6, libm_ops=True),
                              f"{scene_dir}/big_table")
    s = load_scene(path)
    cache = MaterialCache(nc, ne, ctx)
    res = render(s, RenderConfig(width=w, height=h, spp=spp, cache_enabled=True, deterministic=True,
                                 n_cells=nc, n_entries=ne, samples_per_pass=2), external_cache=cache, ctx=ctx)
    oc = oracle.cache_new(nc, ne)
    rad, nodes, samples, hps, st = oracle.render(s.flat, P(w, h, spp, 3, 2, nc, ne), cache=oc)
    np.testing.assert_array_equal(res.frame.nodes_found, nodes)
    np.testing.assert_array_equal(bits(res.frame.radiance), bits(rad))
    words = cache.slot_words()
    np.testing.assert_array_equal(words, oracle.cache_slots(oc, nc, ne))
    assert int((words != 0).sum()) == res.stats.inserts_won > 0
    oracle.cache_free(oc)
    cache.close()
