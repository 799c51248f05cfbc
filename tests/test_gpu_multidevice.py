"""In-process multi-GPU render behind the C ABI (mcg_options.n_devices; the
reference's render() is one synchronous call over every worker,
tracer.hpp:12, 69-70): tiles dealt to the devices, one cache replica per
device, frames gathered on the first device.

This box has one GPU: the context lists device 0 twice, which runs the same
host threads, per-device sharding, replicas and exact zero-outside-my-tiles
gather, with device copies in place of the NCCL reduce (NCCL refuses a
device twice in one communicator). The NCCL call sequence itself runs only
with distinct devices."""
import numpy as np
import pytest

from paper_2305_07238_b200 import (Context, MaterialCache, RenderConfig, load_scene, render, scenes)

import _oracle

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.fixture(scope="module")
def multi(built):
    from conftest import _gpu_available
    if not _gpu_available():
        pytest.skip("no CUDA device")
    c = Context(devices=[0, 0])
    yield c
    c.close()


@pytest.mark.parametrize("shard_mode", [0, 1])
def test_two_device_cache_off_equals_one_device(ctx, multi, scene_dir, shard_mode):
    w, h, spp = 80, 56, 3
    s = load_scene(scenes.build_scene(scenes.SceneSpec("junkshop", w, h, tris_per_side=5), f"{scene_dir}/md"))
    one = render(s, RenderConfig(width=w, height=h, spp=spp), ctx=ctx)
    two = render(s, RenderConfig(width=w, height=h, spp=spp, shard_mode=shard_mode), ctx=multi)
    np.testing.assert_array_equal(bits(two.frame.radiance), bits(one.frame.radiance))
    np.testing.assert_array_equal(two.frame.samples, one.frame.samples)
    assert two.stats.shading_points == one.stats.shading_points
    assert two.stats.paths == one.stats.paths == w * h * spp
    # progressive: a second render accumulates into the same host frame
    render(s, RenderConfig(width=w, height=h, spp=spp, first_sample=spp), ctx=ctx, frame=one.frame)
    render(s, RenderConfig(width=w, height=h, spp=spp, first_sample=spp, shard_mode=shard_mode), ctx=multi,
           frame=two.frame)
    np.testing.assert_array_equal(bits(two.frame.radiance), bits(one.frame.radiance))


def test_two_device_deterministic_equals_per_shard_oracle(multi, oracle, scene_dir):
    """Per-device replicas: each device's table sees only its
    tiles, so the image is the sum of the oracle's per-shard renders, each
    with a fresh table, bit for bit (deterministic mode)."""
    w, h, spp, nc, ne = 64, 48, 4, 4099, 4
    s = load_scene(scenes.build_scene(scenes.SceneSpec("italianflat", w, h, tris_per_side=5, libm_ops=True),
                                      f"{scene_dir}/md_det"))
    res = render(s, RenderConfig(width=w, height=h, spp=spp, cache_enabled=True, deterministic=True,
                                 n_cells=nc, n_entries=ne, samples_per_pass=2), ctx=multi)
    rad = np.zeros((h, w, 3))
    nodes = np.zeros((h, w))
    hits = 0
    for r in range(2):
        oc = oracle.cache_new(nc, ne)
        p = _oracle.RenderParamsC(w, h, spp, 4, 3, 0, nc, ne, 0, 1, 0.2, 16, r, 2, 0, 0, 2)
        a, n, smp, hps, st = oracle.render(s.flat, p, cache=oc)
        rad += a
        nodes += n
        hits += st.hits
        oracle.cache_free(oc)
    np.testing.assert_array_equal(res.frame.nodes_found, nodes)
    np.testing.assert_array_equal(bits(res.frame.radiance), bits(rad))
    assert res.stats.hits == hits > 0
    assert sum(res.stats.hits_per_sample) == hits


def test_multi_device_refuses_external_cache_and_device_frames(multi, scene_dir):
    from paper_2305_07238_b200 import _native as N
    s = load_scene(scenes.build_scene(scenes.SceneSpec("cornell", 16, 16, tris_per_side=2), f"{scene_dir}/md_err"))
    table = MaterialCache(97, 4, Context.default())
    with pytest.raises(ValueError, match="replica"):
        render(s, RenderConfig(width=16, height=16, spp=1, cache_enabled=True, n_cells=97, n_entries=4),
               external_cache=table, ctx=multi)
    with pytest.raises(ValueError, match="shards the image"):
        render(s, RenderConfig(width=16, height=16, spp=1, shard_count=2), ctx=multi)
    import ctypes as C
    fr = N.Frame()
    rc = N.lib().mcg_render_device(multi.handle, C.byref(RenderConfig(width=16, height=16).to_params()), None,
                                   C.byref(fr), None)
    assert rc != 0
