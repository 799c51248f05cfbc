"""Device build of the any-hit (shadow) tree (csrc/mcg_build.cu, SURVEY
§8f.4): the binned-SAH hierarchy over the reference BVH's leaves that the
host builder makes, built level by level on the GPU.

Any hierarchy over the reference's leaves answers Scene::occluded
(scene.cpp:280-298) exactly, so renders must be bit-identical whichever
builder ran; and the device tree is the host's tree: same SAH decisions and
the same leaf order (libstdc++'s partition permutation), only node numbering
differs -- compared as canonical nested tuples from the root."""
import numpy as np
import pytest

from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render, scenes

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def canonical(tree, root):
    """The hierarchy as nested tuples from the root, children in entry order
    (independent of node numbering): leaves by (first, count, box bytes),
    nodes by (box bytes, children)."""
    nodes, (ra, rb) = tree, root

    def entry(a, b, lo, hi):
        if b > 0:
            return ("leaf", int(a), int(b), lo.tobytes(), hi.tobytes())
        return ("node", lo.tobytes() if lo is not None else b"", hi.tobytes() if hi is not None else b"",
                tuple(entry(e["a"], e["b"], e["lo"], e["hi"]) for e in nodes[a] if e["b"] != 0))
    if rb > 0:
        return ("leaf", ra, rb)
    return entry(ra, rb, None, None)


@pytest.mark.parametrize("kind,tps,spheres", [("classroom", 24, 0), ("cornell", 8, 12), ("monster", 40, 0),
                                              ("junkshop", 60, 4)])
def test_device_shadow_tree_equals_host_tree(built, scene_dir, kind, tps, spheres, monkeypatch):
    from conftest import _gpu_available
    if not _gpu_available():
        pytest.skip("no CUDA device")
    w, h, spp = 160, 120, 4
    path = scenes.build_scene(scenes.SceneSpec(kind, w, h, tris_per_side=tps, spheres=spheres),
                              f"{scene_dir}/sb_{kind}_{tps}_{spheres}")
    s = load_scene(path)
    out = {}
    for mode in ("host", "device"):
        monkeypatch.setenv("MCG_SHADOW_BUILD", mode)
        ctx = Context(0)
        try:
            r = render(s, RenderConfig(width=w, height=h, spp=spp), ctx=ctx)
            rays = np.random.default_rng(5).normal(size=(20000, 6)).astype(np.float32)
            rays[:, :3] *= 3.0
            rays[:, 3:] /= np.linalg.norm(rays[:, 3:], axis=1, keepdims=True)
            occ = ctx.occluded_batch(rays, 1e-4, np.full(20000, 4.0, np.float32), 5)
            out[mode] = (r, occ, ctx.shadow_tree())
        finally:
            ctx.close()
    (rh, oh, th), (rd, od, td) = out["host"], out["device"]
    # exact answers whichever builder ran ...
    np.testing.assert_array_equal(bits(rh.frame.radiance), bits(rd.frame.radiance))
    np.testing.assert_array_equal(oh, od)
    assert rh.stats.shadow_occluded == rd.stats.shadow_occluded
    # ... and the same tree (node numbering aside)
    assert th[0].shape == td[0].shape
    assert canonical(*th) == canonical(*td)
