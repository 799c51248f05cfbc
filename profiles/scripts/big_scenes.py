"""Scaling with scene size: the classroom analogue with finer
wall tessellation, 1920x1080x32 with the cache, plus a small cache-off render
checked bit for bit against the oracle. Run on a GPU box."""
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render, scenes  # noqa: E402

import _oracle  # noqa: E402

ctx = Context(0)
orc = _oracle.Oracle()
for tps in (24, 96, 300):
    d = tempfile.mkdtemp()
    t0 = time.perf_counter()
    s = load_scene(scenes.build_scene(scenes.SceneSpec("classroom", 1920, 1080, tris_per_side=tps), d))
    t_load = time.perf_counter() - t0
    t0 = time.perf_counter()
    ctx.upload(s)
    t_up = time.perf_counter() - t0
    cfg = RenderConfig(width=1920, height=1080, spp=32, cache_enabled=True, n_cells=10_000_000, n_entries=10)
    render(s, cfg, ctx=ctx)
    r = render(s, cfg, ctx=ctx)
    small = RenderConfig(width=32, height=24, spp=2)
    g = render(s, small, ctx=ctx).frame.radiance
    P = _oracle.RenderParamsC(32, 24, 2, 4, 0, 0, 1, 1, 0, 1, 0.2, 16, 0, 1, 0, 1, 1)
    o = orc.render(s.flat, P)[0]
    exact = bool(np.array_equal(g.view(np.uint64), o.view(np.uint64)))
    print(f"tris_per_side={tps}: prims={s.flat.n_prims} nodes={s.flat.n_nodes} load+build {t_load:.2f} s "
          f"upload {t_up:.2f} s render {r.stats.device_ms:.1f} ms "
          f"({1920 * 1080 * 32 / r.stats.device_ms / 1e3:.0f} M samples/s) hit rate {r.stats.hit_rate:.4f} "
          f"cache-off 32x24 == oracle: {exact}", flush=True)
