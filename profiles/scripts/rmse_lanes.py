import os, sys, numpy as np, tempfile
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2305_07238_b200 import RenderConfig, load_scene, render, scenes, Context
ctx = Context(0)
w, h, spp, nc, ne = 96, 64, 8, 20011, 8
path = scenes.build_scene(scenes.SceneSpec("classroom", w, h, tris_per_side=6, libm_ops=True), tempfile.mkdtemp())
s = load_scene(path)
off = render(s, RenderConfig(width=w, height=h, spp=spp), ctx=ctx).frame.radiance_image()
rmse = lambda a, b: float(np.sqrt(np.mean((a.astype(np.float64) - b) ** 2)))
for lanes in ("1", "2"):
    os.environ["MCG_LANES"] = lanes
    for spp_pass in (0, 1, 2, 4):
        for det in (False, True):
            r = render(s, RenderConfig(width=w, height=h, spp=spp, cache_enabled=True, n_cells=nc, n_entries=ne,
                                       samples_per_pass=spp_pass, deterministic=det), ctx=ctx)
            print("lanes", lanes, "spp_pass", spp_pass, "det", det, "rmse", round(rmse(r.frame.radiance_image(), off), 4),
                  "hit", round(r.stats.hit_rate, 4), flush=True)
