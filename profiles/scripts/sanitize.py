"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of libmcg once, on sizes that finish in
seconds under the tool. Run as

    compute-sanitizer --tool memcheck  python profiles/scripts/sanitize.py
    compute-sanitizer --tool racecheck python profiles/scripts/sanitize.py

(compute-sanitizer is closed on this GPU pool; profiles/scripts/checked.sh runs
this workload and the -m gpu suite on the bounds-checked build instead)."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2305_07238_b200 import (Context, MaterialCache, RenderConfig, descriptors, load_scene,  # noqa: E402
                                   render, scenes)

ctx = Context(0)
tmp = tempfile.mkdtemp()
r = np.random.default_rng(3)
# descriptor pipeline, table updates (concurrent and ordered), lookups
d = descriptors(r.integers(0, 8, 5000), r.integers(0, 64, 5000), r.integers(0, 17, 5000),
                r.integers(0, 256, 5000), r.integers(0, 256, 5000))
rgb = r.uniform(0, 3, (5000, 3)).astype(np.float32)
ctx.hash_batch(d)
ctx.encode_batch(rgb)
for ne in (4, 10, 12):
    t = MaterialCache(997, ne, ctx)
    t.update_batch(d, rgb, ordered=False)
    t.update_batch(d, rgb, ordered=True)
    t.lookup_batch(d)
    t.insert_log_start(4096)
    t.update_batch(d[::-1].copy(), rgb, ordered=False)
    t.insert_log_read(min(4096, t.insert_log_stop()))
    t.occupied_slots()
    t.close()
# probe microbenchmark variants and the trace replay
t = MaterialCache(10_007, 10, ctx)
for v in (0, 4, 5, 10):
    t.probe_bench(1 << 16, 7, 0 + 16 * v, 1)
    t.probe_bench(1 << 16, 7, 1 + 16 * v, 1)
    t.probe_bench(1 << 16, 8, 2 + 16 * v, 1)
t.probe_replay(d)
t.close()
# renders: cache off, concurrent (two pass lanes, several passes, insert
# log on), deterministic (queued stores, CUB sort, ordered apply), with
# spheres; scene queries through every traversal variant
s = load_scene(scenes.build_scene(scenes.SceneSpec("junkshop", 48, 32, tris_per_side=4, spheres=4),
                                  os.path.join(tmp, "s")))
render(s, RenderConfig(width=48, height=32, spp=2), ctx=ctx)
c = MaterialCache(4099, 10, ctx)
c.insert_log_start(1 << 16)
render(s, RenderConfig(width=48, height=32, spp=6, cache_enabled=True, n_cells=4099, n_entries=10,
                       samples_per_pass=1), external_cache=c, ctx=ctx)
c.insert_log_stop()
render(s, RenderConfig(width=48, height=32, spp=4, cache_enabled=True, deterministic=True, n_cells=4099,
                       n_entries=10, samples_per_pass=2), ctx=ctx)
rays = np.concatenate([r.uniform([-7, 0.1, -9], [7, 4.9, 9], (2000, 3)),
                       r.normal(size=(2000, 3))], 1).astype(np.float32)
rays[:, 3:] /= np.linalg.norm(rays[:, 3:], axis=1, keepdims=True)
for v in range(5):
    ctx.intersect_batch(rays, 1e-4, np.inf, v)
for v in range(6):
    ctx.occluded_batch(rays, 1e-4, np.full(2000, 5.0, np.float32), v)
sp = scenes.random_shading_points(512, 4, uv_range=1.0)
for slot in range(s.n_materials):
    ctx.execute_batch(slot, sp)
ctx.synchronize()
print("sanitize workload done")
