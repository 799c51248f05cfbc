"""Short render of the bench workload (1920x1080, classroom-like, cache 1e7x10)
for ncu captures: spp is small so a `--set full` capture of a few launches
finishes quickly. Usage: python profiles/scripts/prof_render.py [spp] [cache 0|1] [renders]"""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render  # noqa: E402

spp = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cache = (sys.argv[2] != "0") if len(sys.argv) > 2 else True
ctx = Context(0)
scene = load_scene(bench.make_scene(tempfile.mkdtemp()))
cfg = RenderConfig(width=bench.W, height=bench.H, spp=spp, cache_enabled=cache,
                   n_cells=bench.N_CELLS, n_entries=bench.N_ENTRIES, mip_offset=bench.MIP_OFFSET)
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    r = render(scene, cfg, ctx=ctx)
print("ok", r.stats.shading_points, r.stats.hits)
