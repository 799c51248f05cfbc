"""Progressive-fill curve (tracer.hpp:54 hits_per_sample): cache
hits per sample index over the bench render, and the table's occupancy after
it. Writes profiles/fill_curve.csv."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2305_07238_b200 import Context, MaterialCache, RenderConfig, load_scene, render  # noqa: E402

ctx = Context(0)
scene = load_scene(bench.make_scene(tempfile.mkdtemp()))
table = MaterialCache(bench.N_CELLS, bench.N_ENTRIES, ctx)
cfg = RenderConfig(width=bench.W, height=bench.H, spp=bench.SPP, cache_enabled=True, n_cells=bench.N_CELLS,
                   n_entries=bench.N_ENTRIES)
res = render(scene, cfg, external_cache=table, ctx=ctx)
hps = res.stats.hits_per_sample
px = bench.W * bench.H
with open(os.path.join(ROOT, "profiles", "fill_curve.csv"), "w") as f:
    f.write("sample,hits,hits_per_pixel\n")
    for i, h in enumerate(hps):
        f.write(f"{i},{h},{h / px:.6f}\n")
print("samples", len(hps), "first", hps[:3], "last", hps[-3:], "occupied slots", table.occupied_slots())
