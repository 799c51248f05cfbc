import sys, os, tempfile
sys.path.insert(0, "/root/repo")
os.chdir("/root/repo")
import bench
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render
import torch
ctx = Context(0, profile=True)
scene = load_scene(bench.make_scene(tempfile.mkdtemp()))
cfg = RenderConfig(width=bench.W, height=bench.H, spp=bench.SPP, cache_enabled=True, n_cells=bench.N_CELLS, n_entries=bench.N_ENTRIES)
for _ in range(2): r = render(scene, cfg, ctx=ctx)
ctx.reset_kernel_times()
r = render(scene, cfg, ctx=ctx)
kt = ctx.kernel_times()
tot = sum(v["ms"] for v in kt.values())
print("device_ms", r.stats.device_ms, "sum kernel ms", tot, "launches", sum(v["launches"] for v in kt.values()))
