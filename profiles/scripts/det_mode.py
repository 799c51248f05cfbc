"""Deterministic-insert mode on the bench workload (1920x1080x128, cache
1e7x10): device time vs concurrent mode, and run-to-run identity."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render  # noqa: E402

ctx = Context(0)
scene = load_scene(bench.make_scene(tempfile.mkdtemp()))
out = {}
for det in (False, True):
    cfg = RenderConfig(width=bench.W, height=bench.H, spp=bench.SPP, cache_enabled=True, deterministic=det,
                       n_cells=bench.N_CELLS, n_entries=bench.N_ENTRIES, mip_offset=bench.MIP_OFFSET)
    render(scene, cfg, ctx=ctx)
    a = render(scene, cfg, ctx=ctx)
    b = render(scene, cfg, ctx=ctx)
    same = bool(np.array_equal(a.frame.radiance, b.frame.radiance) and
                np.array_equal(a.frame.nodes_found, b.frame.nodes_found))
    ms = min(a.stats.device_ms, b.stats.device_ms)
    out["deterministic" if det else "concurrent"] = ms
    print(f"{'deterministic' if det else 'concurrent'}: {ms:.1f} ms/render "
          f"({bench.W * bench.H * bench.SPP / ms / 1e3:.0f} M samples/s), hit rate {a.stats.hit_rate:.4f}, "
          f"two runs identical: {same}", flush=True)
