"""One render of a scene analogue for ncu captures:
python profiles/scripts/prof_scene.py KIND MIP_OFFSET CACHE(0|1) [SPP] [RENDERS]
(1920x1080, one uv tile per surface, table 1e7x10)."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render, scenes  # noqa: E402

kind, mip, cache = sys.argv[1], int(sys.argv[2]), sys.argv[3] != "0"
spp = int(sys.argv[4]) if len(sys.argv) > 4 else 128
n = int(sys.argv[5]) if len(sys.argv) > 5 else 1
ctx = Context(0)
s = load_scene(scenes.build_scene(scenes.SceneSpec(kind, 1920, 1080, tris_per_side=24, uv_span=0.999),
                                  tempfile.mkdtemp()))
cfg = RenderConfig(width=1920, height=1080, spp=spp, cache_enabled=cache, n_cells=10_000_000, n_entries=10,
                   mip_offset=mip)
for _ in range(n):
    r = render(s, cfg, ctx=ctx)
print(kind, mip, cache, r.stats.device_ms, r.stats.hit_rate, r.stats.lookups, r.stats.inserts_won,
      r.stats.inserts_lost_full, r.stats.stores_attempted)
