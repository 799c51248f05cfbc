import sys, os, json, statistics, tempfile
sys.path.insert(0, os.getcwd())
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render, scenes
ctx = Context(0)
for kind in ("bmw", "classroom"):
    s = load_scene(scenes.build_scene(scenes.SceneSpec(kind, 1920, 1080, tris_per_side=24, uv_span=0.999), tempfile.mkdtemp()))
    base = RenderConfig(width=1920, height=1080, spp=128, n_cells=10_000_000, n_entries=10)
    render(s, base, ctx=ctx)
    off = statistics.median(render(s, base, ctx=ctx).stats.device_ms for _ in range(3))
    on = statistics.median(render(s, RenderConfig(**{**base.__dict__, "cache_enabled": True, "mip_offset": 24}), ctx=ctx).stats.device_ms for _ in range(3))
    print(kind, "off", off, "mip24", on, "throughput vs no cache %", 100 * off / on, flush=True)
