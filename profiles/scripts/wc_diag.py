import sys, os, statistics, tempfile
sys.path.insert(0, os.getcwd())
import torch
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render, scenes
s = load_scene(scenes.build_scene(scenes.SceneSpec("bmw", 1920, 1080, tris_per_side=24, uv_span=0.999), tempfile.mkdtemp()))
base = dict(width=1920, height=1080, spp=128, n_cells=10_000_000, n_entries=10, mip_offset=24)
stream = torch.cuda.Stream()
for name, ctx in (("plain", Context(0)), ("profile", Context(0, profile=True)), ("profile+stream", Context(0, profile=True, stream=stream.cuda_stream))):
    render(s, RenderConfig(**base), ctx=ctx)
    off = [render(s, RenderConfig(**base), ctx=ctx).stats.device_ms for _ in range(2)]
    on = [render(s, RenderConfig(cache_enabled=True, **base), ctx=ctx).stats.device_ms for _ in range(3)]
    print(name, "off", off, "on", on, flush=True)
    ctx.close()
