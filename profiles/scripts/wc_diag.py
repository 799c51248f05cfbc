"""Diagnostic: device time of consecutive renders in one context across
scene / tuning switches (is there a first-render penalty, and where)."""
import os
import sys
import tempfile

sys.path.insert(0, os.getcwd())
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render, scenes  # noqa: E402

bmw = load_scene(scenes.build_scene(scenes.SceneSpec("bmw", 1920, 1080, tris_per_side=24, uv_span=0.999),
                                    tempfile.mkdtemp()))
cls = load_scene(scenes.build_scene(scenes.SceneSpec("classroom", 1920, 1080, tris_per_side=24, uv_span=0.999,
                                                     libm_ops=True), tempfile.mkdtemp()))
ctx = Context(0)
seq = [("cls", 3, True), ("cls", 3, True), ("cls", 3, True), ("bmw", 24, True), ("bmw", 24, True),
       ("bmw", 24, True), ("bmw", 24, False), ("bmw", 24, False), ("bmw", 24, True), ("cls", 3, True),
       ("cls", 3, True), ("bmw", 3, True), ("bmw", 3, True), ("bmw", 24, True), ("bmw", 24, True)]
for name, mip, cache in seq:
    s = bmw if name == "bmw" else cls
    r = render(s, RenderConfig(width=1920, height=1080, spp=128, n_cells=10_000_000, n_entries=10, mip_offset=mip,
                               cache_enabled=cache), ctx=ctx)
    print(name, mip, cache, round(r.stats.device_ms, 1), round(r.stats.wall_time_s, 3), round(r.stats.hit_rate, 4),
          flush=True)
