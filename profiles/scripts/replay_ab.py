"""Trace replay A/B (same call): the bench render's first 2^26 lookups through
a fresh 1e7x10 table, software-pipelined vs not, several blocks/SM."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2305_07238_b200 import Context, MaterialCache, RenderConfig, load_scene, scenes  # noqa: E402
from paper_2305_07238_b200 import _native as N  # noqa: E402

ctx = Context(0)
path = scenes.build_scene(scenes.SceneSpec("classroom", 1920, 1080), "/tmp/replay_ab")
s = load_scene(path)
ctx.upload(s)
cfg = RenderConfig(width=1920, height=1080, spp=16, cache_enabled=True, n_cells=10_000_000, n_entries=10)
t = MaterialCache(10_000_000, 10, ctx)
t.trace_start(1 << 26)
from paper_2305_07238_b200 import render  # noqa: E402
render(s, cfg, external_cache=t, ctx=ctx)
n = t.trace_stop()
tr = t.trace_read(0, n)
t.close()
f = MaterialCache(10_000_000, 10, ctx)
for bps in (8, -8, 4, -4, 6, 12):
    best = None
    for rep in range(3):
        f.clear()
        ms, by, c = f.probe_replay(tr, bps)
        best = ms if best is None else min(best, ms)
    print(f"bps {bps:3d}: {n / best / 1e6:6.1f} G/s  {by / best / 1e6:6.0f} GB/s ({by / best / 1e6 / 6547.5:.3f}) "
          f"hit {c['hits'] / c['lookups']:.4f}", flush=True)
