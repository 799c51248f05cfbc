"""Projected N-GPU scaling from one GPU: the bench render split
into N tile shards (interleaved stripes or contiguous bands), each shard
rendered on its own fresh table replica -- one after another on this one GPU,
no shard waits on another -- and timed with CUDA events. The N-GPU render
takes max over shards (+ one framebuffer reduce over NVLink, ~75 MB);
hit rates show what each replica's smaller share of pixels costs."""
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render  # noqa: E402

ctx = Context(0)
scene = load_scene(bench.make_scene(tempfile.mkdtemp()))
base = dict(width=bench.W, height=bench.H, spp=bench.SPP, cache_enabled=True, n_cells=bench.N_CELLS,
            n_entries=bench.N_ENTRIES, mip_offset=bench.MIP_OFFSET)
render(scene, RenderConfig(**base), ctx=ctx)
full = render(scene, RenderConfig(**base), ctx=ctx)
t1 = full.stats.device_ms
out = {"one_gpu_ms": t1, "one_gpu_hit_rate": full.stats.hit_rate, "shards": {}}
print(f"1 GPU: {t1:.1f} ms, hit rate {full.stats.hit_rate:.4f}", flush=True)
for n in (2, 4, 8):
    for mode, name in ((0, "interleaved"), (1, "bands")):
        ts, hits, looks = [], 0, 0
        for r in range(n):
            res = render(scene, RenderConfig(**base, shard_rank=r, shard_count=n, shard_mode=mode), ctx=ctx)
            ts.append(res.stats.device_ms)
            hits += res.stats.hits
            looks += res.stats.lookups
        proj = max(ts)
        out["shards"][f"{n}_{name}"] = {"max_shard_ms": proj, "min_shard_ms": min(ts), "speedup": t1 / proj,
                                        "efficiency": t1 / proj / n, "hit_rate": hits / max(1, looks)}
        print(f"N={n} {name:11s}: max shard {proj:.1f} ms (min {min(ts):.1f}) -> projected speed-up "
              f"{t1 / proj:.2f}x ({t1 / proj / n * 100:.0f}%), hit rate {hits / max(1, looks):.4f}", flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "shard_projection.json"), "w") as f:
    json.dump(out, f, indent=1)
