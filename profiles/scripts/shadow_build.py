"""Shadow-tree build on the host vs on the device (csrc/mcg_build.cu, SURVEY
§8f.4): scene upload time per builder (the upload includes the 4-wide
collapse of the reference tree, the shadow tree and the transposes), and the
shadow traversal of a 1920x1080x8 cache-off render with each tree (node
visits must be equal: it is the same tree). Classroom analogue at growing
tessellation. Run on a GPU box."""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render, scenes  # noqa: E402

rows = []
for tps in (24, 96, 300):
    s = load_scene(scenes.build_scene(scenes.SceneSpec("classroom", 1920, 1080, tris_per_side=tps),
                                      tempfile.mkdtemp()))
    row = {"tris_per_side": tps, "prims": s.flat.n_prims, "ref_nodes": s.flat.n_nodes}
    for mode in ("host", "device", "host", "device"):
        os.environ["MCG_SHADOW_BUILD"] = mode
        ctx = Context(0)
        t0 = time.perf_counter()
        ctx.upload(s)
        t_up = time.perf_counter() - t0
        render(s, RenderConfig(width=1920, height=1080, spp=8), ctx=ctx)   # warm-up (allocations)
        r = render(s, RenderConfig(width=1920, height=1080, spp=8), ctx=ctx)
        row[mode] = {"upload_s": t_up, "render_ms": r.stats.device_ms,
                     "shadow_nodes": r.stats.bvh_nodes_shadow, "shadow_prims": r.stats.prims_tested_shadow}
        ctx.close()
    print(json.dumps(row), flush=True)
    rows.append(row)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/shadow_build.json", "w") as f:
    json.dump(rows, f, indent=1)
