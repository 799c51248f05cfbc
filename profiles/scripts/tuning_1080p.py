"""Cache speed-up and hit rate of the Classroom-like analogue at the bench
size (1920x1080x128, 1e7 x 10 table) per uv layout and mip_offset: the
tunings SPEC acceptance #5 is checked at (profiles/scripts/fidelity_r2.py)
measured where the bench runs. Device time of one render each (CUDA events
on the render stream), median of `--reps`.

    python profiles/scripts/tuning_1080p.py [--kinds classroom] > out.json
"""
import argparse
import json
import os
import statistics
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", default="classroom")
    ap.add_argument("--spans", default="0,0.999")
    ap.add_argument("--mips", default="0,1,2,3")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--spp", type=int, default=128)
    args = ap.parse_args()
    W, H = 1920, 1080
    ctx = Context(0)
    tmp = tempfile.mkdtemp()
    rows = []
    for kind in args.kinds.split(","):
        for span in (float(x) for x in args.spans.split(",")):
            s = load_scene(scenes.build_scene(scenes.SceneSpec(kind, W, H, tris_per_side=24, uv_span=span),
                                              os.path.join(tmp, f"{kind}_{span}")))
            base = dict(width=W, height=H, spp=args.spp, n_cells=10_000_000, n_entries=10)
            render(s, RenderConfig(**base), ctx=ctx)
            t_off = statistics.median(render(s, RenderConfig(**base), ctx=ctx).stats.device_ms
                                      for _ in range(args.reps))
            for mip in (int(x) for x in args.mips.split(",")):
                rs = [render(s, RenderConfig(cache_enabled=True, mip_offset=mip, **base), ctx=ctx)
                      for _ in range(args.reps)]
                t_on = statistics.median(r.stats.device_ms for r in rs)
                row = {"kind": kind, "uv_span": span, "mip_offset": mip, "ms_no_cache": t_off, "ms_cache": t_on,
                       "speedup": t_off / t_on, "hit_rate": rs[-1].stats.hit_rate,
                       "inserts_won": rs[-1].stats.inserts_won,
                       "samples_per_s_cache": W * H * args.spp / (t_on / 1e3)}
                print(json.dumps(row), file=sys.stderr, flush=True)
                rows.append(row)
    print(json.dumps({"size": [W, H, args.spp], "table": "1e7x10", "rows": rows}))


if __name__ == "__main__":
    main()
