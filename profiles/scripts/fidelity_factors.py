"""Which part of the concurrent schedule moves the cached image's error
(cached vs uncached RMSE / mean |d|)? One scene, one table, the reference's
threaded and epoch-sequential renders beside GPU renders under different
schedules: pass lanes (MCG_LANES), samples per pass, the wavefront sort key
(MCG_SORT), deterministic mode.

    python profiles/scripts/fidelity_factors.py --kind italianflat --span 0 --mip 0
"""
import argparse
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import _oracle  # noqa: E402
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render, scenes  # noqa: E402


def metrics(img, off):
    d = np.abs(img.astype(np.float64) - off.astype(np.float64))
    return {"mean_abs": round(float(d.mean()), 5), "frac_lt_0.05": round(float((d.max(-1) < 0.05).mean()), 4),
            "rmse": round(float(np.sqrt((d ** 2).mean())), 5)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="italianflat")
    ap.add_argument("--span", type=float, default=0.0)
    ap.add_argument("--mip", type=int, default=0)
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--spp", type=int, default=128)
    ap.add_argument("--ref-runs", type=int, default=2)
    args = ap.parse_args()
    w = h = args.size
    spp, nc, ne = args.spp, 10_000_000, 10
    ctx = Context(0)
    tmp = tempfile.mkdtemp()
    path = scenes.build_scene(scenes.SceneSpec(args.kind, w, h, tris_per_side=24, libm_ops=True,
                                               uv_span=args.span), os.path.join(tmp, "s"))
    s = load_scene(path)
    off = render(s, RenderConfig(width=w, height=h, spp=spp), ctx=ctx).frame.radiance_image()
    out = {"kind": args.kind, "span": args.span, "mip": args.mip, "rows": []}

    def gpu(label, env=None, **kw):
        saved = {k: os.environ.get(k) for k in (env or {})}
        os.environ.update(env or {})
        try:
            r = render(s, RenderConfig(width=w, height=h, spp=spp, cache_enabled=True, n_cells=nc, n_entries=ne,
                                       mip_offset=args.mip, **kw), ctx=ctx)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        m = metrics(r.frame.radiance_image(), off)
        m.update({"who": "gpu", "label": label, "hit_rate": round(r.stats.hit_rate, 4)})
        print(json.dumps(m), file=sys.stderr, flush=True)
        out["rows"].append(m)

    for rep in range(2):
        gpu(f"default#{rep}")
    gpu("lanes1", {"MCG_LANES": "1"})
    gpu("sort_material", {"MCG_SORT": "material"})
    gpu("sort_material_lanes1", {"MCG_SORT": "material", "MCG_LANES": "1"})
    for k in (1, 4, 8):
        gpu(f"spp_pass{k}", samples_per_pass=k)
        gpu(f"spp_pass{k}_lanes1", {"MCG_LANES": "1"}, samples_per_pass=k)
    for k in (1, 8):
        gpu(f"deterministic_k{k}", deterministic=True, samples_per_pass=k)
    if _oracle.Ref.available():
        ref = _oracle.Ref()
        rs = ref.scene_load(path)
        threads = os.cpu_count() or 1
        for mode, k, runs in ((2, 1, args.ref_runs), (1, 1, 1), (1, 32, 1), (3, 1, 1)):
            for rep in range(runs):
                P = _oracle.RenderParamsC(w, h, spp, 4, mode, args.mip, nc, ne, 0, 1, 0.2, 16, 0, 1, 0, threads, k)
                rad, nodes, samples, hps, st = ref.render(rs, P, w, h)
                img = (rad / np.maximum(samples, 1)[..., None]).astype(np.float32)
                m = metrics(img, off)
                m.update({"who": "ref", "label": f"mode{mode}_k{k}#{rep}", "hit_rate": round(st.hits / max(1, st.lookups), 4)})
                print(json.dumps(m), file=sys.stderr, flush=True)
                out["rows"].append(m)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
