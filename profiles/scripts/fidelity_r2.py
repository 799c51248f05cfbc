"""SPEC acceptance #5 with the reference beside the GPU, and the
concurrent-mode parity numbers of the timed path.

For each scene analogue x uv layout x mip_offset at 256x256x128:
  * GPU cache-off render (== oracle, bit-exact) = the uncached image;
  * GPU concurrent render (two pass lanes, several passes: the bench path);
  * the reference's own threaded CPU render (oracle/_ref, mode 2: the tile
    queue over every host thread with one shared MaterialCache), `--ref-runs`
    times;
and reports mean |d|, fraction of pixels with max-channel |d| < 0.05, RMSE,
hit rate, plus the SPEC.md:418/420 invariants of the GPU render.

    python profiles/scripts/fidelity_r2.py [--ref-runs 2] [--kinds classroom,...] > out.json
"""
import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import _oracle  # noqa: E402
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render, scenes  # noqa: E402


def metrics(img, off):
    d = np.abs(img.astype(np.float64) - off.astype(np.float64))
    return {"mean_abs": float(d.mean()), "frac_lt_0.05": float((d.max(-1) < 0.05).mean()),
            "rmse": float(np.sqrt((d ** 2).mean())), "max_abs": float(d.max())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref-runs", type=int, default=2)
    ap.add_argument("--gpu-runs", type=int, default=2)
    ap.add_argument("--kinds", default="classroom,junkshop,italianflat,monster,bmw,cornell")
    ap.add_argument("--spans", default="0,0.999")
    ap.add_argument("--mips", default="0,1,2")
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--spp", type=int, default=128)
    ap.add_argument("--nc", type=int, default=10_000_000)
    ap.add_argument("--ne", type=int, default=10)
    args = ap.parse_args()
    w = h = args.size
    spp = args.spp
    ctx = Context(0)
    ref = _oracle.Ref() if _oracle.Ref.available() else None
    threads = os.cpu_count() or 1
    tmp = tempfile.mkdtemp()
    out = {"size": [w, h, spp], "table": [args.nc, args.ne], "ref_threads": threads, "rows": []}
    for kind in args.kinds.split(","):
        for span in (float(x) for x in args.spans.split(",")):
            path = scenes.build_scene(scenes.SceneSpec(kind, w, h, tris_per_side=24, libm_ops=True,
                                                       uv_span=span), os.path.join(tmp, f"{kind}_{span}"))
            s = load_scene(path)
            off = render(s, RenderConfig(width=w, height=h, spp=spp), ctx=ctx)
            off_img = off.frame.radiance_image()
            t_off = off.stats.device_ms
            rs = ref.scene_load(path) if ref else None
            for mip in (int(x) for x in args.mips.split(",")):
                row = {"kind": kind, "uv_span": span, "mip_offset": mip, "gpu_ms_off": t_off, "gpu": [], "ref": []}
                for _ in range(args.gpu_runs):
                    r = render(s, RenderConfig(width=w, height=h, spp=spp, cache_enabled=True, n_cells=args.nc,
                                               n_entries=args.ne, mip_offset=mip), ctx=ctx)
                    m = metrics(r.frame.radiance_image(), off_img)
                    zero = r.frame.nodes_found == 0
                    m.update({"hit_rate": r.stats.hit_rate, "ms": r.stats.device_ms,
                              "zero_hit_pixels": int(zero.sum()),
                              "zero_hit_bit_identical": bool(np.array_equal(
                                  r.frame.radiance[zero].view(np.uint64), off.frame.radiance[zero].view(np.uint64))),
                              "hits_eq_sum_nodes": int(r.stats.hits) == int(r.frame.nodes_found.sum())
                              == int(sum(r.stats.hits_per_sample))})
                    row["gpu"].append(m)
                for _ in range(args.ref_runs if ref else 0):
                    P = _oracle.RenderParamsC(w, h, spp, 4, 2, mip, args.nc, args.ne, 0, 1, 0.2, 16, 0, 1, 0,
                                              threads, 1)
                    t0 = time.perf_counter()
                    rad, nodes, samples, hps, st = ref.render(rs, P, w, h)
                    dt = time.perf_counter() - t0
                    img = (rad / np.maximum(samples, 1)[..., None]).astype(np.float32)
                    m = metrics(img, off_img)
                    m.update({"hit_rate": st.hits / max(1, st.lookups), "s": dt})
                    row["ref"].append(m)
                print(json.dumps(row), file=sys.stderr, flush=True)
                out["rows"].append(row)
            if rs:
                ref.L.ref_scene_free(rs)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
