"""Cached-vs-uncached error of the bench band (tiles 8/16 of the bench frame,
contiguous) per insert schedule: GPU concurrent mode at several samples per
pass and lane counts, GPU deterministic mode, and the reference's own code
(oracle/_ref) in its threaded tile-queue order (mode 2), the wavefront order
with immediate inserts (mode 1) and the deferred order (mode 3).

    python profiles/scripts/order_rmse.py [--spp 32] [--ref] > out.json
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

import bench  # noqa: E402
from paper_2305_07238_b200 import Context, RenderConfig, load_scene, render  # noqa: E402


def err(img, off):
    d = np.abs(img.astype(np.float64) - off.astype(np.float64))
    return {"rmse": float(np.sqrt((d ** 2).mean())), "mean_abs": float(d.mean()),
            "p999_abs": float(np.quantile(d.max(-1), 0.999)), "max_abs": float(d.max())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spp", type=int, default=32)
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--gpu", default="1:2,1:1,2:2,4:2,8:2,32:1,32:2,det1,det32")
    args = ap.parse_args()
    W, H, spp = bench.W, bench.H, args.spp
    NC, NE = bench.N_CELLS, bench.N_ENTRIES
    path = bench.make_scene(tempfile.mkdtemp())
    band = dict(width=W, height=H, spp=spp, n_cells=NC, n_entries=NE, shard_rank=bench.CPU_BAND,
                shard_count=bench.CPU_BANDS, shard_mode=1, mip_offset=bench.MIP_OFFSET)
    rows = []
    s = load_scene(path)
    ctx = Context(0)
    off = render(s, RenderConfig(**band, samples_per_pass=1), ctx=ctx)
    mask = off.frame.samples > 0
    off_img = off.frame.radiance_image()[mask]
    np.save(os.path.join(ROOT, "gpurun_out", "order_off.npy"), off_img)
    for spec in args.gpu.split(","):
        det = spec.startswith("det")
        if det:
            k, lanes = int(spec[3:]), "1"
        else:
            k, lanes = spec.split(":")
            k = int(k)
        os.environ["MCG_LANES"] = lanes
        r = render(s, RenderConfig(cache_enabled=True, deterministic=det, samples_per_pass=k, **band), ctx=ctx)
        e = err(r.frame.radiance_image()[mask], off_img)
        e.update({"impl": "gpu", "spec": spec, "hit_rate": r.stats.hit_rate, "ms": r.stats.device_ms})
        print(json.dumps(e), file=sys.stderr, flush=True)
        rows.append(e)
    os.environ.pop("MCG_LANES", None)
    if args.ref:
        import _oracle
        ref = _oracle.Ref()
        rs = ref.scene_load(path)
        threads = os.cpu_count() or 1
        for name, mode, k, th in [("threaded", 2, 1, threads), ("wavefront_k1", 1, 1, 1),
                                  ("wavefront_k32", 1, 32, 1), ("deferred_k1", 3, 1, 1)]:
            p = _oracle.RenderParamsC(W, H, spp, 4, mode, bench.MIP_OFFSET, NC, NE, 0, 1, 0.2, 16,
                                      bench.CPU_BAND, bench.CPU_BANDS, 1, th, k)
            rad, nodes, samples, hps, st = ref.render(rs, p, W, H)
            img = (rad / np.maximum(samples, 1)[..., None]).astype(np.float32)[mask]
            e = err(img, off_img)
            e.update({"impl": "reference", "spec": name, "hit_rate": st.hits / max(1, st.lookups)})
            print(json.dumps(e), file=sys.stderr, flush=True)
            rows.append(e)
    print(json.dumps({"band": [bench.CPU_BAND, bench.CPU_BANDS], "spp": spp, "rows": rows}))


if __name__ == "__main__":
    main()
