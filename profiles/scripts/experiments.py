"""Round experiments on one B200 (SURVEY §8d configurations C1-C5 and the
SPEC acceptance criteria 5-7), written to profiles/experiments_r1.json,
profiles/sweep_c2_classroom.csv, profiles/sweep_a6_noise_gallery.csv and the
figure artefacts under profiles/figs/.

    python profiles/scripts/experiments.py [--quick]

All renders go through the public Python API (paper_2305_07238_b200.render);
times are the renders' CUDA-event times (RenderStats.device_ms). The CPU
reference (oracle/_ref) is timed for C1 only, on the box's host cores."""
import argparse
import json
import os
import statistics
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from paper_2305_07238_b200 import (Context, RenderConfig, artifacts, image_error, load_scene,  # noqa: E402
                                   render, scenes, stats_to_json, sweep, write_sweep_csv)

OUT = os.path.join(ROOT, "profiles")
FIGS = os.path.join(OUT, "figs")


PATHS = {}


UV_SPAN = 0.0   # --uv-span: 0 = tiled uv (round 1), 0.999 = one uv tile per surface (round-2 bench)


def build(kind, w, h, tmp, tps=24, seed=0):
    path = scenes.build_scene(scenes.SceneSpec(kind, w, h, seed=seed, tris_per_side=tps, uv_span=UV_SPAN),
                              os.path.join(tmp, f"{kind}_{w}x{h}_{tps}"))
    s = load_scene(path)
    PATHS[id(s)] = path
    return s


def timed(scene, cfg, ctx, reps=1):
    ts, last = [], None
    for _ in range(reps):
        last = render(scene, cfg, ctx=ctx)
        ts.append(last.stats.device_ms)
    return statistics.median(ts), last


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="smaller sizes (smoke run)")
    ap.add_argument("--uv-span", type=float, default=0.0)
    ap.add_argument("--mip", type=int, default=0, help="mip_offset of the cached C2/C3/C5 renders")
    ap.add_argument("--sections", default="C1,C3,C2,C5,A5,A6,A7")
    ap.add_argument("--out", default=None, help="output JSON (default profiles/experiments_r1.json)")
    args = ap.parse_args()
    global UV_SPAN
    UV_SPAN = args.uv_span
    sections = set(args.sections.split(","))
    q = args.quick
    os.makedirs(FIGS, exist_ok=True)
    tmp = tempfile.mkdtemp()
    ctx = Context(0)
    res = {"device": "B200 (1 GPU)", "timing": "CUDA events per render (RenderStats.device_ms)"}
    W, H = (480, 270) if q else (1920, 1080)

    # ---- C1: 256x256x4, depth-8 graph, cache 1e5x10, GPU vs reference CPU ----
    if "C1" in sections:
        import _oracle
        sc = build("cornell", 256, 256, tmp, tps=8)
        cfg = RenderConfig(width=256, height=256, spp=4, cache_enabled=True, n_cells=100_000, n_entries=10)
        render(sc, cfg, ctx=ctx)
        ms, r = timed(sc, cfg, ctx, 5)
        c1 = {"gpu_ms": ms, "gpu_samples_per_s": 256 * 256 * 4 / (ms / 1e3), "hit_rate": r.stats.hit_rate}
        off = render(sc, RenderConfig(width=256, height=256, spp=4), ctx=ctx).frame.radiance
        if _oracle.Ref.available():
            ref = _oracle.Ref()
            rs = ref.scene_load(PATHS[id(sc)])
            nthreads = os.cpu_count() or 1
            P = _oracle.RenderParamsC(256, 256, 4, 4, 0, 0, 100_000, 10, 0, 1, 0.2, 16, 0, 1, 0, nthreads, 1)
            t0 = time.perf_counter()
            rad_ref, *_ = ref.render(rs, P, 256, 256)
            c1["ref_cpu_cache_off_s"] = time.perf_counter() - t0
            d = np.abs(rad_ref - off) / np.maximum(np.abs(rad_ref), 1e-30)
            c1["cache_off_max_rel_diff_vs_reference"] = float(d.max())
            P.mode = 2
            t0 = time.perf_counter()
            ref.render(rs, P, 256, 256)
            dt = time.perf_counter() - t0
            c1.update({"ref_cpu_cache_on_s": dt, "ref_cpu_samples_per_s": 256 * 256 * 4 / dt,
                       "ref_cpu_threads": P.threads})
        res["C1"] = c1
        print("C1", c1, flush=True)

    # ---- C3/C4: five analogues at WxHx128, cache 1e7x10 vs no cache ----
    if "C3" in sections:
        c3 = {}
        for kind in ("classroom", "junkshop", "italianflat", "monster", "bmw", "hostile"):
            s = build(kind, W, H, tmp)
            base = RenderConfig(width=W, height=H, spp=128 if not q else 8, n_cells=10_000_000, n_entries=10)
            render(s, base, ctx=ctx)
            t_off, _ = timed(s, base, ctx, 3)
            on = RenderConfig(**{**base.__dict__, "cache_enabled": True, "mip_offset": args.mip})
            t_on, r = timed(s, on, ctx, 3)
            n = W * H * base.spp
            c3[kind] = {"ms_no_cache": t_off, "ms_cache": t_on, "speedup": t_off / t_on,
                        "relative_time_pct": 100 * t_on / t_off, "samples_per_s_cache": n / (t_on / 1e3),
                        "hit_rate": r.stats.hit_rate, "inserts_won": r.stats.inserts_won,
                        "inserts_lost_full": r.stats.inserts_lost_full}
            print("C3", kind, c3[kind], flush=True)
        res["C3_C4"] = c3

    # ---- C2: classroom WxHx32 sweep Nc x Ne ----
    if "C2" in sections:
        s = build("classroom", W, H, tmp)
        rows = sweep(s, RenderConfig(width=W, height=H, spp=32 if not q else 4, mip_offset=args.mip),
                     [100_000, 1_000_000, 10_000_000], [2, 4, 6, 8, 10], repeats=1, ctx=ctx)
        write_sweep_csv(rows, os.path.join(os.path.dirname(args.out) if args.out else OUT, "sweep_c2_classroom.csv"))
        res["C2"] = [r.__dict__ for r in rows]
        print("C2 done", flush=True)

    # ---- C5: classroom 3840x2160x512 on one GPU ----
    if "C5" in sections:
        if not q:
            s5 = build("classroom", 3840, 2160, tmp)
            cfg5 = RenderConfig(width=3840, height=2160, spp=512, cache_enabled=True,
                                n_cells=10_000_000, n_entries=10, mip_offset=args.mip)
            ms5, r5 = timed(s5, cfg5, ctx, 1)
            res["C5"] = {"ms": ms5, "samples_per_s": 3840 * 2160 * 512 / (ms5 / 1e3),
                         "hit_rate": r5.stats.hit_rate, "n_gpus": 1}
            print("C5", res["C5"], flush=True)

    # ---- A5: image fidelity at 256x256x128, mip offsets 0/1/2 ----
    if "A5" in sections:
        a5 = {}
        for kind in ("classroom", "junkshop", "italianflat", "monster", "bmw", "cornell"):
            s = build(kind, 256, 256, tmp, tps=12)
            off = render(s, RenderConfig(width=256, height=256, spp=128), ctx=ctx).frame.radiance_image()
            row = {}
            for mo in (0, 1, 2):
                on = render(s, RenderConfig(width=256, height=256, spp=128, cache_enabled=True,
                                            n_cells=10_000_000, n_entries=10, mip_offset=mo),
                            ctx=ctx)
                img = on.frame.radiance_image()
                d = image_error(img, off)
                px = np.abs(img - off).max(axis=2)
                row[f"mip{mo}"] = {"mean_abs": d.mean_abs, "max_abs": d.max_abs,
                                   "frac_pixels_below_0.05": float((px < 0.05).mean()),
                                   "hit_rate": on.stats.hit_rate}
                if kind == "classroom" and mo == 0:
                    artifacts.write_ppm(os.path.join(FIGS, "classroom_cached.ppm"), img, True)
                    artifacts.write_ppm(os.path.join(FIGS, "classroom_uncached.ppm"), off, True)
                    artifacts.write_diff(img, off, os.path.join(FIGS, "classroom_diff_x5.ppm"))
                    artifacts.write_heatmap(stats_to_json(on.stats, on.frame),
                                            os.path.join(FIGS, "classroom_hits_heatmap.ppm"))
            row["criterion5"] = bool(row["mip0"]["mean_abs"] <= 0.01 and
                                     row["mip0"]["frac_pixels_below_0.05"] >= 0.99 and
                                     row["mip2"]["mean_abs"] <= row["mip0"]["mean_abs"])
            a5[kind] = row
            print("A5", kind, row, flush=True)
        res["A5_image_fidelity"] = a5

    # ---- A6: cache-size trend on the heavy procedural scene ----
    if "A6" in sections:
        s = build("classroom", 256, 256, tmp, tps=12)
        rows = sweep(s, RenderConfig(width=256, height=256, spp=128), [1_000, 10_000, 100_000, 1_000_000],
                     [2, 10], ctx=ctx)
        write_sweep_csv(rows, os.path.join(OUT, "sweep_a6_noise_gallery.csv"))
        hr = {(r.n_cells, r.n_entries): r.hit_rate for r in rows}
        cells = sorted({r.n_cells for r in rows})
        mono = all(hr[(cells[i], e)] <= hr[(cells[i + 1], e)] for e in (2, 10) for i in range(len(cells) - 1))
        ent = all(hr[(c, 10)] >= hr[(c, 2)] for c in cells)
        sat = abs(hr[(cells[-1], 10)] - hr[(cells[-2], 10)]) < 0.01
        res["A6_cache_size_trend"] = {"rows": [r.__dict__ for r in rows], "hit_rate_nondecreasing_in_cells": mono,
                                      "entries10_ge_entries2": ent, "saturated_top_step": sat}
        print("A6", res["A6_cache_size_trend"]["hit_rate_nondecreasing_in_cells"], ent, sat, flush=True)

    # ---- A7: speed-up direction (median of 3) ----
    if "A7" in sections:
        a7 = {}
        for kind in ("classroom", "hostile"):
            s = build(kind, W, H, tmp)
            base = RenderConfig(width=W, height=H, spp=128 if not q else 8, n_cells=10_000_000, n_entries=10)
            render(s, base, ctx=ctx)
            t_off, _ = timed(s, base, ctx, 3)
            t_on, _ = timed(s, RenderConfig(**{**base.__dict__, "cache_enabled": True, "mip_offset": args.mip}),
                            ctx, 3)
            a7[kind] = {"relative_time_pct": 100 * t_on / t_off}
        a7["criterion7"] = bool(a7["classroom"]["relative_time_pct"] <= 95 and
                                a7["hostile"]["relative_time_pct"] <= 103)
        res["A7_speedup_direction"] = a7
        print("A7", a7, flush=True)

    res["tuning"] = {"uv_span": args.uv_span, "mip_offset": args.mip}
    out = args.out or os.path.join(OUT, "experiments_r1.json" if not q else "experiments_quick.json")
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
