"""Benchmark of the progressive-material-cache hot path (BASELINE.json metric:
samples/sec at 1920x1080 128spp + cache speed-up + HBM% on probes).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one render() of the Classroom-like analogue at 1920x1080x128spp
with a fresh 1e7 x 10 table (tracer.hpp:67-68; configs[2] of BASELINE.json,
paper's cache size), concurrent inserts (the paper's single-CAS policy). The
image is tile-sharded across ranks (torchrun, one process per GPU, NCCL
reduce of the framebuffers to rank 0 inside each step): total work is fixed,
so scaling is strong.

Printed JSON line (rank 0):
  value        samples/s, device-timed (CUDA events on the render stream,
               max over ranks), inputs resident in HBM
  e2e          the same metric through the C ABI's host-buffer entry point
               (mcg_upload_scene + mcg_render with pinned host framebuffers):
               scene H2D + framebuffer H2D/D2H inside the timed region
  roofline     dominant kernel's compulsory HBM bytes / its CUDA-event time vs
               the measured HBM peak (MEASURED_PEAKS.json), the ncu DRAM
               traffic per launch, and the L1/L2-served BVH/triangle bytes
  roofline_shade  the same for the material-VM + cache-probe kernel
  probe_roofline  the cache-probe kernel on the 1e7 x 10 table (HBM-bound)
  cache_speedup   t(no cache) / t(cache) on the same workload
  cpu_baseline the reference's own CPU path (oracle/_ref) on the host cores
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

W, H, SPP = 1920, 1080, 128
N_CELLS, N_ENTRIES = 10_000_000, 10
SCENE_KIND = "classroom"
TRIS_PER_SIDE = 24
# The tuning SPEC acceptance #5 holds at for the reference
# itself (profiles/README.md "SPEC #5"): one uv tile per surface (no
# wrapped texels shared across a wall) and mip_offset 3 (texels 1/8 of the
# pixel footprint, "offsetting the mipmap level ... a bit more accurate
# result", PAPER.md). The tiled-uv, offset-0 layout of round 1 is faster
# (hit rate 0.998) but fails SPEC #5 for the reference as well; bench.py
# reports it beside (`tunings`).
UV_SPAN, MIP_OFFSET = 0.999, 3
PROBE_VARIANT, PROBE_BLOCKS_PER_SM = 10, 8         # HBM table: warp-cooperative one-round-trip loads, software-pipelined, scan through shared memory
PROBE_L2_VARIANT, PROBE_L2_BLOCKS_PER_SM = 0, 8    # L2-resident table: per-lane scan (issue-bound)
METRIC = "samples/sec at 1920x1080 128spp (classroom-like, cache 1e7x10)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.rows: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    # control-flow check of the N > 1 path on a one-GPU box (never a
    # measurement): every rank on cuda:0, gloo instead of NCCL
    if os.environ.get("MCG_BENCH_SAME_DEVICE") == "1":
        local = 0
    return rank, world, local


def frame_reduce(dist, tensors):
    """Framebuffer gather to rank 0: reduce(sum) over NCCL (exact: each pixel
    belongs to one rank, the others contribute zeros). With the gloo
    control-flow backend (CUDA tensors support all_reduce only) an
    all_reduce stands in."""
    for t in tensors:
        if dist.get_backend() == "gloo":
            dist.all_reduce(t)
        else:
            dist.reduce(t, 0)


def make_scene(tmp: str):
    from paper_2305_07238_b200 import scenes
    return scenes.build_scene(scenes.SceneSpec(SCENE_KIND, W, H, tris_per_side=TRIS_PER_SIDE,
                                               libm_ops=True, uv_span=UV_SPAN), os.path.join(tmp, "scene"))


# --------------------------------------------------------------------------
# reference arm: the reference's own CPU path on the host cores
# --------------------------------------------------------------------------

# The CPU leg renders the same workload (same scene, camera, 128 spp, 1e7 x
# 10 table, concurrent shared-table inserts) on a band of it: contiguous
# 16x16 tiles 8/16 of the frame (shard_mode 1, rank 8 of 16: a ~1920x68
# band through the middle of the image), so samples/s is like for like in
# spp and in table fill; the full frame would take ~3 min per step. The
# table (MaterialCache(1e7, 10): 800 MB zeroed, cache.cpp:82-92) is built
# before the timer and reported apart (`table_build_s`).
CPU_BAND, CPU_BANDS = 8, 16


def cpu_reference_sample(scene_path: str, threads: int = 0, cache: bool = True, seed: int = 1):
    """Times oracle/_ref's render (reference sources + restated tracer, tile
    queue over worker threads, shared MaterialCache) on a bounded sample:
    a 1/16 band of the 1920x1080x128 frame."""
    import _oracle
    nthreads = threads or os.cpu_count() or 1
    if _oracle.Ref.available():
        ref = _oracle.Ref()
        s = ref.scene_load(scene_path)
        P = _oracle.RenderParamsC(W, H, SPP, 4, 2 if cache else 0, MIP_OFFSET, N_CELLS, N_ENTRIES, 0, seed,
                                  0.2, 16, CPU_BAND, CPU_BANDS, 1, nthreads, 1)
        t0 = time.perf_counter()
        c = ref.cache_new(N_CELLS, N_ENTRIES) if cache else None
        t_table = time.perf_counter() - t0
        t0 = time.perf_counter()
        rad, _, samples, _, st = ref.render(s, P, W, H, cache=c)
        dt = time.perf_counter() - t0
        if c is not None:
            ref.cache_free(c)
        ref.L.ref_scene_free(s)
        return {"kind": "reference", "seconds": dt, "samples": int(samples.sum()), "cores": nthreads,
                "hits": int(st.hits), "lookups": int(st.lookups), "table_build_s": t_table,
                "radiance": rad, "pixel_samples": samples, "seed": seed}
    # Fallback: the C restatement (single thread) on a 1/64 band.
    from paper_2305_07238_b200 import load_scene
    orc = _oracle.Oracle()
    sc = load_scene(scene_path)
    P = _oracle.RenderParamsC(W, H, SPP, 4, 1 if cache else 0, MIP_OFFSET, N_CELLS, N_ENTRIES, 0, 1,
                              0.2, 16, 32, 64, 1, 1, 1)
    t0 = time.perf_counter()
    _, _, samples, _, _ = orc.render(sc.flat, P)
    dt = time.perf_counter() - t0
    return {"kind": "port", "seconds": dt, "samples": int(samples.sum()), "cores": 1, "table_build_s": None}


def cpu_sample_text(info) -> str:
    if info["kind"] == "reference":
        return (f"tiles {CPU_BAND}/{CPU_BANDS} of the {W}x{H}x{SPP}spp frame as one contiguous band "
                f"({info['samples'] // SPP} pixels x {SPP} spp), concurrent inserts into a fresh "
                f"{N_CELLS:.0e}x{N_ENTRIES} MaterialCache per step (built before the timer: "
                f"{info['table_build_s']:.2f} s), tile queue over {info['cores']} threads")
    return f"1/64 band of the {W}x{H}x{SPP}spp frame, 1 thread (C port)"


def run_reference_arm(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    with tempfile.TemporaryDirectory() as tmp:
        path = make_scene(tmp)
        for _ in range(args.warmup):
            cpu_reference_sample(path)
        times = []
        info = None
        for _ in range(args.steps):
            info = cpu_reference_sample(path)
            times.append(info["seconds"])
    t = sum(times) / len(times)
    v = info["samples"] / t
    sample = cpu_sample_text(info)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded classroom-like scene, reference JSON/PPM formats)",
        "config": {"workload": f"{SCENE_KIND}-like {W}x{H} {SPP}spp cache {N_CELLS:.0e}x{N_ENTRIES}, "
                               f"unit uv, mip_offset {MIP_OFFSET}", "sample": sample},
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": info["cores"],
                         "kind": info["kind"], "sample": sample,
                         "table_build_s": info.get("table_build_s"),
                         "hit_rate": info["hits"] / max(1, info["lookups"]) if "hits" in info else None},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def parity_block(frame_cached, frame_off, st, ref_runs, gpu_bands) -> dict:
    import numpy as np
    rad_c, nodes_c, samp_c = frame_cached
    n = np.maximum(samp_c, 1)[..., None].astype(np.float64)
    img_c = (rad_c / n).astype(np.float32)
    img_off = (frame_off / n).astype(np.float32)

    def err(a, b, mask=None):
        d = np.abs(a.astype(np.float64) - b.astype(np.float64))
        if mask is not None:
            d = d[mask]
        return {"rmse": float(np.sqrt((d ** 2).mean())), "mean_abs": float(d.mean())}

    zero = nodes_c == 0
    out = {"config": "the timed render (concurrent inserts, two pass lanes) vs the cache-off render",
           "frame": err(img_c, img_off),
           "zero_hit_pixels": int(zero.sum()),
           "zero_hit_pixels_bit_identical": bool(np.array_equal(rad_c[zero].view(np.uint64),
                                                               frame_off[zero].view(np.uint64))),
           "hits_eq_sum_nodes_found": int(st.hits) == int(nodes_c.sum())}
    if ref_runs and all(r.get("radiance") is not None for r in ref_runs):
        # like for like: the reference rendered one band of tiles with its
        # own table (cpu_baseline, one run per RNG seed); the GPU renders the
        # same band the same way, cached (concurrent) and uncached, per seed.
        # Which sample first inserts a texel is a race in both renderers and
        # the RMSE is carried by a few bright pixels, so one seed is one draw
        # (the reference's own spread reaches ~7%): the north_star bound is
        # checked on the mean over the seeds, with two standard errors of the
        # per-seed differences as the noise allowance.
        import statistics
        seeds, diffs = [], []
        zero_ok, zero_n = True, 0
        for r, (gc, goff) in zip(ref_runs, gpu_bands):
            band = r["pixel_samples"] > 0
            assert np.array_equal(band, gc.samples > 0)
            goff_img = goff.radiance_image()
            rimg = (r["radiance"] / np.maximum(r["pixel_samples"], 1)[..., None]).astype(np.float32)
            gpu = err(gc.radiance_image(), goff_img, band)
            ref = err(rimg, goff_img, band)
            gz = (gc.nodes_found == 0) & band
            zero_n += int(gz.sum())
            zero_ok = zero_ok and bool(np.array_equal(gc.radiance[gz].view(np.uint64),
                                                      goff.radiance[gz].view(np.uint64)))
            seeds.append({"seed": r["seed"], "gpu": gpu, "reference": ref})
            diffs.append(gpu["rmse"] - ref["rmse"])
        mean = statistics.mean(diffs)
        se = statistics.stdev(diffs) / len(diffs) ** 0.5 if len(diffs) > 1 else 0.0
        out["band"] = {"pixels": int((ref_runs[0]["pixel_samples"] > 0).sum()),
                       "what": cpu_sample_text(ref_runs[0]), "per_seed": seeds,
                       "mean_rmse_gpu": statistics.mean(x["gpu"]["rmse"] for x in seeds),
                       "mean_rmse_reference": statistics.mean(x["reference"]["rmse"] for x in seeds),
                       "mean_diff": mean, "se_diff": se,
                       "bound": "mean over seeds of (gpu rmse - reference rmse) <= 1e-4 + 2 SE (north_star)",
                       "within_bound": mean <= 1e-4 + 2.0 * se,
                       "zero_hit_pixels": zero_n, "zero_hit_pixels_bit_identical": zero_ok}
    return out


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip speed-up/probe legs")
    ap.add_argument("--shared-cache", action="store_true",
                    help="N>1: one table striped over the GPUs (SURVEY 8f.3) instead of per-GPU replicas")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("MCG_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2305_07238_b200 import (Context, RenderConfig, load_scene)
    from paper_2305_07238_b200 import _native as N

    stream = torch.cuda.Stream()
    ctx = Context(local, profile=True, stream=stream.cuda_stream)
    L = N.lib()
    tmp = tempfile.mkdtemp()
    scene_path = make_scene(tmp) if rank == 0 else None
    if world > 1:
        obj = [tmp if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        scene_path = os.path.join(obj[0], "scene", "scene.json")
        if rank != 0:  # same seeded generator -> byte-identical files
            scene_path = make_scene(tempfile.mkdtemp())
    scene = load_scene(scene_path)
    ctx.upload(scene)

    cfg = RenderConfig(width=W, height=H, spp=SPP, cache_enabled=True, n_cells=N_CELLS,
                       n_entries=N_ENTRIES, mip_offset=MIP_OFFSET, shard_rank=rank, shard_count=world,
                       shard_mode=0)
    params = cfg.to_params()
    dev = torch.device("cuda", local)
    rad = torch.zeros(H * W * 3, dtype=torch.float64, device=dev)
    nodes = torch.zeros(H * W, dtype=torch.float64, device=dev)
    samples = torch.zeros(H * W, dtype=torch.int32, device=dev)
    dframe = N.Frame(C.cast(C.c_void_p(rad.data_ptr()), C.POINTER(C.c_double)),
                     C.cast(C.c_void_p(nodes.data_ptr()), C.POINTER(C.c_double)),
                     C.cast(C.c_void_p(samples.data_ptr()), C.POINTER(C.c_uint32)))

    shared = None
    if args.shared_cache and world > 1:
        from paper_2305_07238_b200 import dist as D
        shared = D.shared_cache(N_CELLS, N_ENTRIES, ctx, rank, world)

    def step(p=params):
        with torch.cuda.stream(stream):
            rad.zero_(); nodes.zero_(); samples.zero_()
        st = N.RenderStats()
        ext = None
        if shared is not None and p.cache_mode != 0:
            shared.clear()            # a fresh logical table per render, like the replicas
            ctx.synchronize()
            dist.barrier()
            ext = shared.handle
        N.check(L.mcg_render_device(ctx.handle, C.byref(p), ext, C.byref(dframe), C.byref(st)))
        if world > 1:
            with torch.cuda.stream(stream):
                frame_reduce(dist, [rad, nodes, samples])
        return st

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ctx.reset_kernel_times()
        l0 = ctx.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        stats = [fn() for _ in range(steps)]
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, stats, ctx.launch_count() - l0

    # ---- headline: device-timed samples/s ------------------------------
    with ClockSampler(local) as clk:
        ms, stats, launches = timed(step, args.steps, args.warmup)
    ktimes = ctx.kernel_times()
    total_samples = W * H * SPP
    value = total_samples * args.steps / (ms / 1e3)
    st = stats[-1]
    # the last timed render's frame (rank 0 holds the gathered image), kept
    # for the parity block below
    torch.cuda.synchronize()
    frame_off = None
    frame_cached = (rad.cpu().numpy().reshape(H, W, 3).copy(), nodes.cpu().numpy().reshape(H, W).copy(),
                    samples.cpu().numpy().reshape(H, W).copy())

    # ---- e2e through the host-buffer C ABI --------------------------------
    host_rad = torch.zeros(H * W * 3, dtype=torch.float64).pin_memory()
    host_nodes = torch.zeros(H * W, dtype=torch.float64).pin_memory()
    host_samples = torch.zeros(H * W, dtype=torch.int32).pin_memory()
    hframe = N.Frame(C.cast(C.c_void_p(host_rad.data_ptr()), C.POINTER(C.c_double)),
                     C.cast(C.c_void_p(host_nodes.data_ptr()), C.POINTER(C.c_double)),
                     C.cast(C.c_void_p(host_samples.data_ptr()), C.POINTER(C.c_uint32)))
    f = scene.flat
    scene_bytes = (f.n_prims * (48 + 24 + 4) + f.n_nodes * 32 + f.n_code * 16 + f.n_consts * 16
                   + f.n_noise * 16 + f.n_ramp_stops * 16 + f.n_texels * 16)
    frame_bytes = H * W * (24 + 8 + 4)

    def e2e_step():
        # the user's call sequence: scene to HBM, render, image back to host
        N.check(L.mcg_upload_scene(ctx.handle, scene.handle))
        s = N.RenderStats()
        if world == 1:
            host_rad.zero_(); host_nodes.zero_(); host_samples.zero_()
            N.check(L.mcg_render(ctx.handle, C.byref(params), None, C.byref(hframe), C.byref(s)))
            return s
        # N > 1: each rank renders its tiles into device frames, the frames
        # are reduced to rank 0 over NCCL, rank 0 copies the image to host
        with torch.cuda.stream(stream):
            rad.zero_(); nodes.zero_(); samples.zero_()
        N.check(L.mcg_render_device(ctx.handle, C.byref(params), None, C.byref(dframe), C.byref(s)))
        with torch.cuda.stream(stream):
            frame_reduce(dist, [rad, nodes, samples])
            if rank == 0:
                host_rad.copy_(rad, non_blocking=True)
                host_nodes.copy_(nodes, non_blocking=True)
                host_samples.copy_(samples, non_blocking=True)
        stream.synchronize()
        return s

    e2e_steps = max(1, min(args.steps, 2))
    for _ in range(1):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    t_e2e = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([t_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())
    e2e_value = total_samples * e2e_steps / t_e2e
    ctx.upload(scene)

    # ---- extras: cache speed-up and probe roofline (rank 0 leg, N=1 job) ----
    extras = {}
    if not args.no_extras:
        off = RenderConfig(width=W, height=H, spp=SPP, cache_enabled=False,
                           shard_rank=rank, shard_count=world).to_params()
        ms_off, _, _ = timed(lambda: step(off), 1, 1)
        torch.cuda.synchronize()
        frame_off = rad.cpu().numpy().reshape(H, W, 3).copy()
        extras["cache_speedup"] = {"t_nocache_ms": ms_off, "t_cache_ms": ms / args.steps,
                                   "speedup": ms_off / (ms / args.steps)}
        if rank == 0 and world == 1:
            # the same frame at other tunings (one render each after a warm-up,
            # device time): mip_offset 0 on the bench scene, and round 1's
            # tiled-uv scene at mip_offset 0 (hit rate ~0.998, but SPEC #5
            # fails there for the reference too: profiles/README.md)
            from paper_2305_07238_b200 import render as api_render, scenes as S
            tun = {}
            tiled = load_scene(S.build_scene(S.SceneSpec(SCENE_KIND, W, H, tris_per_side=TRIS_PER_SIDE,
                                                         libm_ops=True), os.path.join(tmp, "tiled")))
            for name, sc, mip in (("unit_uv_mip0", scene, 0), ("tiled_uv_mip0", tiled, 0)):
                base = dict(width=W, height=H, spp=SPP, n_cells=N_CELLS, n_entries=N_ENTRIES, mip_offset=mip)
                api_render(sc, RenderConfig(cache_enabled=True, **base), ctx=ctx)
                on = api_render(sc, RenderConfig(cache_enabled=True, **base), ctx=ctx).stats
                t_off = (api_render(sc, RenderConfig(**base), ctx=ctx).stats.device_ms if sc is not scene
                         else ms_off)
                tun[name] = {"ms_cache": on.device_ms, "ms_no_cache": t_off, "speedup": t_off / on.device_ms,
                             "hit_rate": on.hit_rate, "samples_per_s": W * H * SPP / (on.device_ms / 1e3)}
            # BASELINE configs[3]: the Bmw-like analogue with every lookup on
            # the finest virtual level (mip_offset 24: hit rate ~0, the table
            # fills, then every insert finds its cell full) vs its no-cache
            # render -- north_star: >= 90% of no-cache throughput
            bmw = load_scene(S.build_scene(S.SceneSpec("bmw", W, H, tris_per_side=TRIS_PER_SIDE, uv_span=UV_SPAN),
                                           os.path.join(tmp, "bmw")))
            base = dict(width=W, height=H, spp=SPP, n_cells=N_CELLS, n_entries=N_ENTRIES, mip_offset=24)
            api_render(bmw, RenderConfig(**base), ctx=ctx)
            t_off = statistics.median(api_render(bmw, RenderConfig(**base), ctx=ctx).stats.device_ms
                                      for _ in range(2))
            api_render(bmw, RenderConfig(cache_enabled=True, **base), ctx=ctx)   # warm-up (first cached render)
            ons = [api_render(bmw, RenderConfig(cache_enabled=True, **base), ctx=ctx).stats for _ in range(2)]
            t_on = statistics.median(o.device_ms for o in ons)
            extras["worst_case"] = {"scene": "bmw-like, unit uv, mip_offset 24 (BASELINE configs[3])",
                                    "ms_cache": t_on, "ms_no_cache": t_off,
                                    "throughput_vs_no_cache": t_off / t_on, "hit_rate": ons[-1].hit_rate,
                                    "inserts_lost_full": ons[-1].inserts_lost_full, "target": 0.9}
            # the deterministic-insert mode (north_star) on the bench workload
            dcfg = RenderConfig(width=W, height=H, spp=SPP, n_cells=N_CELLS, n_entries=N_ENTRIES,
                                mip_offset=MIP_OFFSET, cache_enabled=True, deterministic=True)
            api_render(scene, dcfg, ctx=ctx)
            dst = api_render(scene, dcfg, ctx=ctx).stats
            extras["deterministic"] = {"ms": dst.device_ms, "samples_per_s": W * H * SPP / (dst.device_ms / 1e3),
                                       "hit_rate": dst.hit_rate,
                                       "note": "epoch-deferred ordered inserts, one pass lane; bit-identical runs"}
            ctx.upload(scene)
            extras["tunings"] = tun
        if rank == 0:
            from paper_2305_07238_b200 import MaterialCache
            peak, _ = measured_peaks()
            n = 1 << 26

            def legs(table, variant, bps):
                cfg = 16 * variant + 256 * bps
                table.probe_bench(n, 7, 0 + cfg, 1)    # warm-up (module load, first touch)
                table.clear()
                ms_ins, b_ins = table.probe_bench(n, 7, 0 + cfg, 1)
                table.probe_bench(n, 7, 1 + cfg, 1)
                ms_look, b_look = table.probe_bench(n, 7, 1 + cfg, 3)
                ms_mix, b_mix = table.probe_bench(n, 8, 2 + cfg, 3)
                leg = lambda b, m: {"achieved": b / m / 1e6, "frac": b / m / 1e6 / peak,  # noqa: E731
                                    "mprobes_per_s": n / m / 1e3}
                return {"variant": variant, "blocks_per_sm": bps, "insert_all": leg(b_ins, ms_ins),
                        "lookup_all": leg(b_look, ms_look), "mix_50_50": leg(b_mix, ms_mix)}

            table = MaterialCache(N_CELLS, N_ENTRIES, ctx)
            pr = {"bound": "hbm", "unit": "GB/s", "peak": peak, "table": "1e7x10 (800 MB)",
                  "kernel": "k_probe_bench", "descriptors": n,
                  # profiles/scripts/rand_read2.cu (B200, 800 MB buffer): random 64-byte
                  # reads by 4 lanes x 16 B top out at 43.9 G accesses/s (each costs a
                  # 128-byte DRAM fetch); one 64-byte head read per lookup at that rate
                  # is 3512 GB/s in 80-byte-cell algorithmic bytes.
                  "random_access_ceiling": {"g_accesses_per_s": 43.9, "bytes_per_access": 64,
                                            "algorithmic_gbs_80B_cells": 3512.0,
                                            "source": "profiles/scripts/rand_read2.cu"}}
            pr.update(legs(table, PROBE_VARIANT, PROBE_BLOCKS_PER_SM))
            table.close()
            # replay of the bench render's own lookups (first 2^26 of them)
            traced = MaterialCache(N_CELLS, N_ENTRIES, ctx)
            traced.trace_start(1 << 26)
            pr_params = cfg.to_params()
            st_t = N.RenderStats()
            N.check(L.mcg_render_device(ctx.handle, C.byref(pr_params), traced.handle, C.byref(dframe),
                                        C.byref(st_t)))
            n_tr = traced.trace_stop()
            trace = traced.trace_read(0, n_tr)
            traced.close()
            fresh = MaterialCache(N_CELLS, N_ENTRIES, ctx)
            fresh.probe_replay(trace[: 1 << 20])          # warm-up
            fresh.clear()
            ms_r, b_r, c_r = fresh.probe_replay(trace)
            fresh.close()
            pr["trace_replay"] = {"descriptors": int(n_tr), "source": "the bench render's first lookups",
                                  "achieved": b_r / ms_r / 1e6, "frac": b_r / ms_r / 1e6 / peak,
                                  # + the 20-byte descriptor records the kernel streams in
                                  "achieved_incl_descriptors": (b_r + 20.0 * n_tr) / ms_r / 1e6,
                                  "mprobes_per_s": n_tr / ms_r / 1e3,
                                  "hit_rate": c_r["hits"] / max(1, c_r["lookups"])}
            small = MaterialCache(100_000, N_ENTRIES, ctx)
            pr["l2_resident_1e5x10"] = legs(small, PROBE_L2_VARIANT, PROBE_L2_BLOCKS_PER_SM)
            pr["l2_resident_1e5x10"]["table"] = "1e5x10 (8 MB, L2-resident)"
            small.close()
            extras["probe_roofline"] = pr

    # ---- roofline of the dominant kernel ----------------------------------
    # The timed renders run two pass lanes and a second stream per vertex
    # (MCG_LANES=2, MCG_OVERLAP): their per-kernel event times overlap and do
    # not add up to the step. The dominant kernel is therefore chosen, and
    # its per-launch time taken, from one serialized side render of the same
    # workload (MCG_LANES=1 MCG_OVERLAP=0: one kernel at a time, so each
    # event pair brackets exactly one kernel) -- what ncu's launch list
    # measures too (profiles/). Its work counters are that render's own.
    peak, peak_src = measured_peaks()
    serial_env = {"MCG_LANES": "1", "MCG_OVERLAP": "0"}
    saved = {k: os.environ.get(k) for k in serial_env}
    os.environ.update(serial_env)
    try:
        step()   # warm-up: the one-lane layout's buffers are allocated on first use
        torch.cuda.synchronize()
        ctx.reset_kernel_times()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st_s = step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_serial = e0.elapsed_time(e1)
        kser = ctx.kernel_times()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    ne = N_ENTRIES
    f = scene.flat
    n_lights = f.n_point_lights + f.n_rect_lights
    closest_hits = min(st_s.closest_rays, max(0, st_s.shading_points - st_s.paths))
    # Per kernel class, per render: (a) SURVEY §8(d)'s algorithmic bytes --
    # 8 Ne per lookup / store attempt (+8 per won CAS), 48 per TexSample,
    # 40 per BVH node visited (the reference's BvhNode), 48 per triangle
    # tested -- and (b) the compulsory HBM bytes, what must cross HBM at
    # least once. The first probe of every lookup runs in the trace kernels'
    # epilogue (look-ahead, before the sort); the shade re-probes the misses
    # (concurrent mode, cells not seen full) and stores. Shade: per shading
    # point the two path records in (64 + 32 B: shading point, direction,
    # look-ahead result; throughput, radiance) and out (32 + 32 B), per
    # shadow-ray candidate 52 B out (16 B per rejected light); closest hit:
    # per ray the ray and path id in (32 + 32 B), per hit the shading point
    # (64 B), look-ahead result (16 B) and sort key/value (8 B) out, the key
    # per miss;
    # per shadow ray 37 B; plus the scene once per launch. The traversal
    # kernels' node and triangle bytes are served by L1/L2 (the bench BVH is
    # a few hundred KB): (a) >> (b) for them.
    nodes_closest = st_s.bvh_nodes - st_s.bvh_nodes_shadow
    prims_closest = st_s.prims_tested - st_s.prims_tested_shadow
    lookahead_bytes = st_s.lookups * 8 * ne
    shade_probe_bytes = ((st_s.lookups - st_s.hits) * 8 * ne + st_s.stores_attempted * 8 * ne
                         + st_s.inserts_won * 8)
    scene_once = f.n_prims * (48 + 24 + 4) + f.n_nodes * 64
    algorithmic = {
        "shade": shade_probe_bytes + st_s.tex_samples * 48,
        "trace_closest": nodes_closest * 40 + prims_closest * 48 + lookahead_bytes,
        "trace_shadow": st_s.bvh_nodes_shadow * 40 + st_s.prims_tested_shadow * 48,
    }
    compulsory = {
        "shade": shade_probe_bytes + st_s.tex_samples * 48 + st_s.shading_points * (96 + 64)
                 + st_s.shadow_rays * 52 + (n_lights * st_s.shading_points - st_s.shadow_rays) * 16,
        "trace_closest": (st_s.closest_rays * 64 + closest_hits * 88 + (st_s.closest_rays - closest_hits) * 8
                          + lookahead_bytes),
        "trace_shadow": st_s.shadow_rays * 37,
    }
    # ncu DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum
    # of every launch of one render, averaged): read back from the committed
    # capture named in `_source`, never measured under this run.
    try:
        with open(os.path.join(ROOT, "profiles", "dram_traffic.json")) as fh:
            traffic_doc = json.load(fh)
    except Exception:
        traffic_doc = {}
    try:
        with open(os.path.join(ROOT, "profiles", "kernel_efficiency.json")) as fh:
            eff = json.load(fh)
    except Exception:
        eff = {}

    def kernel_roofline(kname):
        rec = kser.get(kname, {"ms": 0.0, "launches": 0})
        launches = max(1, rec["launches"])
        per_ms = rec["ms"] / launches
        alg = algorithmic.get(kname, rec.get("bytes", 0.0)) / launches
        comp = compulsory.get(kname, rec.get("bytes", 0.0)) / launches
        if kname in ("trace_closest", "trace_shadow"):
            comp += scene_once
        gbs = (lambda b: b / (per_ms / 1e3) / 1e9 if per_ms > 0 else 0.0)  # noqa: E731
        out = {"bound": "hbm", "kernel": kname, "achieved": gbs(alg), "peak": peak, "unit": "GB/s",
               "frac": gbs(alg) / peak, "traffic": traffic_doc.get(kname),
               "algorithmic_bytes_per_launch": alg,
               "units": "SURVEY 8(d): 8*Ne B per lookup/store attempt (+8 per won CAS), 48 B per TexSample, "
                        "40 B per BVH node visited, 48 B per triangle tested",
               "per_launch_ms": per_ms, "launches_per_step": rec["launches"],
               "hbm_compulsory": {"bytes_per_launch": comp, "achieved": gbs(comp), "frac": gbs(comp) / peak},
               "timing": "serialized side render (MCG_LANES=1 MCG_OVERLAP=0), CUDA events around each launch"}
        if traffic_doc.get("_source"):
            out["traffic_source"] = traffic_doc["_source"]
        if kname in eff:
            out["issue"] = eff[kname]
        return out

    total_ser = sum(x["ms"] for x in kser.values())
    dname = max(kser.items(), key=lambda kv: kv[1]["ms"])[0] if kser else "?"
    roof = kernel_roofline(dname)
    roof["serialized_share"] = {k: round(v["ms"] / max(1e-9, total_ser), 4) for k, v in kser.items()}
    roof["serialized_render_ms"] = ms_serial
    # consistency: the dominant kernel's launches fit inside one timed step
    roof["fits_in_step"] = bool(roof["per_launch_ms"] * roof["launches_per_step"] <= ms / args.steps)
    roof["limiter"] = ("issue/latency: warp divergence in BVH traversal (L1/L2-resident tree) -- the "
                       "8(d) bytes are L1/L2-served, HBM (hbm_compulsory) is not the bound"
                       if dname.startswith("trace") else
                       "random HBM accesses (the path-record gather, re-probes, textures) and dependent "
                       "FP latency in the material VM; see roofline.issue and traffic")
    roof["peak_source"] = peak_src
    # The north-star kernel (material VM + cache probes) beside it.
    roof_shade = kernel_roofline("shade")
    # Render-level: the compulsory bytes of the shade and
    # traversal kernels over the timed step.
    total_bytes = sum(compulsory.values())
    roof["render_level"] = {"compulsory_bytes_per_step": total_bytes,
                            "achieved": total_bytes / (ms / args.steps / 1e3) / 1e9,
                            "frac": total_bytes / (ms / args.steps / 1e3) / 1e9 / peak}
    ktimes_overlapped = {k: {"ms": round(v["ms"], 3), "launches": v["launches"]} for k, v in ktimes.items()}

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            # median of 3 runs, a fresh table each; RNG seeds
            # 1-3, so the runs double as the parity block's reference images
            runs = [cpu_reference_sample(scene_path, seed=sd) for sd in (1, 2, 3)]
            info = sorted(runs, key=lambda r: r["seconds"])[1]
            cpu = {"value": info["samples"] / info["seconds"], "unit": "samples/s",
                   "cores": info["cores"], "kind": info["kind"],
                   "sample": cpu_sample_text(info) + "; median of 3 runs",
                   "table_build_s": info.get("table_build_s"),
                   "hit_rate": info["hits"] / max(1, info["lookups"]) if "hits" in info else None}
            ref_band = runs
        except Exception as e:  # the checker must never break the bench line
            cpu = {"value": None, "unit": "samples/s", "cores": 0, "kind": "unavailable",
                   "sample": str(e)[:200]}
            ref_band = None
        # Parity of the timed path itself (north_star, concurrent mode): the
        # timed render's image vs the cache-off image of the same workload
        # (RMSE), beside the reference's own cached-vs-uncached RMSE on the
        # band it rendered above; pixels without a cache hit must equal the
        # cache-off render bit for bit; hits == sum of the
        # per-pixel hit counts.
        if frame_off is not None:
            try:
                from paper_2305_07238_b200 import render as api_render
                band_cfg = dict(width=W, height=H, spp=SPP, n_cells=N_CELLS, n_entries=N_ENTRIES,
                                mip_offset=MIP_OFFSET, shard_rank=CPU_BAND, shard_count=CPU_BANDS, shard_mode=1,
                                samples_per_pass=2)   # the timed path's schedule (k = 2 at 1080p, two lanes)
                gpu_bands = []
                for r in (ref_band or []):
                    cfg = dict(band_cfg, rng_seed=r["seed"])
                    gpu_bands.append((api_render(scene, RenderConfig(cache_enabled=True, **cfg), ctx=ctx).frame,
                                      api_render(scene, RenderConfig(cache_enabled=False, **cfg), ctx=ctx).frame))
                parity = parity_block(frame_cached, frame_off, st, ref_band, gpu_bands)
            except Exception as e:
                parity = {"error": str(e)[:200]}
        try:
            # the reference's MaterialCache on the 1e7x10 table,
            # 1 thread and every host thread, same descriptor generator as the
            # device probe (2^22 descriptors: insert-all, then lookup-all)
            import _oracle
            if _oracle.Ref.available():
                ref = _oracle.Ref()
                n_cpu = 1 << 22
                pcpu = {"table": "1e7x10 (800 MB)", "descriptors": n_cpu, "kind": "reference"}
                for th in (1, os.cpu_count() or 1):
                    c = ref.cache_new(N_CELLS, N_ENTRIES)
                    ref.probe_bench(c, n_cpu, 11, 1, th)          # first touch of the table
                    t_ins = ref.probe_bench(c, n_cpu, 7, 0, th)
                    t_look = ref.probe_bench(c, n_cpu, 7, 1, th)
                    ref.cache_free(c)
                    pcpu[f"threads_{th}"] = {"insert_mprobes_per_s": n_cpu / t_ins / 1e6,
                                             "lookup_mprobes_per_s": n_cpu / t_look / 1e6}
                extras.setdefault("probe_roofline", {})["cpu_reference"] = pcpu
        except Exception as e:
            extras.setdefault("probe_roofline", {})["cpu_reference"] = {"unavailable": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded classroom-like scene in the reference's JSON/PPM formats)",
            "config": {"workload": f"{SCENE_KIND}-like {W}x{H} {SPP}spp, cache {N_CELLS:.0e}x{N_ENTRIES}, "
                                   f"unit uv, mip_offset {MIP_OFFSET}, concurrent inserts",
                       "width": W, "height": H, "spp": SPP, "uv_span": UV_SPAN, "mip_offset": MIP_OFFSET,
                       "n_cells": N_CELLS, "n_entries": N_ENTRIES, "parallelism": f"tiles/{world}",
                       "cache": "striped over GPUs" if shared is not None else "per-GPU replica",
                       "l2": "inputs larger than L2 (800 MB table re-zeroed per render + "
                             f"{(W * H * 10 * 16) >> 20} MB path state)"},
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": "samples/s",
                    # N = 1: scene + framebuffers in (mcg_render accumulates into
                    # the caller's frame), image out; N > 1: scene in on every
                    # rank, frames reduced to rank 0 over NCCL, image out on rank 0
                    "h2d_bytes_per_step": int(scene_bytes * world + (frame_bytes if world == 1 else 0)),
                    "d2h_bytes_per_step": int(frame_bytes)},
            "gpu_launches": int(launches),
            "roofline": roof,
            "roofline_shade": roof_shade,
            "kernel_event_ms_timed_region": ktimes_overlapped,
            "render_stats": {"hit_rate": st.hits / st.lookups if st.lookups else 0.0,
                             "lookups": st.lookups, "hits": st.hits, "inserts_won": st.inserts_won,
                             "inserts_lost_full": st.inserts_lost_full,
                             "shading_points": st.shading_points, "shadow_rays": st.shadow_rays,
                             "bvh_nodes": st.bvh_nodes, "prims_tested": st.prims_tested,
                             "bvh_nodes_shadow": st.bvh_nodes_shadow,
                             "prims_tested_shadow": st.prims_tested_shadow,
                             "closest_rays": st.closest_rays, "tex_samples": st.tex_samples},
            "cpu_baseline": cpu,
            "parity": parity,
        }
        line.update(extras)
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
