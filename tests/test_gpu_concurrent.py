"""Concurrent mode -- the paper's single-CAS inserts, the path bench.py times
-- against the reference's own concurrent render (oracle/_ref, mode 2: the
tile queue over every host thread sharing one MaterialCache).

Which sample first inserts a texel is a race in both, so the cached image is
a random variable in both; the north star bounds the GPU's cached-vs-uncached
RMSE by the reference's own plus 1e-4. Both are sampled three times and
their medians compared. SPEC.md's render invariants are exact and asserted
on every GPU render: pixels without a cache hit are bit-identical to the
cache-off render and RenderStats.hits equals the sum of the
per-pixel hit counts and of hits_per_sample.
"""
import os
import statistics

import numpy as np
import pytest

from paper_2305_07238_b200 import RenderConfig, load_scene, render, scenes

import _oracle

pytestmark = pytest.mark.gpu

NC, NE = 10_000_000, 10


def errors(img, off):
    d = np.abs(img.astype(np.float64) - off.astype(np.float64))
    return {"rmse": float(np.sqrt((d ** 2).mean())), "mean_abs": float(d.mean()),
            "frac_lt_0.05": float((d.max(-1) < 0.05).mean())}


def check_invariants(res, off):
    zero = res.frame.nodes_found == 0
    np.testing.assert_array_equal(res.frame.radiance[zero].view(np.uint64),
                                  off.frame.radiance[zero].view(np.uint64))
    assert int(res.stats.hits) == int(res.frame.nodes_found.sum()) == sum(res.stats.hits_per_sample)
    assert res.stats.hits > 0


def ref_runs(ref, path, p, w, h, runs=3):
    rs = ref.scene_load(path)
    out = []
    for _ in range(runs):
        rad, nodes, samples, hps, st = ref.render(rs, p, w, h)
        out.append((rad, samples, st))
    ref.L.ref_scene_free(rs)
    return out


@pytest.mark.parametrize("lanes", ["2", "1"])
def test_bench_band_concurrent_rmse_within_reference(ctx, ref, scene_dir, lanes, monkeypatch):
    """The bench's scene, camera, table and tuning at the bench's schedule --
    one sample per pass (what 1920x1080 resolves to), passes alternating on
    two stream lanes (MCG_LANES=2, the default) -- on the band of tiles the
    CPU baseline renders (contiguous tiles 8/16 of the 1080p frame, ~130K
    pixels), 64 spp: 64 passes in flight two at a time.

    Which sample first inserts a texel is a race in both renderers and the
    RMSE is carried by a few bright pixels, so one render is one draw: the
    reference's own run-to-run spread reaches 7% on some seeds
    (profiles/README.md, rmse_seeds). The north star's bound (reference RMSE
    + 1e-4) is therefore asserted on the mean over four RNG seeds -- the GPU's
    median of three renders per seed against one reference render per seed
    -- with the standard error of the per-seed differences as the noise
    allowance (2 SE)."""
    import bench
    monkeypatch.setenv("MCG_LANES", lanes)
    path = bench.make_scene(scene_dir + "/bench_band")
    s = load_scene(path)
    rs = ref.scene_load(path)
    W, H, spp = bench.W, bench.H, 64
    threads = os.cpu_count() or 1
    diffs, rows = [], []
    for seed in (1, 2, 3, 4):
        band = dict(width=W, height=H, spp=spp, n_cells=NC, n_entries=NE, shard_rank=bench.CPU_BAND,
                    shard_count=bench.CPU_BANDS, shard_mode=1, samples_per_pass=1, mip_offset=bench.MIP_OFFSET,
                    rng_seed=seed)
        off = render(s, RenderConfig(**band), ctx=ctx)
        mask = off.frame.samples > 0
        off_img = off.frame.radiance_image()[mask]
        gpu = []
        for _ in range(3):
            r = render(s, RenderConfig(cache_enabled=True, **band), ctx=ctx)
            check_invariants(r, off)
            gpu.append(errors(r.frame.radiance_image()[mask], off_img)["rmse"])
        p = _oracle.RenderParamsC(W, H, spp, 4, 2, bench.MIP_OFFSET, NC, NE, 0, seed, 0.2, 16, bench.CPU_BAND,
                                  bench.CPU_BANDS, 1, threads, 1)
        rad, nodes, samples, hps, st = ref.render(rs, p, W, H)
        np.testing.assert_array_equal(samples > 0, mask)
        rr = errors((rad / np.maximum(samples, 1)[..., None]).astype(np.float32)[mask], off_img)["rmse"]
        rows.append((seed, gpu, rr))
        diffs.append(statistics.median(gpu) - rr)
    ref.L.ref_scene_free(rs)
    mean = statistics.mean(diffs)
    se = statistics.stdev(diffs) / len(diffs) ** 0.5
    print(f"lanes={lanes} per seed (gpu rmse x3, reference rmse): {rows}; mean diff {mean:.5f} se {se:.5f}")
    assert mean <= 1e-4 + 2.0 * se, rows


@pytest.mark.parametrize("kind", ["classroom", "junkshop", "italianflat", "monster", "cornell"])
def test_spec5_image_fidelity_where_the_reference_passes(ctx, ref, scene_dir, kind):
    """SPEC acceptance #5 at 256x256x128: mean |cached -
    uncached| <= 0.01 and >= 99% of pixels within 0.05, and the mean falling
    as mip_offset goes 0 -> 2. With tiled uv (round 1's scenes) the
    reference itself fails it on every scene (profiles/README.md "SPEC #5");
    with one uv tile per surface and mip_offset 3 -- the bench's tuning -- the
    reference passes on these five analogues, and so must the GPU, with a
    mean error within 25% of the reference's (the first-insert race makes
    both random; measured spread ~10%)."""
    w = h = 256
    spp = 128
    path = scenes.build_scene(scenes.SceneSpec(kind, w, h, tris_per_side=24, uv_span=0.999),
                              f"{scene_dir}/spec5_{kind}")
    s = load_scene(path)
    base = dict(width=w, height=h, spp=spp, n_cells=NC, n_entries=NE)
    off = render(s, RenderConfig(**base), ctx=ctx)
    off_img = off.frame.radiance_image()
    means = []
    for mip in (0, 1, 2, 3):
        r = render(s, RenderConfig(cache_enabled=True, mip_offset=mip, **base), ctx=ctx)
        check_invariants(r, off)
        means.append(errors(r.frame.radiance_image(), off_img))
    gpu = means[3]
    assert gpu["mean_abs"] <= 0.01 and gpu["frac_lt_0.05"] >= 0.99, gpu
    assert means[0]["mean_abs"] >= means[1]["mean_abs"] >= means[2]["mean_abs"], means
    threads = os.cpu_count() or 1
    p = _oracle.RenderParamsC(w, h, spp, 4, 2, 3, NC, NE, 0, 1, 0.2, 16, 0, 1, 0, threads, 1)
    (rad, samples, st), = ref_runs(ref, path, p, w, h, runs=1)
    rerr = errors((rad / np.maximum(samples, 1)[..., None]).astype(np.float32), off_img)
    print(kind, "gpu", gpu, "ref", rerr)
    assert rerr["mean_abs"] <= 0.01 and rerr["frac_lt_0.05"] >= 0.99, rerr
    assert abs(gpu["mean_abs"] - rerr["mean_abs"]) <= 0.25 * rerr["mean_abs"] + 1e-4, (gpu, rerr)
