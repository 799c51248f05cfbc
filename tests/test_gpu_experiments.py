"""The sweep driver and the figure artefacts on the GPU path (
SPEC.md:456-476 examples)."""
import numpy as np
import pytest

from paper_2305_07238_b200 import (RenderConfig, artifacts, load_scene, memory_bytes, render, scenes,
                                   stats_to_json, sweep, write_sweep_csv)

pytestmark = pytest.mark.gpu


def test_sweep_rows_and_hit_rate_trend(ctx, scene_dir, tmp_path):
    path = scenes.build_scene(scenes.SceneSpec("classroom", 64, 48, tris_per_side=6), f"{scene_dir}/sweep")
    s = load_scene(path)
    rows = sweep(s, RenderConfig(width=64, height=48, spp=16), [100_000, 1_000, 10_000], [10, 2], ctx=ctx)
    assert [(r.n_cells, r.n_entries) for r in rows] == [(1_000, 2), (1_000, 10), (10_000, 2), (10_000, 10),
                                                       (100_000, 2), (100_000, 10)]
    for r in rows:
        assert r.memory_bytes == memory_bytes(r.n_cells, r.n_entries) and r.wall_time_s > 0
        assert r.relative_time_pct > 0
    hr = {(r.n_cells, r.n_entries): r.hit_rate for r in rows}
    for e in (2, 10):
        assert hr[(1_000, e)] <= hr[(10_000, e)] + 1e-3 <= hr[(100_000, e)] + 2e-3
    out = tmp_path / "sweep.csv"
    write_sweep_csv(rows, str(out))
    lines = out.read_text().splitlines()
    assert lines[0] == "n_cells,n_entries,wall_time_s,relative_time_pct,hit_rate,inserts_lost_full,memory_bytes"
    assert len(lines) == 7
    with pytest.raises(ValueError):
        sweep(s, RenderConfig(width=8, height=8, spp=1), [0], [2], ctx=ctx)


def test_render_artifacts(ctx, scene_dir, tmp_path):
    path = scenes.build_scene(scenes.SceneSpec("junkshop", 40, 30, tris_per_side=4), f"{scene_dir}/art")
    s = load_scene(path)
    off = render(s, RenderConfig(width=40, height=30, spp=4), ctx=ctx)
    on = render(s, RenderConfig(width=40, height=30, spp=4, cache_enabled=True, n_cells=4099, n_entries=4),
                ctx=ctx)
    assert on.stats.device_ms > 0 and off.stats.hits == 0
    a, b = on.frame.radiance_image(), off.frame.radiance_image()
    artifacts.write_pfm(str(tmp_path / "a.pfm"), a)
    np.testing.assert_array_equal(artifacts.read_pfm(str(tmp_path / "a.pfm")), a)
    d = artifacts.write_diff(a, b, str(tmp_path / "d.ppm"))
    assert d.diff.shape == a.shape and 0.0 <= d.mean_abs <= d.max_abs
    heat = artifacts.write_heatmap(stats_to_json(on.stats, on.frame), str(tmp_path / "h.ppm"))
    assert heat.shape == (30, 40, 3)
    # pixels with no hits map to viridis(0)
    zero = on.frame.nodes_found_avg() == 0
    assert (heat[zero] == artifacts.viridis(0.0)).all()


def test_descriptor_trace_and_replay(ctx, scene_dir):
    """the lookups of a render are recorded in order and replayed
    through a fresh table (lookup, insert on a miss)."""
    from paper_2305_07238_b200 import MaterialCache
    path = scenes.build_scene(scenes.SceneSpec("classroom", 48, 32, tris_per_side=4), f"{scene_dir}/trace")
    s = load_scene(path)
    t = MaterialCache(4099, 4, ctx)
    t.trace_start(1 << 20)
    res = render(s, RenderConfig(width=48, height=32, spp=8, cache_enabled=True, n_cells=4099, n_entries=4),
                 external_cache=t, ctx=ctx)
    n = t.trace_stop()
    assert n == res.stats.lookups > 0
    tr = t.trace_read(0, n)
    assert (tr["mip_level"] <= 24).all() and (tr["mat_idx"] < s.n_materials).all()
    assert (tr["texel_x"] < (1 << tr["mip_level"].astype(np.uint64))).all()
    fresh = MaterialCache(4099, 4, ctx)
    ms, nbytes, c = fresh.probe_replay(tr)
    assert c["lookups"] == n and ms > 0 and nbytes >= n * 32
    keys = {tuple(x) for x in tr[["mat_idx", "node_idx", "mip_level", "texel_x", "texel_y"]].tolist()}
    assert c["inserts_won"] + c["inserts_lost_full"] >= len(keys) - (n - c["hits"] - c["inserts_won"]
                                                                     - c["inserts_lost_full"])
    assert c["hits"] + c["inserts_won"] + c["inserts_lost_full"] <= n
    # the replayed table answers every traced key that found room
    hit, _ = fresh.lookup_batch(tr)
    assert hit.mean() > 0.9
    # a small capacity keeps the first records only
    t.clear()
    t.trace_start(100)
    render(s, RenderConfig(width=48, height=32, spp=2, cache_enabled=True, n_cells=4099, n_entries=4),
           external_cache=t, ctx=ctx)
    assert t.trace_stop() == 100
