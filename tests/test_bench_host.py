"""Host-side logic of bench.py's parity block (CPU): the concurrent-mode
bound is checked on the mean over RNG seeds of (GPU RMSE - reference RMSE)
with two standard errors of the per-seed differences as the allowance; the
zero-hit and hit-count invariants are exact."""
import numpy as np

import bench


class _Frame:
    def __init__(self, rad, nodes, samples):
        self.radiance, self.nodes_found, self.samples = rad, nodes, samples

    def radiance_image(self):
        return (self.radiance / np.maximum(self.samples, 1)[..., None]).astype(np.float32)


class _Stats:
    def __init__(self, hits):
        self.hits = hits


def _band(h, w, seed, noise):
    r = np.random.default_rng(seed)
    samples = np.zeros((h, w), np.uint32)
    samples[h // 4: h // 2] = 4
    off = r.uniform(0, 1, (h, w, 3)) * samples[..., None]
    cached = off + (r.normal(0, noise, off.shape) * (samples[..., None] > 0))
    nodes = (samples > 0).astype(np.float64) * 3
    nodes[h // 4, :5] = 0
    cached[h // 4, :5] = off[h // 4, :5]          # zero-hit pixels equal the cache-off render
    return off, cached, nodes, samples


def _case(noise_gpu, noise_ref):
    h, w = 16, 24
    ref_runs, gpu_bands = [], []
    for seed in (1, 2, 3):
        off, cached, nodes, samples = _band(h, w, seed, noise_gpu)
        _, rcached, _, _ = _band(h, w, seed, noise_ref)
        ref_runs.append({"kind": "reference", "radiance": rcached, "pixel_samples": samples, "seed": seed,
                         "samples": int(samples.sum()), "table_build_s": 0.1, "cores": 4})
        gpu_bands.append((_Frame(cached, nodes, samples), _Frame(off, np.zeros_like(nodes), samples)))
    off, cached, nodes, samples = _band(h, w, 9, noise_gpu)
    return bench.parity_block((cached, nodes, samples), off, _Stats(int(nodes.sum())), ref_runs, gpu_bands)


def test_parity_block_within_bound_when_errors_match():
    p = _case(0.01, 0.01)
    assert p["hits_eq_sum_nodes_found"] and p["zero_hit_pixels_bit_identical"]
    b = p["band"]
    assert len(b["per_seed"]) == 3 and b["zero_hit_pixels_bit_identical"]
    assert b["within_bound"]


def test_parity_block_flags_a_larger_error():
    assert not _case(0.05, 0.01)["band"]["within_bound"]
