"""ctypes access to the CPU checkers (TEST INFRASTRUCTURE):

* ``Oracle``: oracle/_build/libmcoracle.so, the C restatement of the path;
* ``Ref``: oracle/_ref/libmcref.so, the reference's own sources compiled in
  place plus the restated render (None when it was not built -- it needs
  /root/reference at build time).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2305_07238_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libmcoracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libmcref.so")

vp = C.c_void_p


def ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class RenderParamsC(C.Structure):
    """mco_render_params / RefRenderParams (identical layouts)."""
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("spp", C.c_int32),
                ("max_bounces", C.c_int32), ("mode", C.c_int32), ("mip_offset", C.c_int32),
                ("n_cells", C.c_uint64), ("n_entries", C.c_uint32), ("first_sample", C.c_uint32),
                ("rng_seed", C.c_uint64), ("diffuse_spread", C.c_float), ("tile_size", C.c_int32),
                ("shard_rank", C.c_int32), ("shard_count", C.c_int32), ("shard_mode", C.c_int32),
                ("threads", C.c_int32), ("samples_per_pass", C.c_int32)]


class RenderStatsC(C.Structure):
    _fields_ = [("wall_time_s", C.c_double), ("lookups", C.c_uint64), ("hits", C.c_uint64),
                ("inserts_won", C.c_uint64), ("inserts_lost_full", C.c_uint64),
                ("stores_attempted", C.c_uint64), ("stores_won", C.c_uint64),
                ("instructions_executed", C.c_uint64), ("paths", C.c_uint64),
                ("shading_points", C.c_uint64)]


MODE_OFF, MODE_SEQUENTIAL, MODE_THREADED, MODE_DETERMINISTIC = 0, 1, 2, 3


def build_oracle(ref: bool = True) -> None:
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                   stdout=subprocess.DEVNULL)
    if ref and os.path.isdir("/root/reference"):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8", "ref"], check=True,
                       stdout=subprocess.DEVNULL)


def _render_outputs(w, h, spp):
    return (np.zeros((h, w, 3), np.float64), np.zeros((h, w), np.float64),
            np.zeros((h, w), np.uint32), np.zeros(spp, np.uint64))


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle(ref=False)
        self.L = C.CDLL(path)
        L = self.L
        L.mco_hash_batch.argtypes = [vp, C.c_size_t, vp, vp]
        L.mco_encode_batch.argtypes = [vp, C.c_size_t, vp]
        L.mco_decode_batch.argtypes = [vp, C.c_size_t, vp]
        L.mco_mip_texel_batch.argtypes = [vp, vp, vp, C.c_size_t, C.c_int, vp, vp]
        L.mco_footprint_batch.argtypes = [vp, C.c_size_t, vp]
        L.mco_fbm_batch.argtypes = [vp, vp, vp, C.c_size_t, vp]
        L.mco_sin_wave_batch.argtypes = [vp, C.c_size_t, vp]
        L.mco_power_batch.argtypes = [vp, vp, C.c_size_t, vp]
        L.mco_atan2f_batch.argtypes = [vp, vp, C.c_size_t, vp]
        L.mco_acosf_batch.argtypes = [vp, C.c_size_t, vp]
        L.mco_rng.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32]
        L.mco_rng.restype = C.c_float
        L.mco_cache_new.argtypes = [C.c_uint64, C.c_uint32]
        L.mco_cache_new.restype = vp
        L.mco_cache_free.argtypes = [vp]
        L.mco_cache_update_batch.argtypes = [vp, vp, vp, C.c_size_t, vp, vp, vp]
        L.mco_cache_lookup_batch.argtypes = [vp, vp, C.c_size_t, vp, vp]
        L.mco_cache_slots.argtypes = [vp]
        L.mco_cache_slots.restype = C.POINTER(C.c_uint64)
        L.mco_cache_counters.argtypes = [vp, vp]
        L.mco_execute_batch.argtypes = [C.POINTER(N.FlatScene), C.c_uint32, vp, C.c_size_t, vp,
                                        C.c_int, vp, vp, vp]
        L.mco_execute_batch_deferred.argtypes = [C.POINTER(N.FlatScene), C.c_uint32, vp,
                                                 C.c_size_t, vp, C.c_int, vp, vp, vp]
        L.mco_intersect_batch.argtypes = [C.POINTER(N.FlatScene), vp, C.c_size_t, C.c_float,
                                          C.c_float, vp]
        L.mco_occluded_batch.argtypes = [C.POINTER(N.FlatScene), vp, C.c_size_t, C.c_float, vp, vp]
        L.mco_camera_setup.argtypes = [C.POINTER(N.FlatScene), C.c_int, C.c_int, vp]
        L.mco_render.argtypes = [C.POINTER(N.FlatScene), C.POINTER(RenderParamsC), vp, vp, vp,
                                 vp, vp, C.POINTER(RenderStatsC)]

    def hash(self, desc):
        n = desc.shape[0]
        cell, chk = np.zeros(n, np.uint64), np.zeros(n, np.uint32)
        self.L.mco_hash_batch(ptr(desc), n, ptr(cell), ptr(chk))
        return cell, chk

    def encode(self, rgb):
        rgb = np.ascontiguousarray(rgb, np.float32)
        out = np.zeros(rgb.shape[0], np.uint32)
        self.L.mco_encode_batch(ptr(rgb), rgb.shape[0], ptr(out))
        return out

    def decode(self, packed):
        packed = np.ascontiguousarray(packed, np.uint32)
        out = np.zeros((packed.shape[0], 3), np.float32)
        self.L.mco_decode_batch(ptr(packed), packed.shape[0], ptr(out))
        return out

    def mip_texel(self, uv, g1, g2, off=0):
        uv, g1, g2 = (np.ascontiguousarray(a, np.float32) for a in (uv, g1, g2))
        n = uv.shape[0]
        mip, txy = np.zeros(n, np.uint8), np.zeros((n, 2), np.uint32)
        self.L.mco_mip_texel_batch(ptr(uv), ptr(g1), ptr(g2), n, off, ptr(mip), ptr(txy))
        return mip, txy

    def footprint(self, inp):
        inp = np.ascontiguousarray(inp, np.float32)
        out = np.zeros((inp.shape[0], 4), np.float32)
        self.L.mco_footprint_batch(ptr(inp), inp.shape[0], ptr(out))
        return out

    def fbm(self, octaves, fp, uv):
        octaves = np.ascontiguousarray(octaves, np.int32)
        fp, uv = np.ascontiguousarray(fp, np.float32), np.ascontiguousarray(uv, np.float32)
        out = np.zeros(octaves.shape[0], np.float32)
        self.L.mco_fbm_batch(ptr(octaves), ptr(fp), ptr(uv), octaves.shape[0], ptr(out))
        return out

    def sin_wave(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros_like(x)
        self.L.mco_sin_wave_batch(ptr(x), x.shape[0], ptr(out))
        return out

    def atan2f(self, y, x):
        y, x = np.ascontiguousarray(y, np.float32), np.ascontiguousarray(x, np.float32)
        out = np.zeros_like(x)
        self.L.mco_atan2f_batch(ptr(y), ptr(x), x.shape[0], ptr(out))
        return out

    def acosf(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros_like(x)
        self.L.mco_acosf_batch(ptr(x), x.shape[0], ptr(out))
        return out

    def power(self, x, y):
        x, y = np.ascontiguousarray(x, np.float32), np.ascontiguousarray(y, np.float32)
        out = np.zeros_like(x)
        self.L.mco_power_batch(ptr(x), ptr(y), x.shape[0], ptr(out))
        return out

    # table
    def cache_new(self, nc, ne):
        return self.L.mco_cache_new(nc, ne)

    def cache_free(self, c):
        self.L.mco_cache_free(c)

    def cache_update(self, c, desc, rgb):
        n = desc.shape[0]
        rgb = np.ascontiguousarray(rgb, np.float32)
        o, s, p = np.zeros(n, np.uint8), np.zeros(n, np.uint64), np.zeros(n, np.uint64)
        self.L.mco_cache_update_batch(c, ptr(desc), ptr(rgb), n, ptr(o), ptr(s), ptr(p))
        return o, s, p

    def cache_lookup(self, c, desc):
        n = desc.shape[0]
        hit, rgb = np.zeros(n, np.uint8), np.zeros((n, 3), np.float32)
        self.L.mco_cache_lookup_batch(c, ptr(desc), n, ptr(hit), ptr(rgb))
        return hit.astype(bool), rgb

    def cache_slots(self, c, nc, ne):
        p = self.L.mco_cache_slots(c)
        return np.ctypeslib.as_array(p, shape=(nc * ne,)).copy()

    def cache_counters(self, c):
        out = np.zeros(5, np.uint64)
        self.L.mco_cache_counters(c, ptr(out))
        return out

    def execute(self, flat, slot, sp, cache=None, mip_offset=0, deferred=False):
        sp = np.ascontiguousarray(sp, np.float32)
        n = sp.shape[0]
        vals, nodes, instr = np.zeros((n, 4), np.float32), np.zeros(n, np.uint32), np.zeros(n, np.uint32)
        fn = self.L.mco_execute_batch_deferred if deferred else self.L.mco_execute_batch
        fn(C.byref(flat), slot, ptr(sp), n, cache, mip_offset, ptr(vals), ptr(nodes), ptr(instr))
        return vals, nodes, instr

    def intersect(self, flat, rays, tmin=1e-4, tmax=np.inf):
        rays = np.ascontiguousarray(rays, np.float32)
        out = np.zeros((rays.shape[0], 24), np.float32)
        self.L.mco_intersect_batch(C.byref(flat), ptr(rays), rays.shape[0], tmin, tmax, ptr(out))
        return out

    def occluded(self, flat, rays, tmin, tmax):
        rays = np.ascontiguousarray(rays, np.float32)
        tmax = np.ascontiguousarray(tmax, np.float32)
        out = np.zeros(rays.shape[0], np.uint8)
        self.L.mco_occluded_batch(C.byref(flat), ptr(rays), rays.shape[0], tmin, ptr(tmax), ptr(out))
        return out

    def camera(self, flat, w, h):
        out = np.zeros(12, np.float32)
        self.L.mco_camera_setup(C.byref(flat), w, h, ptr(out))
        return out

    def render(self, flat, params: RenderParamsC, cache=None):
        w = params.width or flat.cam_width
        h = params.height or flat.cam_height
        rad, nodes, samples, hps = _render_outputs(w, h, params.spp)
        st = RenderStatsC()
        rc = self.L.mco_render(C.byref(flat), C.byref(params), cache, ptr(rad), ptr(nodes),
                               ptr(samples), ptr(hps), C.byref(st))
        assert rc == 0, "oracle render failed"
        return rad, nodes, samples, hps, st


class Ref:
    """The reference's compiled code (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        self.L = C.CDLL(path)
        L = self.L
        L.ref_last_error.restype = C.c_char_p
        L.ref_hash.argtypes = [vp, C.c_size_t, vp, vp]
        L.ref_encode.argtypes = [vp, C.c_size_t, vp]
        L.ref_decode.argtypes = [vp, C.c_size_t, vp]
        L.ref_mip_texel.argtypes = [vp, vp, vp, C.c_size_t, C.c_int, vp, vp]
        L.ref_footprint.argtypes = [vp, C.c_size_t, vp]
        L.ref_cone_spread.argtypes = [C.c_float, C.c_int]
        L.ref_cone_spread.restype = C.c_float
        L.ref_rng.argtypes = [C.c_uint64, vp, vp, vp, C.c_size_t, vp]
        L.ref_fbm.argtypes = [vp, vp, vp, C.c_size_t, vp]
        L.ref_perlin.argtypes = [vp, C.c_size_t, vp]
        L.ref_sin_wave.argtypes = [vp, C.c_size_t, vp]
        L.ref_power.argtypes = [vp, vp, C.c_size_t, vp]
        L.ref_checker.argtypes = [C.c_float, vp, C.c_size_t, vp]
        L.ref_bilinear.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, C.c_size_t, vp]
        L.ref_memory_bytes.argtypes = [C.c_uint64, C.c_uint64, vp]
        L.ref_write_ppm.argtypes = [C.c_char_p, C.c_int, C.c_int, vp, C.c_int]
        L.ref_write_pfm.argtypes = [C.c_char_p, C.c_int, C.c_int, vp]
        L.ref_read_pfm.argtypes = [C.c_char_p, vp, vp, vp]
        L.ref_cache_new.argtypes = [C.c_uint64, C.c_uint32, C.POINTER(vp)]
        L.ref_cache_free.argtypes = [vp]
        L.ref_cache_update.argtypes = [vp, vp, vp, C.c_size_t, vp, vp, vp]
        L.ref_cache_lookup.argtypes = [vp, vp, C.c_size_t, vp, vp]
        L.ref_cache_slots.argtypes = [vp, C.c_uint64, C.c_size_t, vp]
        L.ref_cache_counters.argtypes = [vp, vp]
        L.ref_probe_bench.argtypes = [vp, C.c_uint64, C.c_uint64, C.c_int, C.c_int]
        L.ref_probe_bench.restype = C.c_double
        L.ref_cache_dump.argtypes = [vp, C.c_char_p]
        L.ref_audit.argtypes = [C.c_char_p, vp, C.c_char_p, C.c_size_t]
        L.ref_scene_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
        L.ref_scene_free.argtypes = [vp]
        L.ref_scene_materials.argtypes = [vp]
        L.ref_scene_disassemble.argtypes = [vp, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.ref_scene_analysis_json.argtypes = [vp, C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.ref_scene_execute.argtypes = [vp, C.c_int, vp, C.c_size_t, vp, C.c_int, vp, vp, vp]
        L.ref_scene_eval_reference.argtypes = [vp, C.c_int, vp, C.c_size_t, vp]
        L.ref_scene_intersect.argtypes = [vp, vp, C.c_size_t, C.c_float, C.c_float, vp]
        L.ref_scene_occluded.argtypes = [vp, vp, C.c_size_t, C.c_float, vp, vp]
        L.ref_scene_bvh.argtypes = [vp, vp, C.c_size_t]
        L.ref_scene_bvh.restype = C.c_size_t
        L.ref_render.argtypes = [vp, C.POINTER(RenderParamsC), vp, vp, vp, vp, vp,
                                 C.POINTER(RenderStatsC)]

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def err(self):
        return self.L.ref_last_error().decode()

    def hash(self, desc):
        n = desc.shape[0]
        cell, chk = np.zeros(n, np.uint64), np.zeros(n, np.uint32)
        self.L.ref_hash(ptr(desc), n, ptr(cell), ptr(chk))
        return cell, chk

    def encode(self, rgb):
        rgb = np.ascontiguousarray(rgb, np.float32)
        out = np.zeros(rgb.shape[0], np.uint32)
        self.L.ref_encode(ptr(rgb), rgb.shape[0], ptr(out))
        return out

    def decode(self, packed):
        packed = np.ascontiguousarray(packed, np.uint32)
        out = np.zeros((packed.shape[0], 3), np.float32)
        self.L.ref_decode(ptr(packed), packed.shape[0], ptr(out))
        return out

    def mip_texel(self, uv, g1, g2, off=0):
        uv, g1, g2 = (np.ascontiguousarray(a, np.float32) for a in (uv, g1, g2))
        n = uv.shape[0]
        mip, txy = np.zeros(n, np.uint8), np.zeros((n, 2), np.uint32)
        self.L.ref_mip_texel(ptr(uv), ptr(g1), ptr(g2), n, off, ptr(mip), ptr(txy))
        return mip, txy

    def footprint(self, inp):
        inp = np.ascontiguousarray(inp, np.float32)
        out = np.zeros((inp.shape[0], 4), np.float32)
        self.L.ref_footprint(ptr(inp), inp.shape[0], ptr(out))
        return out

    def rng(self, seed, pixel, sample, dim):
        pixel = np.ascontiguousarray(pixel, np.uint64)
        sample = np.ascontiguousarray(sample, np.uint64)
        dim = np.ascontiguousarray(dim, np.uint32)
        out = np.zeros(pixel.shape[0], np.float32)
        self.L.ref_rng(seed, ptr(pixel), ptr(sample), ptr(dim), pixel.shape[0], ptr(out))
        return out

    def fbm(self, octaves, fp, uv):
        octaves = np.ascontiguousarray(octaves, np.int32)
        fp, uv = np.ascontiguousarray(fp, np.float32), np.ascontiguousarray(uv, np.float32)
        out = np.zeros(octaves.shape[0], np.float32)
        self.L.ref_fbm(ptr(octaves), ptr(fp), ptr(uv), octaves.shape[0], ptr(out))
        return out

    def sin_wave(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros_like(x)
        self.L.ref_sin_wave(ptr(x), x.shape[0], ptr(out))
        return out

    def power(self, x, y):
        x, y = np.ascontiguousarray(x, np.float32), np.ascontiguousarray(y, np.float32)
        out = np.zeros_like(x)
        self.L.ref_power(ptr(x), ptr(y), x.shape[0], ptr(out))
        return out

    def probe_bench(self, c, n, seed, phase, threads):
        """Seconds for n reference update() (phase 0) / lookup() (phase 1)
        calls over `threads` host threads (ref_probe_bench)."""
        return float(self.L.ref_probe_bench(c, n, seed, phase, threads))

    def cache_new(self, nc, ne):
        h = vp()
        rc = self.L.ref_cache_new(nc, ne, C.byref(h))
        if rc:
            raise {1: ValueError, 2: OverflowError}.get(rc, RuntimeError)(self.err())
        return h

    def cache_free(self, c):
        self.L.ref_cache_free(c)

    def cache_update(self, c, desc, rgb):
        n = desc.shape[0]
        rgb = np.ascontiguousarray(rgb, np.float32)
        o, s, p = np.zeros(n, np.uint8), np.zeros(n, np.uint64), np.zeros(n, np.uint64)
        self.L.ref_cache_update(c, ptr(desc), ptr(rgb), n, ptr(o), ptr(s), ptr(p))
        return o, s, p

    def cache_lookup(self, c, desc):
        n = desc.shape[0]
        hit, rgb = np.zeros(n, np.uint8), np.zeros((n, 3), np.float32)
        self.L.ref_cache_lookup(c, ptr(desc), n, ptr(hit), ptr(rgb))
        return hit.astype(bool), rgb

    def cache_slots(self, c, n):
        out = np.zeros(n, np.uint64)
        self.L.ref_cache_slots(c, 0, n, ptr(out))
        return out

    def cache_counters(self, c):
        out = np.zeros(5, np.uint64)
        self.L.ref_cache_counters(c, ptr(out))
        return out

    def scene_load(self, path, min_subtree=3):
        h = vp()
        rc = self.L.ref_scene_load(os.fsencode(path), min_subtree, C.byref(h))
        if rc:
            raise {3: N.GraphError, 4: N.CompileError, 5: N.SceneError, 6: N.ImageIoError}.get(
                rc, RuntimeError)(self.err())
        return h

    def _text(self, fn, s, slot):
        n = C.c_size_t()
        fn(s, slot, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        fn(s, slot, buf, n.value + 1, C.byref(n))
        return buf.value.decode()

    def disassemble(self, s, slot):
        return self._text(self.L.ref_scene_disassemble, s, slot)

    def analysis_json(self, s, slot):
        return self._text(self.L.ref_scene_analysis_json, s, slot)

    def execute(self, s, slot, sp, cache=None, mip_offset=0):
        sp = np.ascontiguousarray(sp, np.float32)
        n = sp.shape[0]
        vals, nodes, instr = np.zeros((n, 4), np.float32), np.zeros(n, np.uint32), np.zeros(n, np.uint32)
        self.L.ref_scene_execute(s, slot, ptr(sp), n, cache, mip_offset, ptr(vals), ptr(nodes), ptr(instr))
        return vals, nodes, instr

    def eval_reference(self, s, slot, sp):
        sp = np.ascontiguousarray(sp, np.float32)
        vals = np.zeros((sp.shape[0], 4), np.float32)
        self.L.ref_scene_eval_reference(s, slot, ptr(sp), sp.shape[0], ptr(vals))
        return vals

    def intersect(self, s, rays, tmin=1e-4, tmax=np.inf):
        rays = np.ascontiguousarray(rays, np.float32)
        out = np.zeros((rays.shape[0], 24), np.float32)
        self.L.ref_scene_intersect(s, ptr(rays), rays.shape[0], tmin, tmax, ptr(out))
        return out

    def bvh(self, s):
        """The reference Scene's BVH nodes as (n, 10) uint32: min, max (float
        bits), left, right, first, count."""
        n = self.L.ref_scene_bvh(s, None, 0)
        out = np.zeros((n, 10), np.uint32)
        self.L.ref_scene_bvh(s, ptr(out), n)
        return out

    def occluded(self, s, rays, tmin, tmax):
        rays = np.ascontiguousarray(rays, np.float32)
        tmax = np.ascontiguousarray(tmax, np.float32)
        out = np.zeros(rays.shape[0], np.uint8)
        self.L.ref_scene_occluded(s, ptr(rays), rays.shape[0], tmin, ptr(tmax), ptr(out))
        return out

    def render(self, s, params: RenderParamsC, w, h, cache=None):
        rad, nodes, samples, hps = _render_outputs(w, h, params.spp)
        st = RenderStatsC()
        rc = self.L.ref_render(s, C.byref(params), cache, ptr(rad), ptr(nodes), ptr(samples),
                               ptr(hps), C.byref(st))
        if rc:
            raise RuntimeError(self.err())
        return rad, nodes, samples, hps, st
