"""B200-native progressive material caching (arXiv 2305.07238 hot path).

Python mirror of the reference's renderer API (/root/reference/proj/core/
include/matcache): ``load_scene`` (scene.hpp:127), ``RenderConfig`` /
``FrameBuffers`` / ``RenderStats`` / ``render`` (tracer.hpp:7-70),
``MaterialCache`` (cache.hpp:69-115), the descriptor hashes and RGBE codec
(cache.hpp:28-46), ``audit_dump`` (cache.hpp:128) and the experiment outputs
``image_error`` / ``stats_to_json`` / ``parse_stats_json`` (tracer.hpp:72-92).

Every call goes through the C ABI of libmcg.so (include/mcg.h); material
evaluation, cache probes and inserts, ray generation and BVH traversal run in
hand-written sm_100a kernels. There is no CPU fallback: without the built
library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from ._native import (CompileError, CudaError, GraphError, ImageIoError, MCGError,  # noqa: F401
                      NoDeviceError, SceneError, check)

__all__ = [
    "Context", "Scene", "load_scene", "MaterialCache", "RenderConfig", "FrameBuffers",
    "RenderStats", "RenderResult", "render", "hash_cell", "hash_check", "encode_value",
    "decode_value", "memory_bytes", "audit_dump", "AuditReport", "image_error", "DiffStats",
    "stats_to_json", "parse_stats_json", "GraphError", "CompileError", "SceneError",
    "ImageIoError", "CudaError", "NoDeviceError", "CACHE_OFF", "CACHE_CONCURRENT",
    "CACHE_DETERMINISTIC", "artifacts", "sweep", "SweepRow",
]

CACHE_OFF, CACHE_CONCURRENT, CACHE_DETERMINISTIC = 0, 1, 2
INSERT_OUTCOMES = ("Won", "LostRace", "AlreadyPresent", "CellFull")  # cache.hpp:51-56

DESC_DTYPE = np.dtype([("mat_idx", "<u4"), ("node_idx", "<u4"), ("mip_level", "u1"),
                       ("pad_", "u1", 3), ("texel_x", "<u4"), ("texel_y", "<u4")])
assert DESC_DTYPE.itemsize == 20
INSERT_RECORD_DTYPE = np.dtype([("desc", DESC_DTYPE), ("entry", "<u4"), ("payload", "<u4")])  # mcg_insert_record
assert INSERT_RECORD_DTYPE.itemsize == 28


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def descriptors(mat, node, mip, tx, ty) -> np.ndarray:
    """Array of CacheDescriptor records (cache.hpp:17-25)."""
    mat = np.atleast_1d(np.asarray(mat, np.uint32))
    n = mat.shape[0]
    d = np.zeros(n, DESC_DTYPE)
    d["mat_idx"] = mat
    d["node_idx"] = np.broadcast_to(np.asarray(node, np.uint32), (n,))
    d["mip_level"] = np.broadcast_to(np.asarray(mip, np.uint8), (n,))
    d["texel_x"] = np.broadcast_to(np.asarray(tx, np.uint32), (n,))
    d["texel_y"] = np.broadcast_to(np.asarray(ty, np.uint32), (n,))
    return d


# --------------------------------------------------------------------------
# Host helpers (no device needed)
# --------------------------------------------------------------------------

def _one_desc(d) -> N.Descriptor:
    if isinstance(d, np.void) or (isinstance(d, np.ndarray) and d.dtype == DESC_DTYPE):
        d = tuple(int(d[k]) for k in ("mat_idx", "node_idx", "mip_level", "texel_x", "texel_y"))
    mat, node, mip, tx, ty = d
    r = N.Descriptor()
    r.mat_idx, r.node_idx, r.mip_level, r.texel_x, r.texel_y = mat, node, mip, tx, ty
    return r


def hash_cell(desc) -> int:
    """hash_cell (cache.cpp:34); desc = (mat, node, mip, tx, ty)."""
    return int(N.lib().mcg_hash_cell(C.byref(_one_desc(desc))))


def hash_check(desc) -> int:
    """hash_check (cache.cpp:36-39); never 0."""
    return int(N.lib().mcg_hash_check(C.byref(_one_desc(desc))))


def encode_value(rgb: Sequence[float]) -> int:
    """encode_value (cache.cpp:41-61): shared-exponent RGBE word."""
    a = (C.c_float * 3)(*[float(x) for x in rgb])
    return int(N.lib().mcg_encode_value(a))


def decode_value(packed: int) -> tuple[float, float, float]:
    """decode_value (cache.cpp:63-71)."""
    a = (C.c_float * 3)()
    N.lib().mcg_decode_value(C.c_uint32(packed), a)
    return (a[0], a[1], a[2])


def memory_bytes(n_cells: int, n_entries: int) -> int:
    """memory_bytes (cache.cpp:73-80); OverflowError when it does not fit."""
    out = C.c_uint64()
    check(N.lib().mcg_memory_bytes(n_cells, n_entries, C.byref(out)))
    return int(out.value)


@dataclass
class AuditReport:
    """AuditReport (cache.hpp:117-124)."""
    n_cells: int = 0
    n_entries: int = 0
    occupied: int = 0
    clean: bool = False
    problem: str = ""
    bad_cell: int = -1


def audit_dump(path: str) -> AuditReport:
    """audit_dump (cache.cpp:175-230)."""
    r = N.AuditReport()
    check(N.lib().mcg_audit_dump(os.fsencode(path), C.byref(r)))
    return AuditReport(r.n_cells, r.n_entries, r.occupied, bool(r.clean),
                       r.problem.decode(errors="replace"), r.bad_cell)


# --------------------------------------------------------------------------
# Device context
# --------------------------------------------------------------------------

class Context:
    """One CUDA device + stream (mcg_ctx). ``profile=True`` times every kernel
    launch with CUDA events on the context's stream. ``devices=[...]``: one
    context over several GPUs (include/mcg.h mcg_options.n_devices): render()
    deals the image's 16x16 tiles to the devices, one host thread and cache
    replica each, and gathers the frames with NCCL on the first device."""

    _defaults: dict[int, "Context"] = {}

    def __init__(self, device: int = 0, profile: bool = False, stream: Optional[int] = None,
                 devices: Optional[Sequence[int]] = None):
        devs = [int(d) for d in devices] if devices else []
        arr = (C.c_int32 * len(devs))(*devs) if devs else None
        opt = N.Options(devs[0] if devs else device, 1 if profile else 0,
                        C.c_void_p(stream) if stream else None, len(devs),
                        C.cast(arr, C.POINTER(C.c_int32)) if arr is not None else None)
        h = C.c_void_p()
        check(N.lib().mcg_create(C.byref(opt), C.byref(h)))
        self.handle = h
        self.device = devs[0] if devs else device
        self.devices = devs or [device]
        self._scene = None

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._defaults:
            cls._defaults[device] = cls(device)
        return cls._defaults[device]

    def close(self) -> None:
        if self.handle:
            N.lib().mcg_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return N.lib().mcg_stream(self.handle) or 0

    def synchronize(self) -> None:
        check(N.lib().mcg_synchronize(self.handle))

    def launch_count(self) -> int:
        return int(N.lib().mcg_launch_count(self.handle))

    def kernel_times(self) -> dict[str, dict]:
        buf = (N.KernelTime * 128)()
        n = C.c_int32()
        check(N.lib().mcg_kernel_times(self.handle, buf, 128, C.byref(n)))
        return {buf[i].name.decode(): {"launches": buf[i].launches, "ms": buf[i].ms,
                                       "bytes": buf[i].algorithmic_bytes}
                for i in range(min(n.value, 128))}

    def reset_kernel_times(self) -> None:
        check(N.lib().mcg_kernel_times_reset(self.handle))

    def upload(self, scene: "Scene") -> None:
        check(N.lib().mcg_upload_scene(self.handle, scene.handle))
        self._scene = scene

    # Batched descriptor pipeline on the device (parity surface).
    def hash_batch(self, desc: np.ndarray):
        desc = np.ascontiguousarray(desc, DESC_DTYPE)
        n = desc.shape[0]
        cell = np.zeros(n, np.uint64)
        chk = np.zeros(n, np.uint32)
        check(N.lib().mcg_hash_batch(self.handle, _ptr(desc), n, _ptr(cell), _ptr(chk)))
        return cell, chk

    def encode_batch(self, rgb: np.ndarray) -> np.ndarray:
        rgb = np.ascontiguousarray(rgb, np.float32).reshape(-1, 3)
        out = np.zeros(rgb.shape[0], np.uint32)
        check(N.lib().mcg_encode_batch(self.handle, _ptr(rgb), rgb.shape[0], _ptr(out)))
        return out

    def decode_batch(self, packed: np.ndarray) -> np.ndarray:
        packed = np.ascontiguousarray(packed, np.uint32)
        out = np.zeros((packed.shape[0], 3), np.float32)
        check(N.lib().mcg_decode_batch(self.handle, _ptr(packed), packed.shape[0], _ptr(out)))
        return out

    def mip_texel_batch(self, uv, g1, g2, mip_offset: int = 0):
        uv = np.ascontiguousarray(uv, np.float32).reshape(-1, 2)
        g1 = np.ascontiguousarray(g1, np.float32).reshape(-1, 2)
        g2 = np.ascontiguousarray(g2, np.float32).reshape(-1, 2)
        n = uv.shape[0]
        mip = np.zeros(n, np.uint8)
        txy = np.zeros((n, 2), np.uint32)
        check(N.lib().mcg_mip_texel_batch(self.handle, _ptr(uv), _ptr(g1), _ptr(g2), n,
                                          mip_offset, _ptr(mip), _ptr(txy)))
        return mip, txy

    def execute_batch(self, slot: int, sp: np.ndarray, cache: "MaterialCache" = None,
                      cache_mode: int = CACHE_CONCURRENT, mip_offset: int = 0):
        """execute (stackvm.cpp:248-368) for n shading points (n x 15 floats)
        of material `slot` of the uploaded scene."""
        sp = np.ascontiguousarray(sp, np.float32).reshape(-1, 15)
        n = sp.shape[0]
        vals = np.zeros((n, 4), np.float32)
        nodes = np.zeros(n, np.uint32)
        instrs = np.zeros(n, np.uint32)
        check(N.lib().mcg_execute_batch(self.handle, slot, _ptr(sp), n,
                                        cache.handle if cache is not None else None,
                                        cache_mode if cache is not None else CACHE_OFF,
                                        mip_offset, _ptr(vals), _ptr(nodes), _ptr(instrs)))
        return vals, nodes, instrs

    def intersect_batch(self, rays: np.ndarray, t_min: float = 1e-4, t_max: float = np.inf,
                        variant: int = 3) -> np.ndarray:
        """Scene::intersect (scene.cpp:252-278) on the uploaded scene for n
        rays (n x 6: origin, direction) -> n x 24 floats (found, t, position,
        normal, uv, slot, e1, e2, duv1, duv2). variant: the traversal
        (0 per-thread DFS, 1 child pairs, 2 4-wide, 3 speculative 4-wide, 4 packets)."""
        rays = np.ascontiguousarray(rays, np.float32).reshape(-1, 6)
        out = np.zeros((rays.shape[0], 24), np.float32)
        check(N.lib().mcg_intersect_batch(self.handle, _ptr(rays), rays.shape[0], t_min, t_max,
                                          variant, _ptr(out)))
        return out

    def occluded_batch(self, rays: np.ndarray, t_min: float, t_max: np.ndarray,
                       variant: int = 3) -> np.ndarray:
        """Scene::occluded (scene.cpp:280-298) per ray with its own t_max."""
        rays = np.ascontiguousarray(rays, np.float32).reshape(-1, 6)
        t_max = np.ascontiguousarray(t_max, np.float32).reshape(-1)
        out = np.zeros(rays.shape[0], np.uint8)
        check(N.lib().mcg_occluded_batch(self.handle, _ptr(rays), rays.shape[0], t_min, _ptr(t_max),
                                         variant, _ptr(out)))
        return out


    def shadow_tree(self):
        """The uploaded scene's any-hit hierarchy (include/mcg.h mcg_shadow_tree):
        ((n, 4) structured array of mcg_bvh_node entries, (root_a, root_b))."""
        n, ra, rb = C.c_size_t(), C.c_int32(), C.c_int32()
        check(N.lib().mcg_shadow_tree(self.handle, None, 0, C.byref(n), C.byref(ra), C.byref(rb)))
        dt = np.dtype([("lo", np.float32, 3), ("a", np.int32), ("hi", np.float32, 3), ("b", np.int32)])
        out = np.zeros(n.value * 4, dt)
        check(N.lib().mcg_shadow_tree(self.handle, _ptr(out), out.shape[0], C.byref(n), C.byref(ra),
                                      C.byref(rb)))
        return out.reshape(-1, 4), (ra.value, rb.value)


# --------------------------------------------------------------------------
# Material cache (cache.hpp:69-115), resident in HBM
# --------------------------------------------------------------------------

class MaterialCache:
    """Nc x Ne table of 64-bit slots ``(hash_check << 32) | rgbe``; 0 = empty."""

    APPLY_CONCURRENT, APPLY_ORDERED = 0, 1

    def __init__(self, n_cells: int, n_entries: int, ctx: Optional[Context] = None, *,
                 rank: int = 0, world: int = 1):
        self.ctx = ctx or Context.default()
        h = C.c_void_p()
        if world == 1:
            check(N.lib().mcg_cache_create(self.ctx.handle, int(n_cells), int(n_entries), C.byref(h)))
        else:
            check(N.lib().mcg_cache_create_stripe(self.ctx.handle, int(n_cells), int(n_entries), int(rank),
                                                  int(world), C.byref(h)))
        self.handle = h
        self.n_cells, self.n_entries = int(n_cells), int(n_entries)
        self.rank, self.world = int(rank), int(world)

    # ---- striped shared table (include/mcg.h) ----
    @classmethod
    def stripe(cls, n_cells: int, n_entries: int, rank: int, world: int,
               ctx: Optional[Context] = None) -> "MaterialCache":
        """This device's stripe of one logical n_cells x n_entries table
        shared by `world` GPUs (cells c with c % world == rank)."""
        return cls(n_cells, n_entries, ctx, rank=rank, world=world)

    def local_cells(self) -> int:
        out = C.c_uint64()
        check(N.lib().mcg_cache_stripe_info(self.handle, None, None, C.byref(out)))
        return int(out.value)

    def attach_local(self, stripes: Sequence["MaterialCache"]) -> None:
        """Address the other stripes directly (same process: peers or, on one
        GPU, an emulated striped table)."""
        arr = (C.c_void_p * len(stripes))(*[st.handle.value for st in stripes])
        check(N.lib().mcg_cache_attach_local(self.handle, arr, len(stripes)))

    def ipc_handle(self) -> bytes:
        """CUDA IPC handle of this stripe (64 bytes) for the other ranks."""
        buf = C.create_string_buffer(64)
        check(N.lib().mcg_cache_ipc_handle(self.handle, buf, 64))
        return buf.raw

    def attach_ipc(self, handles: Sequence[bytes]) -> None:
        """Map every rank's stripe (handles in rank order; own entry ignored)."""
        blob = b"".join(bytes(h).ljust(64, b"\0")[:64] for h in handles)
        buf = C.create_string_buffer(blob, len(blob))
        check(N.lib().mcg_cache_attach_ipc(self.handle, buf, len(handles)))

    def close(self) -> None:
        if getattr(self, "handle", None):
            N.lib().mcg_cache_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def slot_count(self) -> int:
        """Slots held by this object (this stripe's, for a striped table)."""
        return (self.n_cells if self.world == 1 else self.local_cells()) * self.n_entries

    def bytes(self) -> int:
        return self.slot_count() * 8

    def clear(self) -> None:
        check(N.lib().mcg_cache_clear(self.handle))

    def update_batch(self, desc: np.ndarray, rgb: np.ndarray, ordered: bool = True):
        """update() for every element; ordered=True applies them as one thread
        in array order (lowest index wins), else all at once (concurrent CAS)."""
        desc = np.ascontiguousarray(desc, DESC_DTYPE)
        rgb = np.ascontiguousarray(rgb, np.float32).reshape(-1, 3)
        n = desc.shape[0]
        outcome = np.zeros(n, np.uint8)
        slot = np.zeros(n, np.uint64)
        packed = np.zeros(n, np.uint64)
        check(N.lib().mcg_cache_update_batch(self.handle, _ptr(desc), _ptr(rgb), n,
                                             1 if ordered else 0, _ptr(outcome), _ptr(slot),
                                             _ptr(packed)))
        return outcome, slot, packed

    def lookup_batch(self, desc: np.ndarray):
        desc = np.ascontiguousarray(desc, DESC_DTYPE)
        n = desc.shape[0]
        hit = np.zeros(n, np.uint8)
        rgb = np.zeros((n, 3), np.float32)
        check(N.lib().mcg_cache_lookup_batch(self.handle, _ptr(desc), n, _ptr(hit), _ptr(rgb)))
        return hit.astype(bool), rgb

    def update(self, desc, value):
        """UpdateResult as (outcome name, slot, packed) (cache.cpp:94-119)."""
        o, s, p = self.update_batch(np.array([_one_desc_tuple(desc)], DESC_DTYPE),
                                    np.asarray([value], np.float32))
        return INSERT_OUTCOMES[int(o[0])], int(s[0]), int(p[0])

    def lookup(self, desc):
        """Decoded rgb on a hit, else None (cache.cpp:121-136)."""
        hit, rgb = self.lookup_batch(np.array([_one_desc_tuple(desc)], DESC_DTYPE))
        return tuple(float(x) for x in rgb[0]) if hit[0] else None

    def slot_words(self, first: int = 0, n: Optional[int] = None) -> np.ndarray:
        n = self.slot_count() - first if n is None else n
        out = np.zeros(n, np.uint64)
        check(N.lib().mcg_cache_read_slots(self.handle, first, n, _ptr(out)))
        return out

    def slot_word(self, slot: int) -> int:
        return int(self.slot_words(slot, 1)[0])

    def write_slots(self, words: np.ndarray, first: int = 0) -> None:
        """Host words -> slots [first, first + len(words)) (seeding a table)."""
        words = np.ascontiguousarray(words, np.uint64)
        check(N.lib().mcg_cache_write_slots(self.handle, int(first), words.shape[0], _ptr(words)))

    # ---- won-insert log (include/mcg.h mcg_cache_insert_log_*) ----
    def insert_log_start(self, capacity: int) -> None:
        check(N.lib().mcg_cache_insert_log_start(self.handle, int(capacity)))

    def insert_log_stop(self) -> int:
        out = C.c_uint64()
        check(N.lib().mcg_cache_insert_log_stop(self.handle, C.byref(out)))
        return int(out.value)

    def insert_log_read(self, n: int, first: int = 0) -> np.ndarray:
        """Records (desc fields, entry, payload) as a structured array."""
        out = np.zeros(max(0, n), INSERT_RECORD_DTYPE)
        check(N.lib().mcg_cache_insert_log_read(self.handle, int(first), out.shape[0], _ptr(out)))
        return out

    def occupied_slots(self) -> int:
        out = C.c_uint64()
        check(N.lib().mcg_cache_occupied(self.handle, C.byref(out)))
        return int(out.value)

    def counters(self) -> dict:
        c = N.CacheCounters()
        check(N.lib().mcg_cache_counters_get(self.handle, C.byref(c)))
        return {"lookups": c.lookups, "hits": c.hits, "inserts_won": c.inserts_won,
                "inserts_lost_full": c.inserts_lost_full}

    def reset_counters(self) -> None:
        check(N.lib().mcg_cache_counters_reset(self.handle))

    def dump(self, path: str) -> None:
        check(N.lib().mcg_cache_dump(self.handle, os.fsencode(path)))

    # ---- descriptor trace ----
    def trace_start(self, capacity: int) -> None:
        """Record the descriptors of the lookups made through this table."""
        check(N.lib().mcg_cache_trace_start(self.handle, int(capacity)))

    def trace_stop(self) -> int:
        out = C.c_uint64()
        check(N.lib().mcg_cache_trace_stop(self.handle, C.byref(out)))
        return int(out.value)

    def trace_read(self, first: int = 0, n: Optional[int] = None, recorded: Optional[int] = None) -> np.ndarray:
        n = (recorded if recorded is not None else 0) - first if n is None else n
        out = np.zeros(max(0, n), DESC_DTYPE)
        check(N.lib().mcg_cache_trace_read(self.handle, first, out.shape[0], _ptr(out)))
        return out

    def probe_replay(self, desc: np.ndarray, blocks_per_sm: int = 8):
        """Lookup + insert-on-miss of `desc` in order; (ms, algorithmic bytes, counters)."""
        desc = np.ascontiguousarray(desc, DESC_DTYPE)
        ms, by = C.c_double(), C.c_double()
        cc = N.CacheCounters()
        check(N.lib().mcg_probe_replay(self.handle, _ptr(desc), desc.shape[0], blocks_per_sm, C.byref(ms),
                                       C.byref(by), C.byref(cc)))
        return ms.value, by.value, {"lookups": cc.lookups, "hits": cc.hits, "inserts_won": cc.inserts_won,
                                    "inserts_lost_full": cc.inserts_lost_full}

    def probe_bench(self, n: int, seed: int, phase: int, iters: int = 1):
        ms, by = C.c_double(), C.c_double()
        check(N.lib().mcg_probe_bench(self.handle, n, seed, phase, iters, C.byref(ms), C.byref(by)))
        return ms.value, by.value


def _one_desc_tuple(d):
    if isinstance(d, (tuple, list)):
        mat, node, mip, tx, ty = d
        return (mat, node, mip, (0, 0, 0), tx, ty)
    return d


# --------------------------------------------------------------------------
# Scenes (scene.hpp:91-127)
# --------------------------------------------------------------------------

class Scene:
    """A loaded, analyzed and compiled scene (host side)."""

    def __init__(self, handle):
        self.handle = handle
        f = N.FlatScene()
        check(N.lib().mcg_scene_flat(handle, C.byref(f)))
        self.flat = f

    def __del__(self):  # pragma: no cover
        try:
            if self.handle:
                N.lib().mcg_scene_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    @property
    def n_materials(self) -> int:
        return self.flat.n_programs

    @property
    def camera_size(self) -> tuple[int, int]:
        return self.flat.cam_width, self.flat.cam_height

    def program(self, slot: int) -> dict:
        p = self.flat.programs[slot]
        return {"material_id": p.material_id, "code_len": p.code_len,
                "max_stack": p.max_stack, "cache_point_count": p.cache_point_count}

    def _text(self, fn, slot: int) -> str:
        n = C.c_size_t()
        check(fn(self.handle, slot, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(fn(self.handle, slot, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def disassemble(self, slot: int) -> str:
        """disassemble(program) (stackvm.cpp:370-443)."""
        return self._text(N.lib().mcg_scene_disassemble, slot)

    def analysis_json(self, slot: int) -> str:
        """analysis_to_json (analysis.cpp:160-184)."""
        return self._text(N.lib().mcg_scene_analysis_json, slot)

    def camera_setup(self, width: int, height: int) -> np.ndarray:
        out = (C.c_float * 12)()
        check(N.lib().mcg_camera_setup(C.byref(self.flat), width, height, out))
        return np.array(out[:], np.float32)


def load_scene(path: str, min_subtree_size: int = 3) -> Scene:
    """load_scene (scene.cpp:300-387): JSON scene + materials + PPM textures,
    analyzed (AnalysisOptions.min_subtree_size) and compiled."""
    h = C.c_void_p()
    check(N.lib().mcg_scene_load(os.fsencode(path), min_subtree_size, C.byref(h)))
    return Scene(h)


# --------------------------------------------------------------------------
# render (tracer.hpp:7-70)
# --------------------------------------------------------------------------

@dataclass
class RenderConfig:
    """RenderConfig (tracer.hpp:7-20) plus the B200 path's knobs."""
    width: int = 0
    height: int = 0
    spp: int = 16
    max_bounces: int = 4
    threads: int = 0                 # accepted for API parity; the GPU ignores it
    cache_enabled: bool = False
    n_cells: int = 1 << 20
    n_entries: int = 8
    mip_offset: int = 0
    rng_seed: int = 1
    diffuse_spread: float = 0.2
    tile_size: int = 16
    deterministic: bool = False      # epoch-deferred inserts
    samples_per_pass: int = 0        # 0 = auto
    first_sample: int = 0
    shard_rank: int = 0
    shard_count: int = 1
    shard_mode: int = 0              # 0 interleaved tiles, 1 contiguous bands

    def cache_mode(self) -> int:
        if not self.cache_enabled:
            return CACHE_OFF
        return CACHE_DETERMINISTIC if self.deterministic else CACHE_CONCURRENT

    def to_params(self) -> N.RenderParams:
        return N.RenderParams(self.width, self.height, self.spp, self.max_bounces,
                              self.cache_mode(), self.mip_offset, self.n_cells, self.n_entries,
                              self.first_sample, self.rng_seed, self.diffuse_spread,
                              self.tile_size, self.shard_rank, self.shard_count, self.shard_mode,
                              self.samples_per_pass)


@dataclass
class FrameBuffers:
    """FrameBuffers (tracer.hpp:24-43): double accumulators per pixel."""
    width: int
    height: int
    radiance: np.ndarray = None      # (H, W, 3) float64
    nodes_found: np.ndarray = None   # (H, W) float64
    samples: np.ndarray = None       # (H, W) uint32

    def __post_init__(self):
        if self.radiance is None:
            self.radiance = np.zeros((self.height, self.width, 3), np.float64)
            self.nodes_found = np.zeros((self.height, self.width), np.float64)
            self.samples = np.zeros((self.height, self.width), np.uint32)

    def radiance_image(self) -> np.ndarray:
        s = np.maximum(self.samples, 1)[..., None].astype(np.float64)
        return (self.radiance / s).astype(np.float32)

    def nodes_found_avg(self) -> np.ndarray:
        s = np.maximum(self.samples, 1).astype(np.float64)
        return (self.nodes_found / s).astype(np.float32)

    def mean_radiance(self) -> np.ndarray:
        return self.radiance_image().reshape(-1, 3).mean(axis=0)


@dataclass
class RenderStats:
    """RenderStats (tracer.hpp:45-55) plus device-side work counters."""
    wall_time_s: float = 0.0
    lookups: int = 0
    hits: int = 0
    hit_rate: float = 0.0
    inserts_won: int = 0
    inserts_lost_full: int = 0
    stores_attempted: int = 0
    instructions_executed: int = 0
    hits_per_sample: list = field(default_factory=list)
    shading_points: int = 0
    shadow_rays: int = 0
    paths: int = 0
    device_ms: float = 0.0       # CUDA-event time of the render on the context's stream
    shadow_occluded: int = 0     # shadow rays that found an occluder
    bvh_nodes: int = 0           # traversal work: closest hit + shadow rays
    prims_tested: int = 0
    bvh_nodes_shadow: int = 0
    prims_tested_shadow: int = 0
    closest_rays: int = 0
    tex_samples: int = 0


@dataclass
class RenderResult:
    frame: FrameBuffers
    stats: RenderStats


def render(scene: Scene, config: RenderConfig, external_cache: Optional[MaterialCache] = None,
           ctx: Optional[Context] = None, frame: Optional[FrameBuffers] = None) -> RenderResult:
    """render(scene, config, external_cache) (tracer.hpp:69-70) on the GPU.
    Host framebuffers in, host framebuffers out (the copies are part of the
    call, as for the reference's caller)."""
    ctx = ctx or (external_cache.ctx if external_cache is not None else Context.default())
    if ctx._scene is not scene:
        ctx.upload(scene)
    w = config.width or scene.flat.cam_width
    h = config.height or scene.flat.cam_height
    fb = frame or FrameBuffers(w, h)
    fr = N.Frame(fb.radiance.ctypes.data_as(C.POINTER(C.c_double)),
                 fb.nodes_found.ctypes.data_as(C.POINTER(C.c_double)),
                 fb.samples.ctypes.data_as(C.POINTER(C.c_uint32)))
    hps = np.zeros(config.spp, np.uint64)
    st = N.RenderStats()
    st.hits_per_sample = hps.ctypes.data_as(C.POINTER(C.c_uint64))
    params = config.to_params()
    check(N.lib().mcg_render(ctx.handle, C.byref(params),
                             external_cache.handle if external_cache is not None else None,
                             C.byref(fr), C.byref(st)))
    stats = RenderStats(st.wall_time_s, st.lookups, st.hits,
                        (st.hits / st.lookups) if st.lookups else 0.0, st.inserts_won,
                        st.inserts_lost_full, st.stores_attempted, st.instructions_executed,
                        [int(x) for x in hps], st.shading_points, st.shadow_rays, st.paths,
                        st.device_ms, st.shadow_occluded, st.bvh_nodes, st.prims_tested,
                        st.bvh_nodes_shadow, st.prims_tested_shadow, st.closest_rays, st.tex_samples)
    return RenderResult(fb, stats)


# --------------------------------------------------------------------------
# Experiment outputs (tracer.hpp:72-92)
# --------------------------------------------------------------------------

@dataclass
class DiffStats:
    mean_abs: float
    max_abs: float
    diff: np.ndarray   # clamp(scale * |a - b|, 0, 1)


def image_error(a: np.ndarray, b: np.ndarray, scale: float = 5.0) -> DiffStats:
    """image_error (tracer.hpp:72-80): ValueError on a resolution mismatch."""
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    if a.shape != b.shape:
        raise ValueError(f"image_error: resolution mismatch {a.shape} vs {b.shape}")
    d = np.abs(a.astype(np.float64) - b.astype(np.float64))
    return DiffStats(float(d.mean()) if d.size else 0.0, float(d.max()) if d.size else 0.0,
                     np.clip(np.float32(scale) * d.astype(np.float32), 0.0, 1.0))


def stats_to_json(stats: RenderStats, frame: FrameBuffers) -> str:
    """Stats JSON (tracer.hpp:82-86)."""
    doc = {
        "wall_time_s": stats.wall_time_s, "hits": stats.hits, "lookups": stats.lookups,
        "hit_rate": stats.hit_rate, "inserts_won": stats.inserts_won,
        "inserts_lost_full": stats.inserts_lost_full, "width": frame.width,
        "height": frame.height,
        "per_pixel_nodes_found": [float(x) for x in frame.nodes_found_avg().reshape(-1)],
    }
    return json.dumps(doc)


@dataclass
class StatsFile:
    width: int
    height: int
    per_pixel_nodes_found: np.ndarray


def parse_stats_json(text: str) -> StatsFile:
    """parse_stats_json (tracer.hpp:88-92)."""
    doc = json.loads(text)
    if "per_pixel_nodes_found" not in doc:
        raise ValueError("stats JSON lacks per_pixel_nodes_found")
    w, h = int(doc["width"]), int(doc["height"])
    v = np.asarray(doc["per_pixel_nodes_found"], np.float32)
    if v.size != w * h:
        raise ValueError("per_pixel_nodes_found size does not match width*height")
    return StatsFile(w, h, v.reshape(h, w))


# --------------------------------------------------------------------------
# Cache-size sweep (SweepReport SPEC.md:441-444; Fig.
# "cacheSize" of the paper): baseline without cache, then every (Nc, Ne).
# --------------------------------------------------------------------------

@dataclass
class SweepRow:
    """One SweepReport row; relative_time_pct = 100 * time / no-cache time."""
    n_cells: int
    n_entries: int
    wall_time_s: float
    relative_time_pct: float
    hit_rate: float
    inserts_lost_full: int
    memory_bytes: int


def sweep(scene: "Scene", config: RenderConfig, cells_list: Sequence[int],
          entries_list: Sequence[int], repeats: int = 1, ctx: Optional[Context] = None,
          device_time: bool = True) -> list:
    """cmd_sweep: render once without the cache (the 100% baseline), then
    every (n_cells, n_entries) combination with a fresh table, `repeats`
    times each (median). Times are the device's (CUDA events around the
    render on the context's stream; device_time=False: the call's wall
    time). Rows sorted by (n_cells, n_entries)."""
    import dataclasses
    import statistics
    if not cells_list or not entries_list:
        raise ValueError("sweep needs non-empty cells and entries lists")
    for v in list(cells_list) + list(entries_list):
        if int(v) <= 0:
            raise ValueError("cache sizes must be positive")
    ctx = ctx or Context.default()

    def timed(cfg):
        ts, last = [], None
        for _ in range(max(1, repeats)):
            last = render(scene, cfg, ctx=ctx)
            ts.append(last.stats.device_ms / 1e3 if device_time else last.stats.wall_time_s)
        return statistics.median(ts), last

    base_cfg = dataclasses.replace(config, cache_enabled=False)
    t0, _ = timed(base_cfg)
    rows = []
    for nc in sorted(int(c) for c in cells_list):
        for ne in sorted(int(e) for e in entries_list):
            cfg = dataclasses.replace(config, cache_enabled=True, n_cells=nc, n_entries=ne)
            t, res = timed(cfg)
            rows.append(SweepRow(nc, ne, t, 100.0 * t / t0 if t0 > 0 else 0.0, res.stats.hit_rate,
                                 res.stats.inserts_lost_full, memory_bytes(nc, ne)))
    return rows


def write_sweep_csv(rows: Sequence[SweepRow], path: str) -> None:
    """SweepReport as CSV, one row per (n_cells, n_entries), fixed column order."""
    cols = ["n_cells", "n_entries", "wall_time_s", "relative_time_pct", "hit_rate",
            "inserts_lost_full", "memory_bytes"]
    with open(path, "w") as f:
        f.write(",".join(cols) + "\n")
        for r in sorted(rows, key=lambda r: (r.n_cells, r.n_entries)):
            f.write(f"{r.n_cells},{r.n_entries},{r.wall_time_s:.9g},{r.relative_time_pct:.6g},"
                    f"{r.hit_rate:.9g},{r.inserts_lost_full},{r.memory_bytes}\n")


from . import artifacts  # noqa: E402  (image I/O, heatmap, diff)
