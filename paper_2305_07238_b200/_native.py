"""ctypes binding of libmcg.so (include/mcg.h). Loads the in-tree build and
fails loudly when it is missing: there is no CPU fallback for any call that
reaches the device."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MCG_LIB_PATH: an alternative in-tree build (kernel A/B experiments,
# profiles/scripts/build_variant.sh); default the normal build.
LIB_PATH = os.environ.get("MCG_LIB_PATH") or os.path.join(HERE, "_lib", "libmcg.so")

u8, u32, u64, i32, i64, f32, f64 = C.c_uint8, C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_float, C.c_double
P = C.POINTER
vp = C.c_void_p


class Descriptor(C.Structure):
    _fields_ = [("mat_idx", u32), ("node_idx", u32), ("mip_level", u8), ("pad_", u8 * 3),
                ("texel_x", u32), ("texel_y", u32)]


class Options(C.Structure):
    _fields_ = [("device", i32), ("profile", i32), ("stream", vp), ("n_devices", i32), ("devices", P(i32))]


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", u64), ("ms", f64), ("algorithmic_bytes", f64)]


class CacheCounters(C.Structure):
    _fields_ = [("lookups", u64), ("hits", u64), ("inserts_won", u64), ("inserts_lost_full", u64)]


class AuditReport(C.Structure):
    _fields_ = [("n_cells", u64), ("n_entries", u64), ("occupied", u64), ("clean", i32),
                ("bad_cell", i64), ("problem", C.c_char * 160)]


class Insn(C.Structure):
    _fields_ = [("op", u8), ("flags", u8), ("sp", u8), ("tags", u8), ("arg", u32),
                ("bracket", C.c_uint16), ("store_ord", u8), ("pad_", u8), ("imm", u32)]


class Program(C.Structure):
    _fields_ = [("material_id", u32), ("code_offset", u32), ("code_len", u32), ("max_stack", u32),
                ("cache_point_count", u32)]


class FlatScene(C.Structure):
    _fields_ = [
        ("cam_position", f32 * 3), ("cam_look_at", f32 * 3), ("cam_up", f32 * 3),
        ("cam_vfov_deg", f32), ("cam_width", i32), ("cam_height", i32), ("env", f32 * 3),
        ("n_prims", u32), ("prim_geom", P(f32)), ("prim_uv", P(f32)), ("prim_info", P(u32)),
        ("n_nodes", u32), ("nodes", vp),
        ("n_point_lights", u32), ("n_rect_lights", u32), ("point_lights", vp), ("rect_lights", vp),
        ("n_programs", u32), ("programs", P(Program)),
        ("n_code", u32), ("code", P(Insn)),
        ("n_consts", u32), ("consts", vp),
        ("n_noise", u32), ("noise", vp),
        ("n_ramps", u32), ("ramps", vp),
        ("n_ramp_stops", u32), ("ramp_stops", vp),
        ("n_textures", u32), ("textures", vp),
        ("n_texels", u64), ("texels", P(f32)),
    ]


class RenderParams(C.Structure):
    _fields_ = [("width", i32), ("height", i32), ("spp", i32), ("max_bounces", i32),
                ("cache_mode", i32), ("mip_offset", i32), ("n_cells", u64), ("n_entries", u32),
                ("first_sample", u32), ("rng_seed", u64), ("diffuse_spread", f32),
                ("tile_size", i32), ("shard_rank", i32), ("shard_count", i32), ("shard_mode", i32),
                ("samples_per_pass", i32)]


class Frame(C.Structure):
    _fields_ = [("radiance", P(f64)), ("nodes_found", P(f64)), ("samples", P(u32))]


class RenderStats(C.Structure):
    _fields_ = [("wall_time_s", f64), ("device_ms", f64), ("lookups", u64), ("hits", u64),
                ("inserts_won", u64), ("inserts_lost_full", u64), ("stores_attempted", u64),
                ("stores_won", u64), ("instructions_executed", u64), ("max_stack_seen", u64),
                ("paths", u64), ("shading_points", u64), ("shadow_rays", u64),
                ("bvh_nodes", u64), ("prims_tested", u64), ("tex_samples", u64),
                ("bvh_nodes_shadow", u64), ("prims_tested_shadow", u64), ("closest_rays", u64),
                ("shadow_occluded", u64), ("launches", u64), ("hits_per_sample", P(u64))]


# (name, restype, argtypes)
_SIGS = [
    ("mcg_last_error", C.c_char_p, []),
    ("mcg_abi_version", C.c_int, []),
    ("mcg_hash_cell", u64, [P(Descriptor)]),
    ("mcg_hash_check", u32, [P(Descriptor)]),
    ("mcg_encode_value", u32, [P(f32)]),
    ("mcg_decode_value", None, [u32, P(f32)]),
    ("mcg_memory_bytes", C.c_int, [u64, u64, P(u64)]),
    ("mcg_create", C.c_int, [P(Options), P(vp)]),
    ("mcg_device_count", C.c_int, [P(i32)]),
    ("mcg_destroy", C.c_int, [vp]),
    ("mcg_synchronize", C.c_int, [vp]),
    ("mcg_stream", vp, [vp]),
    ("mcg_kernel_times", C.c_int, [vp, P(KernelTime), i32, P(i32)]),
    ("mcg_kernel_times_reset", C.c_int, [vp]),
    ("mcg_launch_count", u64, [vp]),
    ("mcg_hash_batch", C.c_int, [vp, vp, C.c_size_t, vp, vp]),
    ("mcg_encode_batch", C.c_int, [vp, vp, C.c_size_t, vp]),
    ("mcg_decode_batch", C.c_int, [vp, vp, C.c_size_t, vp]),
    ("mcg_mip_texel_batch", C.c_int, [vp, vp, vp, vp, C.c_size_t, i32, vp, vp]),
    ("mcg_cache_create", C.c_int, [vp, u64, u32, P(vp)]),
    ("mcg_cache_destroy", C.c_int, [vp]),
    ("mcg_cache_clear", C.c_int, [vp]),
    ("mcg_cache_shape", C.c_int, [vp, P(u64), P(u32)]),
    ("mcg_cache_update_batch", C.c_int, [vp, vp, vp, C.c_size_t, i32, vp, vp, vp]),
    ("mcg_cache_lookup_batch", C.c_int, [vp, vp, C.c_size_t, vp, vp]),
    ("mcg_cache_update_device", C.c_int, [vp, vp, vp, C.c_size_t, i32, vp]),
    ("mcg_cache_lookup_device", C.c_int, [vp, vp, C.c_size_t, vp, vp]),
    ("mcg_cache_read_slots", C.c_int, [vp, u64, C.c_size_t, vp]),
    ("mcg_cache_write_slots", C.c_int, [vp, u64, C.c_size_t, vp]),
    ("mcg_cache_occupied", C.c_int, [vp, P(u64)]),
    ("mcg_cache_counters_get", C.c_int, [vp, P(CacheCounters)]),
    ("mcg_cache_counters_reset", C.c_int, [vp]),
    ("mcg_cache_dump", C.c_int, [vp, C.c_char_p]),
    ("mcg_cache_device_slots", vp, [vp]),
    ("mcg_cache_create_stripe", C.c_int, [vp, u64, u32, u32, u32, P(vp)]),
    ("mcg_cache_attach_local", C.c_int, [vp, P(vp), u32]),
    ("mcg_cache_ipc_handle", C.c_int, [vp, vp, C.c_size_t]),
    ("mcg_cache_attach_ipc", C.c_int, [vp, vp, u32]),
    ("mcg_cache_stripe_info", C.c_int, [vp, P(u32), P(u32), P(u64)]),
    ("mcg_audit_dump", C.c_int, [C.c_char_p, P(AuditReport)]),
    ("mcg_probe_bench", C.c_int, [vp, u64, u64, i32, i32, P(f64), P(f64)]),
    ("mcg_cache_trace_start", C.c_int, [vp, u64]),
    ("mcg_cache_trace_stop", C.c_int, [vp, P(u64)]),
    ("mcg_cache_trace_read", C.c_int, [vp, u64, C.c_size_t, vp]),
    ("mcg_cache_insert_log_start", C.c_int, [vp, u64]),
    ("mcg_cache_insert_log_stop", C.c_int, [vp, C.POINTER(u64)]),
    ("mcg_cache_insert_log_read", C.c_int, [vp, u64, C.c_size_t, vp]),
    ("mcg_probe_replay", C.c_int, [vp, vp, u64, i32, P(f64), P(f64), P(CacheCounters)]),
    ("mcg_scene_load", C.c_int, [C.c_char_p, i32, P(vp)]),
    ("mcg_scene_destroy", C.c_int, [vp]),
    ("mcg_scene_flat", C.c_int, [vp, P(FlatScene)]),
    ("mcg_scene_disassemble", C.c_int, [vp, u32, C.c_char_p, C.c_size_t, P(C.c_size_t)]),
    ("mcg_scene_analysis_json", C.c_int, [vp, u32, C.c_char_p, C.c_size_t, P(C.c_size_t)]),
    ("mcg_scene_build", C.c_int, [vp, P(vp)]),
    ("mcg_schedule_program", C.c_int, [vp, u32, vp, u32, P(u32)]),
    ("mcg_upload_scene", C.c_int, [vp, vp]),
    ("mcg_render", C.c_int, [vp, P(RenderParams), vp, P(Frame), P(RenderStats)]),
    ("mcg_render_device", C.c_int, [vp, P(RenderParams), vp, P(Frame), P(RenderStats)]),
    ("mcg_camera_setup", C.c_int, [P(FlatScene), i32, i32, P(f32)]),
    ("mcg_execute_batch", C.c_int, [vp, u32, vp, C.c_size_t, vp, i32, i32, vp, vp, vp]),
    ("mcg_intersect_batch", C.c_int, [vp, vp, C.c_size_t, f32, f32, i32, vp]),
    ("mcg_occluded_batch", C.c_int, [vp, vp, C.c_size_t, f32, vp, i32, vp]),
    ("mcg_shadow_tree", C.c_int, [vp, vp, C.c_size_t, P(C.c_size_t), P(i32), P(i32)]),
]

EXPORTED = [s[0] for s in _SIGS]

_lib = None


ABI_VERSION = 4   # include/mcg.h MCG_ABI_VERSION (the struct layouts below)


def lib():
    """The loaded libmcg (raises ImportError when the build is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libmcg.so not built at {LIB_PATH}; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.mcg_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH}: ABI version {L.mcg_abi_version()}, this binding expects "
                              f"{ABI_VERSION}; rebuild with __graft_entry__.build()")
        _lib = L
    return _lib


class MCGError(RuntimeError):
    """Base class of errors raised through the C ABI."""


class GraphError(MCGError):
    """matcache::GraphError (graph.hpp:89-96)."""


class CompileError(MCGError):
    """matcache::CompileError (stackvm.hpp:65-68)."""


class SceneError(MCGError):
    """matcache::SceneError (scene.hpp:66-69)."""


class ImageIoError(MCGError):
    """matcache::ImageIoError (image.hpp:24-27)."""


class CudaError(MCGError):
    """A CUDA runtime failure (no reference analogue)."""


class NoDeviceError(CudaError):
    """No CUDA device is visible."""


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib().mcg_last_error().decode(errors="replace")
    exc = {1: ValueError, 2: OverflowError, 3: GraphError, 4: CompileError, 5: SceneError,
           6: ImageIoError, 7: OSError, 8: CudaError, 9: NoDeviceError}.get(status, MCGError)
    raise exc(msg)
