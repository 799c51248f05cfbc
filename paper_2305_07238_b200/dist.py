"""Multi-GPU tile sharding: one process per GPU, each rendering
its 16x16 tiles (tracer.hpp:19) with a private table replica, and one
reduce(sum) per framebuffer to rank 0 over torch.distributed (NCCL over
NVLink on GPUs, gloo in the CPU tests). The reduce is exact: every pixel is
non-zero on exactly one rank and x + 0 = x.

`shared_cache` builds the alternative of SURVEY §8f.3: one logical table
striped by cell over the ranks (each rank's stripe mapped into every other
rank through CUDA IPC, inserts are CASes on peer memory over NVLink), so all
ranks share what any of them cached.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import replace
from typing import Optional

import numpy as np

from . import _native as N
from . import Context, RenderConfig, RenderStats, Scene

SHARD_INTERLEAVED, SHARD_BANDS = 0, 1


def tile_owner(tile: int, n_tiles: int, world: int, mode: int) -> int:
    """Rank that renders tile `tile` (mirrors csrc/mcg_render.cu tile_mine)."""
    if world <= 1:
        return 0
    if mode == SHARD_INTERLEAVED:
        return tile % world
    for r in range(world):
        lo = n_tiles * r // world
        hi = n_tiles * (r + 1) // world
        if lo <= tile < hi:
            return r
    raise ValueError("tile out of range")


def shard_mask(width: int, height: int, tile: int, rank: int, world: int, mode: int) -> np.ndarray:
    """Boolean (height, width) mask of the pixels rank `rank` renders."""
    tx = (width + tile - 1) // tile
    ty = (height + tile - 1) // tile
    owners = np.array([tile_owner(t, tx * ty, world, mode) for t in range(tx * ty)]).reshape(ty, tx)
    return np.repeat(np.repeat(owners, tile, 0), tile, 1)[:height, :width] == rank


def shard_config(config: RenderConfig, rank: int, world: int, mode: int = SHARD_INTERLEAVED) -> RenderConfig:
    return replace(config, shard_rank=rank, shard_count=world, shard_mode=mode)


def gather_frame(tensors, dst: int = 0, group=None) -> None:
    """reduce(sum) of each framebuffer tensor to `dst` (in place)."""
    import torch.distributed as dist
    for t in tensors:
        dist.reduce(t, dst, group=group)


def exchange_handles(handle: bytes, world: int, group=None) -> list:
    """all_gather of the ranks' 64-byte stripe handles (rank order)."""
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, bytes(handle), group=group)
    return out


def shared_cache(n_cells: int, n_entries: int, ctx: Context, rank: int, world: int, group=None):
    """This rank's stripe of a table shared by all ranks, every stripe
    attached (collective: every rank calls it)."""
    from . import MaterialCache
    import torch.distributed as dist
    st = MaterialCache.stripe(n_cells, n_entries, rank, world, ctx)
    st.attach_ipc(exchange_handles(st.ipc_handle(), world, group))
    dist.barrier(group=group)   # every stripe zeroed and mapped before anyone inserts
    return st


def render_sharded(scene: Scene, config: RenderConfig, ctx: Context, rank: int, world: int,
                   mode: int = SHARD_INTERLEAVED, gather: bool = True, cache=None):
    """Renders this rank's tiles into device framebuffers (torch tensors on
    the context's device) and reduces them to rank 0; `cache` (e.g. a
    shared_cache stripe) replaces the rank's private table. Returns
    (radiance, nodes_found, samples, stats) tensors (valid on rank 0)."""
    import torch
    if ctx._scene is not scene:
        ctx.upload(scene)
    w = config.width or scene.flat.cam_width
    h = config.height or scene.flat.cam_height
    dev = torch.device("cuda", ctx.device)
    rad = torch.zeros(h * w * 3, dtype=torch.float64, device=dev)
    nodes = torch.zeros(h * w, dtype=torch.float64, device=dev)
    samples = torch.zeros(h * w, dtype=torch.int32, device=dev)
    frame = N.Frame(C.cast(C.c_void_p(rad.data_ptr()), C.POINTER(C.c_double)),
                    C.cast(C.c_void_p(nodes.data_ptr()), C.POINTER(C.c_double)),
                    C.cast(C.c_void_p(samples.data_ptr()), C.POINTER(C.c_uint32)))
    params = shard_config(config, rank, world, mode).to_params()
    st = N.RenderStats()
    torch.cuda.current_stream(dev).synchronize()
    N.check(N.lib().mcg_render_device(ctx.handle, C.byref(params), cache.handle if cache is not None else None,
                                      C.byref(frame), C.byref(st)))
    ctx.synchronize()
    if gather and world > 1:
        gather_frame([rad, nodes, samples])
    stats = RenderStats(st.wall_time_s, st.lookups, st.hits,
                        (st.hits / st.lookups) if st.lookups else 0.0, st.inserts_won,
                        st.inserts_lost_full, st.stores_attempted, st.instructions_executed, [],
                        st.shading_points, st.shadow_rays, st.paths)
    return rad.view(h, w, 3), nodes.view(h, w), samples.view(h, w), stats
