"""The N>1 path on CPU: two processes over torch.distributed (gloo), each
rendering its tile shard (with the CPU oracle standing in for the device,
which this container lacks) and reducing the framebuffers to rank 0 with
paper_2305_07238_b200.dist.gather_frame -- exactly as bench.py does over NCCL.
The gathered frame must equal the single-process render bit for bit."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_07238_b200 import dist as D
from paper_2305_07238_b200 import load_scene, scenes


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


W, H, SPP = 45, 33, 2


def _worker(rank, world, port, scene_path, mode, cache, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import _oracle
    orc = _oracle.Oracle()
    s = load_scene(scene_path)
    P = _oracle.RenderParamsC(W, H, SPP, 4, 1 if cache else 0, 0, 211, 4, 0, 1, 0.2, 16, rank, world, mode, 0, 1)
    c = orc.cache_new(211, 4) if cache else None   # per-rank table replica
    rad, nodes, samples, hps, st = orc.render(s.flat, P, cache=c)
    mask = D.shard_mask(W, H, 16, rank, world, mode)
    assert (samples[~mask] == 0).all() and (samples[mask] == SPP).all()
    tr = torch.from_numpy(rad.copy())
    tn = torch.from_numpy(nodes.copy())
    ts = torch.from_numpy(samples.astype(np.int64))
    D.gather_frame([tr, tn, ts])
    if rank == 0:
        np.save(os.path.join(out_dir, "rad.npy"), tr.numpy())
        np.save(os.path.join(out_dir, "nodes.npy"), tn.numpy())
        np.save(os.path.join(out_dir, "samples.npy"), ts.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [D.SHARD_INTERLEAVED, D.SHARD_BANDS])
@pytest.mark.parametrize("cache", [False, True])
def test_two_rank_gather_is_exact(built, scene_dir, mode, cache):
    path = scenes.build_scene(scenes.SceneSpec("cornell", W, H, tris_per_side=3), f"{scene_dir}/mp")
    out = tempfile.mkdtemp()
    mp.start_processes(_worker, args=(2, _free_port(), path, mode, cache, out), nprocs=2,
                       join=True, start_method="spawn")
    import _oracle
    orc = _oracle.Oracle()
    s = load_scene(path)
    rad = np.load(os.path.join(out, "rad.npy"))
    samples = np.load(os.path.join(out, "samples.npy"))
    assert (samples == SPP).all()
    if not cache:
        full = orc.render(s.flat, _oracle.RenderParamsC(W, H, SPP, 4, 0, 0, 211, 4, 0, 1, 0.2, 16, 0, 1, 0, 0, 1))
        np.testing.assert_array_equal(rad.view(np.uint64), full[0].view(np.uint64))
    else:
        # per-shard replicas: each rank's pixels equal that rank's own cached render
        for r in range(2):
            c = orc.cache_new(211, 4)
            part = orc.render(s.flat, _oracle.RenderParamsC(W, H, SPP, 4, 1, 0, 211, 4, 0, 1, 0.2, 16, r, 2, mode, 0, 1), cache=c)
            m = D.shard_mask(W, H, 16, r, 2, mode)
            np.testing.assert_array_equal(rad[m].view(np.uint64), part[0][m].view(np.uint64))
            orc.cache_free(c)


def test_shard_masks_partition_the_image():
    for mode in (D.SHARD_INTERLEAVED, D.SHARD_BANDS):
        for world in (1, 2, 3, 4, 8):
            cover = sum(D.shard_mask(1920, 1080, 16, r, world, mode).astype(int) for r in range(world))
            assert (cover == 1).all()


def _handle_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = bytes([rank]) * 64          # stands for this rank's 64-byte CUDA IPC handle
    got = D.exchange_handles(mine, world)
    with open(os.path.join(out_dir, f"h{rank}.bin"), "wb") as f:
        f.write(b"".join(got))
    dist.barrier()
    dist.destroy_process_group()


def test_shared_cache_handle_exchange(built):
    """The shared (striped) table's set-up step on CPU: every rank ends with
    every rank's stripe handle, in rank order (dist.shared_cache then maps
    them with mcg_cache_attach_ipc)."""
    out = tempfile.mkdtemp()
    world = 3
    mp.start_processes(_handle_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    want = b"".join(bytes([r]) * 64 for r in range(world))
    for r in range(world):
        with open(os.path.join(out, f"h{r}.bin"), "rb") as f:
            assert f.read() == want
