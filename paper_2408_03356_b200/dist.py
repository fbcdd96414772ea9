"""Multi-GPU plumbing: one process per GPU, torch.distributed
for the process group.  Rays are independent, the scene and its BVH
are replicated; the only exchange on the path is the data-parallel sum of the
per-Gaussian gradients of a training step (NCCL all-reduce over NVLink).

  * view / tile sharding: which views (or interleaved 16x16 tiles) a rank owns;
  * GradBuffer: the eight gradient groups as views of ONE flat fp32 buffer so
    that a step issues a single all_reduce (129.6 MB at C2, 864 MB at C3).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

GROUPS = ("mean", "quat", "scale", "density", "sh", "sg_amp", "sg_sharp", "sg_axis")


def env_world():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str | None = None):
    """Initialise the default process group from the torchrun environment."""
    rank, world, local = env_world()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world, local


def shard_views(n_views: int, rank: int, world: int):
    """Views owned by `rank` (round robin; equal counts when world | n_views)."""
    return list(range(rank, n_views, world))


def shard_tiles(width: int, height: int, rank: int, world: int, tile: int = 16):
    """Interleaved tile sharding (load balance across ranks): list of pixel
    rectangles (x0, y0, x1, y1) owned by `rank`, covering the image exactly
    once over all ranks."""
    rects = []
    k = 0
    for ty in range(0, height, tile):
        for tx in range(0, width, tile):
            if k % world == rank:
                rects.append((tx, ty, min(tx + tile, width), min(ty + tile, height)))
            k += 1
    return rects


class GradBuffer:
    """Gradient groups as views of one contiguous buffer (caller layouts of rg.h)."""

    def __init__(self, shapes: dict, device, dtype=torch.float32):
        sizes = {k: int(torch.Size(shapes[k]).numel()) for k in GROUPS}
        self.flat = torch.zeros(sum(sizes.values()), dtype=dtype, device=device)
        self.views = {}
        off = 0
        for k in GROUPS:
            self.views[k] = self.flat[off:off + sizes[k]].view(shapes[k])
            off += sizes[k]

    @classmethod
    def like(cls, scene):
        return cls({k: tuple(getattr(scene, k).shape) for k in GROUPS}, scene.mean.device)

    def zero_(self):
        self.flat.zero_()
        return self

    def all_reduce(self, group=None):
        """Sum over ranks in place (one collective).  No-op for world size 1."""
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)
        return self

    @property
    def nbytes(self):
        return self.flat.numel() * self.flat.element_size()
