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


class ShardedAdam:
    """Reduce-scatter -> sharded Adam -> all-gather: each
    rank owns the Gaussian rows [rank*s, (rank+1)*s) of every parameter group
    (s = ceil(n / world)); the summed gradient of its rows arrives by one
    reduce-scatter per group, its Adam state is 1/world of the full one, and the
    updated activated parameters are all-gathered back into the replicated scene
    the renderer reads.  Group arrays keep the rg.h caller layouts (row slices of
    padded [n_pad, ...] storage), so the same kernels run on a shard.

    `make_local(act_shard: dict) -> obj with .step(grads: dict, it)` builds the
    per-shard optimiser that updates `act_shard` in place (rg.Adam on the GPU)."""

    PAD_ROW = dict(quat=(1.0, 0.0, 0.0, 0.0))

    def __init__(self, scene, make_local, group=None):
        from . import rg
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        n = scene.n
        self.n = n
        self.s = -(-n // self.world) if n > 0 else 0
        n_pad = self.s * self.world
        self.full, self.grad = {}, {}
        for k in GROUPS:
            t = getattr(scene, k)
            buf = torch.zeros((n_pad,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            buf[:n] = t
            if n_pad > n:          # valid dummy rows: zero gradient keeps them fixed
                if k == "quat":
                    buf[n:, 0] = 1.0
                elif k == "sg_axis":
                    buf[n:, ..., 2] = 1.0
                elif k in ("scale", "density"):
                    buf[n:] = 1.0
            self.full[k] = buf
            self.grad[k] = torch.zeros_like(buf)
        self.scene = rg.Gaussians(*[self.full[k][:n] for k in GROUPS], sh_degree=scene.sh_degree,
                                  sg_count=scene.sg_count)
        self.grad_views = {k: self.grad[k][:n] for k in GROUPS}
        lo, hi = self.rank * self.s, (self.rank + 1) * self.s
        self.act_shard = {k: self.full[k][lo:hi].clone() for k in GROUPS}
        self.grad_shard = {k: torch.zeros_like(self.act_shard[k]) for k in GROUPS}
        self.local = make_local(self.act_shard)

    def zero_grad(self):
        for k in GROUPS:
            self.grad[k].zero_()

    def step(self, it=None):
        multi = dist.is_initialized() and self.world > 1
        for k in GROUPS:
            if self.grad[k].numel() == 0:
                continue
            if multi:
                dist.reduce_scatter_tensor(self.grad_shard[k].view(-1), self.grad[k].view(-1),
                                           op=dist.ReduceOp.SUM, group=self.group)
            else:
                self.grad_shard[k].copy_(self.grad[k])
        self.local.step(self.grad_shard, it)
        for k in GROUPS:
            if self.full[k].numel() == 0:
                continue
            if multi:
                dist.all_gather_into_tensor(self.full[k].view(-1), self.act_shard[k].view(-1),
                                            group=self.group)
            else:
                self.full[k].copy_(self.act_shard[k])

    @staticmethod
    def gpu_local(sh_degree, sg_count, **adam_kw):
        """factory of the production per-shard optimiser (fused rg_adam_step)"""
        from . import rg

        class _Local:
            def __init__(self, act):
                self.scene = rg.Gaussians(*[act[k] for k in GROUPS], sh_degree=sh_degree,
                                          sg_count=sg_count)
                self.opt = rg.Adam(self.scene, **adam_kw)

            def step(self, grads, it):
                self.opt.step(grads, it=it)
        return _Local
