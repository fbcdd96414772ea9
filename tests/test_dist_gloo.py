"""Multi-process (world size 2, gloo, CPU) tests of the data-parallel plumbing
(SURVEY.md §8(e)): rays/tiles sharded across ranks over a replicated scene,
per-Gaussian gradients summed with ONE all_reduce of a flat buffer.  The
per-rank gradients come from the oracle on each rank's shard; the all-reduced
result must equal the oracle's full-batch gradient, and the sharded images
must tile the full image exactly once."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_03356_b200 import dist as rgd
from paper_2408_03356_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        from oracle import oracle as O
        r, w, _ = rgd.init("gloo")
        assert (r, w) == (rank, world)
        sc = synth.random_scene(77, 30, sh_degree=1, sg_count=2, density_range=(5, 30),
                                scale_range=(0.05, 0.15), extent=0.3)
        p = synth.RenderParams(dt=5e-3, t_eps=1e-4)
        cam = synth.orbit_camera(1.6, 20, 20, 20, 12, 20.0)
        o_all, d_all = O.camera_rays(cam)
        rng = np.random.default_rng(5)
        up_all = rng.normal(size=(len(o_all), 3))
        # interleaved 16x16 tiles -> pixel indices of this rank
        idx = []
        for (x0, y0, x1, y1) in rgd.shard_tiles(cam.width, cam.height, rank, world, tile=8):
            for y in range(y0, y1):
                idx.extend(range(y * cam.width + x0, y * cam.width + x1))
        idx = np.array(idx, int)
        g = O.backward(sc, p, o_all[idx], d_all[idx], up_all[idx], mode=2)
        shapes = {k: tuple(v.shape) for k, v in g.items()}
        gb = rgd.GradBuffer(shapes, device="cpu", dtype=torch.float64)
        for k in rgd.GROUPS:
            gb.views[k].copy_(torch.from_numpy(g[k]))
        gb.all_reduce()
        full = O.backward(sc, p, o_all, d_all, up_all, mode=2)
        err = max(float(np.abs(gb.views[k].numpy() - full[k]).max() /
                        max(np.abs(full[k]).max(), 1e-300)) for k in rgd.GROUPS)
        # every pixel covered exactly once across ranks
        cnt = torch.zeros(cam.width * cam.height, dtype=torch.int64)
        cnt[torch.from_numpy(idx)] += 1
        dist.all_reduce(cnt)
        q.put((rank, err, int(cnt.min()), int(cnt.max())))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), -1, -1))


def test_gloo_world2_sharded_gradient_allreduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=180) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for rank, err, cmin, cmax in res:
        assert not isinstance(err, str), err
        assert err < 1e-12, (rank, err)
        assert cmin == 1 and cmax == 1


def test_shard_helpers():
    for world in (1, 2, 3, 8):
        seen = np.zeros((37, 53), int)
        for r in range(world):
            for (x0, y0, x1, y1) in rgd.shard_tiles(53, 37, r, world):
                seen[y0:y1, x0:x1] += 1
        assert np.all(seen == 1)
        views = [rgd.shard_views(8, r, world) for r in range(world)]
        assert sorted(v for vs in views for v in vs) == list(range(8))
    gb = rgd.GradBuffer({k: (5, 3) for k in rgd.GROUPS}, device="cpu")
    gb.views["sh"].fill_(2.0)
    assert gb.flat.sum() == 30.0 and gb.nbytes == 8 * 15 * 4
    gb.all_reduce()   # world size 1: no-op
    assert gb.flat.sum() == 30.0


# ---------------------------------------------------------------------------
# reduce-scatter -> sharded Adam -> all-gather (dist.ShardedAdam), host logic with
# the oracle's Adam as the per-shard step
# ---------------------------------------------------------------------------

class _OracleLocal:
    def __init__(self, act):
        from oracle import train as T
        self.T, self.act = T, act
        self.raw = {k: act[k].numpy().astype(np.float64) for k in rgd.GROUPS}
        self.raw["scale"] = np.log(self.raw["scale"])
        self.raw["density"] = np.log(self.raw["density"])
        self.m = {k: np.zeros_like(v) for k, v in self.raw.items()}
        self.v = {k: np.zeros_like(v) for k, v in self.raw.items()}

    def step(self, grads, it):
        g = {k: grads[k].numpy().astype(np.float64) for k in rgd.GROUPS}
        self.raw, self.m, self.v, a = self.T.adam_step(self.raw, self.m, self.v, g, it)
        for k in rgd.GROUPS:
            self.act[k].copy_(torch.from_numpy(a[k]).float())


def _sharded_adam_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        from paper_2408_03356_b200 import rg
        rgd.init("gloo")
        sc = synth.random_scene(91, 31, sh_degree=2, sg_count=3)     # 31 rows: padding
        g = rg.Gaussians(*[torch.from_numpy(a.copy()) for a in sc.arrays()],
                         sh_degree=sc.sh_degree, sg_count=sc.sg_count)
        sa = rgd.ShardedAdam(g, _OracleLocal)
        assert sa.s == 16 and sa.full["mean"].shape[0] == 32
        for it in range(3):
            sa.zero_grad()
            rng = np.random.default_rng(1000 * it + rank)   # each rank its own gradient
            for k in rgd.GROUPS:
                sa.grad_views[k].copy_(torch.from_numpy(
                    rng.normal(size=tuple(sa.grad_views[k].shape)).astype(np.float32)))
            sa.step(it)
        q.put((rank, {k: getattr(sa.scene, k).numpy().copy() for k in rgd.GROUPS}))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_sharded_adam_equals_full_adam():
    from oracle import train as T
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_sharded_adam_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    # reference: the unsharded oracle step on the summed gradient, from the same fp32 start
    sc = synth.random_scene(91, 31, sh_degree=2, sg_count=3)
    raw = {k: np.asarray(a, np.float64) for k, a in zip(rgd.GROUPS, sc.arrays())}
    raw["scale"] = np.log(np.asarray(sc.scale, np.float32).astype(np.float64))
    raw["density"] = np.log(np.asarray(sc.density, np.float32).astype(np.float64))
    m = {k: np.zeros_like(v) for k, v in raw.items()}
    v = {k: np.zeros_like(x) for k, x in raw.items()}
    for it in range(3):
        gsum = {k: np.zeros_like(raw[k]) for k in rgd.GROUPS}
        for r in range(world):                      # the workers' draws: one generator per
            rng = np.random.default_rng(1000 * it + r)   # (iteration, rank), groups in order
            for k in rgd.GROUPS:
                gsum[k] += rng.normal(size=raw[k].shape).astype(np.float32).astype(np.float64)
        raw, m, v, act = T.adam_step(raw, m, v, gsum, it)
        # the sharded path rounds the activated values to fp32 each step and
        # re-derives nothing from them (raw stays fp64 in the oracle local), so
        # only the final fp32 rounding differs
    for r in range(world):
        for k in rgd.GROUPS:
            assert np.allclose(res[r][k], act[k], rtol=2e-6, atol=1e-7), (r, k)
    assert all(np.array_equal(res[0][k], res[1][k]) for k in rgd.GROUPS)   # replicas identical


def test_bench_relaunch_world2_tile_plumbing():
    """bench.py's `--gpus N` re-launch (torch.distributed.run, 127.0.0.1) at world
    size 2 on CPU/gloo, running the tile-sharding plumbing check: per-rank
    rg_camera tile cameras of the C1 and C3 views, rg_camera_ray_count (host) =
    the slot count, and the ranks' slots cover every pixel exactly once."""
    import bench
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    rc = bench.relaunch_distributed(2, script=os.path.join(root, "tools", "dist_tile_check.py"),
                                    argv=[])
    assert rc == 0
