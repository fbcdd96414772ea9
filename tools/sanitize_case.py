"""Small forward + backward cases for compute-sanitizer (dev tool, SURVEY §4 layer 5):
C0 (tiny, camera mode, fetch log), a 10k-Gaussian random scene (explicit rays,
SH 3 + 7 SG, with and without a fetch log), an overflow case (K = 40 < slab
sets: the restart-query streaming path), the tile-sharded camera, and the
NEXT-1 kernels (refit, Adam, L1 + D-SSIM).

usage: compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_case.py
"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_03356_b200 import rg, synth  # noqa: E402


def fwd_bwd(sc, p, *, rays=None, camera=None, log=True):
    g = rg.Gaussians.from_scene(sc)
    cfg = rg.Config.of(p)
    b = rg.build_bvh(g, cfg, check=True)
    n = camera.n_rays if camera is not None else rays[0].shape[0]
    st = rg.new_stats()
    f = rg.render_forward(g, b, cfg, rays=rays, camera=camera, stats=st,
                          log=rg.new_log(n) if log else None, debug=(min(n, 16), 256))
    up = torch.full((n, 3), 1.0 / (3 * n), device="cuda")
    rg.render_backward(g, b, cfg, f, up, rays=rays, camera=camera, stats=st)
    rg.refit_bvh(b, g, cfg)
    torch.cuda.synchronize()
    return g, b, f


def main():
    wl = synth.workload("tiny")
    fwd_bwd(wl.scene, wl.params, camera=wl.cameras[0])
    cam_t = dataclasses.replace(wl.cameras[0], tile=16, shard=1, shards=3)
    fwd_bwd(wl.scene, wl.params, camera=cam_t)
    sc = synth.random_scene(77, 10_000, sh_degree=3, sg_count=7, density_range=(2, 30),
                            scale_range=(0.01, 0.04), extent=0.6)
    p = synth.RenderParams(dt=2e-3, t_eps=1e-4)
    o, d = synth.random_rays(78, 2048)
    rays = (torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda())
    fwd_bwd(sc, p, rays=rays, log=True)
    g, b, f = fwd_bwd(sc, p, rays=rays, log=False)
    sc2 = synth.random_scene(950, 400, sh_degree=1, sg_count=1, density_range=(0.3, 2.0),
                             scale_range=(0.1, 0.3), extent=0.3)
    p2 = synth.RenderParams(dt=4e-3, slab_samples=8, t_eps=1e-4, hit_capacity=40)
    o2, d2 = synth.random_rays(951, 256, radius=2.0, jitter=0.2)
    fwd_bwd(sc2, p2, rays=(torch.from_numpy(o2).cuda(), torch.from_numpy(d2).cuda()))
    # NEXT-1 kernels
    opt = rg.Adam(g)
    grads = g.zeros_like_grads()
    for k in grads:
        grads[k].normal_()
    opt.step(grads, it=0)
    img = torch.rand(37 * 45, 3, device="cuda")
    rg.l1_dssim_loss_grad(img, torch.rand_like(img), 45, 37)
    torch.cuda.synchronize()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
