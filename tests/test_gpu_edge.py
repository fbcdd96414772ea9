"""GPU parity on the configurations and edge cases round 1 left untested
(VERDICT r1 "what's weak" #3), through the C-ABI against the oracle:

  * radius_mode = 1 (the north star's "3-sigma ellipsoid AABBs", DESIGN L3);
  * t_near > 0 (L13: t0 = max(box entry, t_near));
  * ray origins inside supports (negative t_entry: the sign-flip order key, L8);
  * non-finite Gaussians inside a render (inactive, counted, zero gradient);
  * bit-exact builds at the full C3 (2M) and C4 (5M) sizes;
  * a grid scene whose balanced tree exceeds the old n/2 + 2 wide-node bound;
  * per-slab hit sets of 256 hitting rays of the full-size C1 view.
Bars as tests/test_gpu_parity.py: bit-exact sets / build arrays, pixels
<= 1e-4, gradients per group and elementwise <= 1e-3.
"""
import numpy as np
import pytest
import torch

from paper_2408_03356_b200 import rg, synth
from test_gpu_parity import compare_pixels, gpu_build, gpu_forward, grad_check

pytestmark = pytest.mark.gpu


def fwd_bwd_case(oracle, sc, p, o, d, *, debug_rays=256, cap=20000, up_seed=0, log=True):
    """forward (hit-set dump) + backward through explicit rays, vs the oracle"""
    g, b = gpu_build(sc, p)
    r = gpu_forward(g, b, p, o, d, debug=(min(debug_rays, len(o)), cap))
    ref = oracle.render(sc, p, o, d, mode=2, dump_cap=cap)
    ok = compare_pixels(oracle, sc, p, o, d, r, ref)
    for k in range(min(debug_rays, len(o))):
        if ok[k]:
            n = r["debug_counts"][k]
            assert np.array_equal(r["debug_records"][k, :n], ref["dump"][k][:cap]), k
    cfg = rg.Config.of(p)
    to, td = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
    fwd = rg.render_forward(g, b, cfg, rays=(to, td), log=rg.new_log(len(o)) if log else None)
    up = np.random.default_rng(up_seed).normal(size=(len(o), 3)).astype(np.float32)
    st = rg.new_stats()
    grads = rg.render_backward(g, b, cfg, fwd, torch.from_numpy(up).cuda(), rays=(to, td), stats=st)
    torch.cuda.synchronize()
    gref = oracle.backward(sc, p, o, d, up.astype(np.float64), mode=2)
    grad_check(grads, gref)
    return r, ref, grads, gref


@pytest.mark.parametrize("log", [True, False])
def test_ksigma_supports(oracle, log):
    """radius_mode 1, k = 3: every active Gaussian's support is its 3-sigma
    ellipsoid (north star), independent of sigma~."""
    sc = synth.random_scene(2001, 120, sh_degree=3, sg_count=7, density_range=(2, 30),
                            scale_range=(0.03, 0.1), extent=0.45)
    p = synth.RenderParams(dt=3e-3, t_eps=1e-4, radius_mode=1, k_sigma=3.0,
                           background=(0.2, 0.3, 0.4))
    o, d = oracle.camera_rays(synth.orbit_camera(2.2, 70, 25, 28, 28, 32.0))
    r, ref, _, _ = fwd_bwd_case(oracle, sc, p, o, d, log=log)
    assert ref["counters"]["evals"] > 0
    # a different k gives a different (larger) support set: the mode is really used
    ref5 = oracle.render(sc, p.replace(k_sigma=5.0), o, d, mode=2)
    assert ref5["counters"]["evals"] > ref["counters"]["evals"]


def test_t_near_positive(oracle):
    """t0 = max(bbox entry, t_near) (L13): a near plane that cuts the scene."""
    sc = synth.random_scene(2002, 150, sh_degree=1, sg_count=2, density_range=(2, 30),
                            scale_range=(0.03, 0.12), extent=0.5)
    cam = synth.orbit_camera(2.2, 20, 15, 24, 24, 30.0)
    o, d = oracle.camera_rays(cam)
    p0 = synth.RenderParams(dt=3e-3, t_eps=1e-4, background=(1, 1, 1))
    p = p0.replace(t_near=2.1)     # the camera is 2.2 from the centre: cuts the front half
    r, ref, _, _ = fwd_bwd_case(oracle, sc, p, o, d)
    full = oracle.render(sc, p0, o, d, mode=2)
    assert np.abs(full["rgb"] - ref["rgb"]).max() > 1e-2     # the near plane matters


def test_origins_inside_supports(oracle):
    """Ray origins inside ellipsoids: negative t_entry (order key sign flip,
    L8), pairs active from the first slab."""
    sc = synth.random_scene(2003, 200, sh_degree=2, sg_count=3, density_range=(1, 12),
                            scale_range=(0.08, 0.3), extent=0.5)
    rng = np.random.default_rng(5)
    n = 400
    o = rng.uniform(-0.3, 0.3, size=(n, 3)).astype(np.float32)
    d = rng.normal(size=(n, 3))
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    p = synth.RenderParams(dt=3e-3, t_eps=1e-4, background=(0.1, 0.2, 0.3))
    r, ref, _, _ = fwd_bwd_case(oracle, sc, p, o, d)
    # the case is exercised: pairs whose support interval starts behind the origin
    neg = 0
    for l in range(sc.n):
        M, r2, _, fl = oracle.prim_setup(sc, p, l)
        if not fl & 2:
            continue
        for k in range(40):
            hit, te, tx = oracle.isect(M, r2, sc.mean[l], o[k], d[k])
            neg += hit and te < 0 < tx
    assert neg > 10


def test_nonfinite_gaussians_in_render(oracle):
    """Non-finite parameters make a Gaussian inactive (rg.h data errors):
    pixels and gradients of the rest match the oracle; the bad rows get zero
    gradient; no non-finite gradient is produced."""
    sc = synth.random_scene(2004, 160, sh_degree=2, sg_count=2, density_range=(2, 30),
                            scale_range=(0.03, 0.12), extent=0.45)
    sc.mean[3, 1] = np.nan
    sc.scale[7, 0] = np.inf
    sc.density[11] = np.nan
    sc.sh[13, 2, 1] = np.inf
    sc.sg_amp[17, 1, 0] = -np.inf
    sc.sg_axis[19, 0, 2] = np.nan
    sc.quat[23, 0] = np.nan
    bad = [3, 7, 11, 13, 17, 19, 23]
    p = synth.RenderParams(dt=3e-3, t_eps=1e-4)
    o, d = oracle.camera_rays(synth.orbit_camera(2.2, 50, 25, 24, 24, 30.0))
    r, ref, grads, gref = fwd_bwd_case(oracle, sc, p, o, d)
    for k, t in grads.items():
        a = t.cpu().numpy()
        assert np.isfinite(a).all(), k
        if a.size:
            assert np.all(a[bad] == 0), k


@pytest.mark.parametrize("dims", [(16, 16, 8), (64, 32, 32)])
def test_grid_scene_wide_capacity(oracle, dims):
    """Gaussians on a power-of-two grid give a balanced Karras tree whose greedy
    32-wide collapse has more than n/2 + 2 wide nodes: the build
    must stay within wide_capacity, flag nothing and render correctly."""
    nx, ny, nz = dims
    n = nx * ny * nz
    gx, gy, gz = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    mean = (np.stack([gx, gy, gz], -1).reshape(-1, 3) / max(dims) - 0.5).astype(np.float32)
    sc = synth.random_scene(2005, n, density_range=(1, 5), scale_range=(0.2 / max(dims), 0.4 / max(dims)))
    sc.mean[:] = mean
    sc.scale[:] = 0.3 / max(dims)          # identical isotropic Gaussians: equal-area ties
    sc.quat[:] = (1.0, 0.0, 0.0, 0.0)      # (a numpy model of the greedy collapse gives
    sc.density[:] = 3.0                    # 1057 > 1026 and 33825 > 32770 wide nodes)
    p = synth.RenderParams(dt=2e-3, t_eps=1e-4)
    g, b = gpu_build(sc, p)
    b.check()
    info = b.debug_views()["wide_info"].cpu().numpy()
    assert info[0] > n // 2 + 2                                  # the old bound is exceeded
    assert info[0] <= n // 2 + n // 62 + 4
    ref = oracle.BVH(sc, p)
    from test_gpu_parity import check_wide_tree
    check_wide_tree(b, ref, n)
    o, d = oracle.camera_rays(synth.orbit_camera(2.0, 30, 20, 16, 16, 20.0))
    rr = gpu_forward(g, b, p, o, d)
    refr = oracle.render(sc, p, o, d, mode=2, bvh=ref)
    compare_pixels(oracle, sc, p, o, d, rr, refr)


@pytest.mark.parametrize("name", ["mip", "stress"])
def test_build_bitexact_full_size(oracle, name):
    """Morton codes, sort order, Karras topology, refit boxes and the wide
    tree bit-exact at the full C3 (2M) and C4 (5M) sizes."""
    from test_gpu_parity import check_wide_tree
    wl = synth.workload(name)
    sc, p = wl.scene, wl.params
    g, b = gpu_build(sc, p)
    b.check()
    v = {k: t.cpu().numpy() for k, t in b.debug_views().items()}
    ref = oracle.BVH(sc, p)
    assert np.array_equal(v["codes"].view(np.uint32), ref.codes)
    assert np.array_equal(v["sorted_codes"].view(np.uint32), ref.sorted_codes)
    assert np.array_equal(v["order"].view(np.uint32), ref.order)
    assert np.array_equal(v["leaf_box"], ref.leaf_boxes)
    assert np.array_equal(v["root_box"], ref.root)
    nodes = v["nodes"]
    assert np.array_equal(nodes[:, 12].view(np.int32), ref.left)
    assert np.array_equal(nodes[:, 13].view(np.int32), ref.right)
    lb = np.where((ref.left < 0)[:, None], ref.leaf_boxes[np.where(ref.left < 0, ~ref.left, 0)],
                  ref.node_boxes[np.maximum(ref.left, 0)])
    rb = np.where((ref.right < 0)[:, None], ref.leaf_boxes[np.where(ref.right < 0, ~ref.right, 0)],
                  ref.node_boxes[np.maximum(ref.right, 0)])
    assert np.array_equal(nodes[:, 0:6], lb) and np.array_equal(nodes[:, 6:12], rb)
    check_wide_tree(b, ref, sc.n)


def test_full_size_blender_hit_sets(oracle):
    """Per-slab hit sets bit-exact on 256 HITTING rays of the full-size C1
    view (explicit-ray launch of the bench's kernel), pixels within the bar."""
    wl = synth.workload("blender")
    sc, cam, p = wl.scene, wl.cameras[0], wl.params
    o_all, d_all = oracle.camera_rays(cam)
    g, b = gpu_build(sc, p)
    full = rg.render_forward(g, b, rg.Config.of(p), camera=cam)
    T = full["T"].cpu().numpy()
    cand = np.nonzero(T < 0.999)[0]
    idx = np.random.default_rng(9).choice(cand, 256, replace=False)
    o, d = o_all[idx], d_all[idx]
    ref_bvh = oracle.BVH(sc, p)
    r = gpu_forward(g, b, p, o, d, debug=(256, 20000))
    ref = oracle.render(sc, p, o, d, mode=2, bvh=ref_bvh, dump_cap=20000)
    ok = compare_pixels(oracle, sc, p, o, d, r, ref)
    assert ok.sum() >= 250
    for k in range(256):
        if ok[k]:
            n = r["debug_counts"][k]
            assert n > 0
            assert np.array_equal(r["debug_records"][k, :n], ref["dump"][k]), k


@pytest.mark.parametrize("tile,shards", [(16, 3), (8, 1), (6, 4)])
def test_tile_sharded_camera(oracle, tile, shards):
    """Interleaved tile sharding (rg_camera.tile; rays are
    independent): the shards' rays are exactly the full frame's
    (camera rays bit-exact through the slot -> pixel map, ragged squares' slots
    are misses), the rendered pixels are bit-identical to the full-frame
    render, and the gradients summed over the shards equal the full frame's."""
    import dataclasses
    sc = synth.random_scene(2006, 150, sh_degree=2, sg_count=2, density_range=(2, 30),
                            scale_range=(0.03, 0.12), extent=0.45)
    p = synth.RenderParams(dt=3e-3, t_eps=1e-4, background=(0.3, 0.2, 0.1))
    cam = synth.orbit_camera(2.2, 40, 20, 45, 37, 50.0)        # ragged in both axes
    cam.rect = (2, 1, 43, 36)
    g, b = gpu_build(sc, p)
    cfg = rg.Config.of(p)
    full = rg.render_forward(g, b, cfg, camera=cam, log=rg.new_log(cam.n_rays))
    fo, fd = rg.camera_rays(cam)
    up = torch.from_numpy(np.random.default_rng(1).normal(size=(cam.n_rays, 3)).astype(np.float32)).cuda()
    gfull = rg.render_backward(g, b, cfg, full, up, camera=cam)
    acc = g.zeros_like_grads()
    seen = np.zeros(cam.n_rays, int)
    for r in range(shards):
        c = dataclasses.replace(cam, tile=tile, shard=r, shards=shards)
        assert rg.camera_ray_count(c) == c.n_rays
        pix = c.slot_pixels()
        ins = pix >= 0
        seen[pix[ins]] += 1
        o, d = rg.camera_rays(c)
        assert np.array_equal(o.cpu().numpy()[ins], fo.cpu().numpy()[pix[ins]])
        assert np.array_equal(d.cpu().numpy()[ins], fd.cpu().numpy()[pix[ins]])
        out = rg.render_forward(g, b, cfg, camera=c, log=rg.new_log(c.n_rays))
        rgb, T, rep = (out[k].cpu().numpy() for k in ("rgb", "T", "replay"))
        assert np.array_equal(rgb[ins], full["rgb"].cpu().numpy()[pix[ins]])
        assert np.array_equal(T[ins], full["T"].cpu().numpy()[pix[ins]])
        assert np.array_equal(rep[ins], full["replay"].cpu().numpy()[pix[ins]])
        assert np.all(rgb[~ins] == np.float32(p.background)) and np.all(T[~ins] == 1)
        assert np.all(rep[~ins] == -1)
        ups = torch.zeros(c.n_rays, 3, device="cuda")
        ups[torch.from_numpy(np.nonzero(ins)[0]).cuda()] = up[torch.from_numpy(pix[ins]).cuda()]
        rg.render_backward(g, b, cfg, out, ups, camera=c, grads=acc)
    assert np.all(seen == 1)
    torch.cuda.synchronize()
    for k in gfull:
        a, bb = acc[k].double(), gfull[k].double()
        scale = bb.abs().max().item()
        if scale > 0:
            assert (a - bb).abs().max().item() <= 1e-5 * scale, k
