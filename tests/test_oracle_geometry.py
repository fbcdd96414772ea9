"""Pins of the oracle's fp32 decision path (rotation, support ellipsoid, AABB,
segment test, Morton, sort, Karras, refit, rays, bbox clip) against values the
paper/SPEC print, textbook identities and independent computations.
All CPU-only (-m "not gpu")."""
import json
import math
import os

import numpy as np
import pytest

from paper_2408_03356_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def one_gaussian(mu=(0, 0, 0), q=(1, 0, 0, 0), s=(1, 1, 1), dens=1.0, sh_degree=0):
    nc = (sh_degree + 1) ** 2
    return synth.Scene(np.array([mu], np.float32), np.array([q], np.float32),
                       np.array([s], np.float32), np.array([dens], np.float32),
                       np.zeros((1, nc, 3), np.float32), np.zeros((1, 0, 3), np.float32),
                       np.zeros((1, 0), np.float32), np.zeros((1, 0, 3), np.float32),
                       sh_degree, 0)


def qmul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.array([aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx, aw * bz + ax * by - ay * bx + az * bw])


def test_rotation_hamilton_convention(oracle):
    """R(q) v == q (0,v) q*  (textbook Hamilton rotation; P:183 reading L11)."""
    rng = np.random.default_rng(0)
    for _ in range(200):
        q = rng.normal(size=4); q /= np.linalg.norm(q)
        v = rng.normal(size=3)
        R = oracle.rotation(q.astype(np.float32)).astype(np.float64)
        qc = q * np.array([1, -1, -1, -1])
        rv = qmul(qmul(q, np.concatenate([[0], v])), qc)[1:]
        assert np.allclose(R @ v, rv, atol=1e-5)
        assert np.allclose(R @ R.T, np.eye(3), atol=1e-5)
        assert abs(np.linalg.det(R) - 1) < 1e-5
    # 90 deg about z maps x -> y
    R = oracle.rotation(np.array([math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)], np.float32))
    assert np.allclose(R @ [1, 0, 0], [0, 1, 0], atol=1e-6)


@pytest.mark.parametrize("ex", GOLD["covariance"], ids=lambda e: e["cite"])
def test_covariance_examples(oracle, ex):
    """Sigma = R S S^T R^T; SPEC S:60-62 worked examples."""
    sc = one_gaussian(q=ex["quat"], s=ex["scale"])
    M, r2, box, fl = oracle.prim_setup(sc, synth.RenderParams(sigma_eps=0.1), 0)
    # M = S^-1 R^T  =>  M^T M = Sigma^-1
    sig_inv = M.astype(np.float64).T @ M.astype(np.float64)
    assert np.allclose(np.linalg.inv(sig_inv), np.array(ex["sigma"], float), atol=1e-5)


@pytest.mark.parametrize("ex", GOLD["mahalanobis"], ids=lambda e: e["cite"])
def test_mahalanobis_examples(oracle, ex):
    sc = one_gaussian(s=ex["scale"])
    M, *_ = oracle.prim_setup(sc, synth.RenderParams(sigma_eps=0.1), 0)
    y = M.astype(np.float64) @ np.array(ex["dx"], float)
    assert abs(np.linalg.norm(y) - ex["value"]) < 1e-6


def test_mahalanobis_matches_inverse_covariance(oracle):
    """|M(x-mu)|^2 == (x-mu)^T Sigma^-1 (x-mu) with Sigma built and inverted by
    numpy from an independently computed rotation (quaternion algebra)."""
    rng = np.random.default_rng(1)
    for _ in range(100):
        q = rng.normal(size=4); q /= np.linalg.norm(q)
        s = np.exp(rng.uniform(-3, 0, 3))
        sc = one_gaussian(q=q, s=s)
        M, *_ = oracle.prim_setup(sc, synth.RenderParams(sigma_eps=0.1), 0)
        R = np.stack([qmul(qmul(q, np.concatenate([[0], e])), q * [1, -1, -1, -1])[1:]
                      for e in np.eye(3)], axis=1)
        Sig = R @ np.diag(s ** 2) @ R.T
        v = rng.normal(size=3) * s.max()
        ref = v @ np.linalg.solve(Sig, v)
        got = np.sum((M.astype(np.float64) @ v) ** 2)
        assert abs(got - ref) <= 1e-4 * ref + 1e-6


@pytest.mark.parametrize("ex", GOLD["support_radius"], ids=lambda e: e["cite"])
def test_support_radius(oracle, ex):
    """r = phi^-1(sigma_eps/sigma~) for the Gaussian."""
    sc = one_gaussian(dens=ex["sigma_tilde"])
    _, r2, _, fl = oracle.prim_setup(sc, synth.RenderParams(sigma_eps=ex["sigma_eps"]), 0)
    assert fl == 3
    assert abs(math.sqrt(r2) - ex["radius"]) < ex["tol"]


def test_support_inverse_consistency(oracle):
    """sigma~ * phi(r) == sigma_eps and sigma~ <= sigma_eps is inactive."""
    rng = np.random.default_rng(2)
    for _ in range(100):
        seps = float(np.exp(rng.uniform(-5, 0)))
        dens = seps * float(np.exp(rng.uniform(0.01, 8)))
        _, r2, _, fl = oracle.prim_setup(one_gaussian(dens=dens), synth.RenderParams(sigma_eps=seps), 0)
        assert fl == 3
        assert abs(np.float32(dens) * math.exp(-0.5 * r2) / np.float32(seps) - 1) < 1e-5
    _, _, box, fl = oracle.prim_setup(one_gaussian(dens=0.1), synth.RenderParams(sigma_eps=0.1), 0)
    assert fl == 1 and box[0] > box[3]
    # k-sigma mode: r = k
    _, r2, _, _ = oracle.prim_setup(one_gaussian(dens=5.0), synth.RenderParams(sigma_eps=0.1, radius_mode=1, k_sigma=3.0), 0)
    assert r2 == 9.0


def test_nonfinite_inactive(oracle):
    sc = one_gaussian(mu=(float("nan"), 0, 0), dens=5.0)
    _, _, _, fl = oracle.prim_setup(sc, synth.RenderParams(), 0)
    assert fl == 0


@pytest.mark.parametrize("ex", GOLD["tight_aabb"], ids=lambda e: e["cite"])
def test_tight_aabb_example(oracle, ex):
    """AABB half-extents: 90 deg z-rotation of (2,1,1) -> (1,2,1).
    The oracle pads by relative 2^-8 + (|mu|+e) 2^-18 (ARITH-4)."""
    # semi-axes s~ = s * r with r = 1: choose sigma so that r^2 = 1 exactly-ish -> use k-sigma mode
    sc = one_gaussian(q=ex["quat"], s=ex["semi_axes"], dens=5.0)
    p = synth.RenderParams(sigma_eps=0.1, radius_mode=1, k_sigma=1.0)
    _, r2, box, _ = oracle.prim_setup(sc, p, 0)
    half = (box[3:] - box[:3]) / 2
    e = np.array(ex["half_extents"], float)
    expect = e * (1 + 2 ** -8) + e * 2 ** -18
    assert np.allclose(half, expect, rtol=1e-6, atol=1e-6)


def test_aabb_contains_ellipsoid_and_is_tight(oracle):
    """Every boundary point inside the box; each face within the pad of the
    ellipsoid's extremal point."""
    rng = np.random.default_rng(3)
    for _ in range(30):
        q = rng.normal(size=4); q /= np.linalg.norm(q)
        s = np.exp(rng.uniform(-4, -1, 3))
        mu = rng.uniform(-2, 2, 3)
        sc = one_gaussian(mu=mu, q=q, s=s, dens=float(rng.uniform(1, 100)))
        M, r2, box, _ = oracle.prim_setup(sc, synth.RenderParams(sigma_eps=0.1), 0)
        Minv = np.linalg.inv(M.astype(np.float64))
        u = rng.normal(size=(10000, 3)); u /= np.linalg.norm(u, axis=1, keepdims=True)
        pts = mu.astype(np.float32).astype(np.float64) + (Minv @ (u.T * math.sqrt(r2))).T
        assert np.all(pts >= box[:3] - 1e-7) and np.all(pts <= box[3:] + 1e-7)
        # extremal extents from the support function: sqrt(r2 * e_i^T Sigma e_i)
        Sig = Minv @ Minv.T
        ext = np.sqrt(r2 * np.diag(Sig))
        half = (box[3:].astype(np.float64) - box[:3]) / 2
        assert np.all(half >= ext) and np.all(half <= ext * (1 + 2 ** -8) + (np.abs(mu) + ext) * 2 ** -17 + 1e-6)


def test_segment_examples(oracle):
    """unit sphere, o=(-2,0,0), d=+x -> roots 1 and 3."""
    M = np.eye(3, dtype=np.float32)
    for ex in GOLD["segment"]:
        hit, te, tx = oracle.isect(M, 1.0, [0, 0, 0], ex["o"], ex["d"])
        assert hit
        overl = te <= ex["seg"][1] and tx >= ex["seg"][0]
        assert overl == ex["hit"]
        if "t_entry" in ex:
            assert te == ex["t_entry"] and tx == ex["t_exit"]
    hit, te, tx = oracle.isect(M, 1.0, [0, 0, 0], [0.2, 0.1, 0], [0, 1, 0])
    assert hit and te < 0 < tx   # origin inside: segment containing t=0 hits


def test_segment_matches_fp64_quadratic(oracle):
    """[t_entry, t_exit] within fp32 rounding of the roots of
    (o+td-mu)^T Sigma^-1 (o+td-mu) = r^2 solved in fp64 (Haines form)."""
    rng = np.random.default_rng(4)
    nhit = 0
    for _ in range(2000):
        q = rng.normal(size=4); q /= np.linalg.norm(q)
        s = np.exp(rng.uniform(-3, -1, 3))
        mu = rng.uniform(-0.5, 0.5, 3)
        sc = one_gaussian(mu=mu, q=q, s=s, dens=float(rng.uniform(1, 100)))
        M, r2, _, _ = oracle.prim_setup(sc, synth.RenderParams(sigma_eps=0.1), 0)
        o = rng.normal(size=3); o = o / np.linalg.norm(o) * 2
        d = rng.uniform(-0.3, 0.3, 3) - o; d /= np.linalg.norm(d)
        o32, d32, mu32 = o.astype(np.float32), d.astype(np.float32), mu.astype(np.float32)
        hit, te, tx = oracle.isect(M, r2, mu32, o32, d32)
        Md = M.astype(np.float64)
        a = Md @ d32.astype(float); b = Md @ (o32.astype(float) - mu32)
        A, B, Cq = a @ a, a @ b, b @ b - r2
        disc = B * B - A * Cq
        if disc > 1e-6 * B * B:
            assert hit
            nhit += 1
            r1 = (-B - math.sqrt(disc)) / A
            r2_ = (-B + math.sqrt(disc)) / A
            assert abs(te - r1) < 1e-4 * (1 + abs(r1)) and abs(tx - r2_) < 1e-4 * (1 + abs(r2_))
        elif disc < -1e-6 * B * B:
            assert not hit
    assert nhit > 100


def _morton_magic(q):
    x = np.uint64(q)
    x = (x * np.uint64(0x00010001)) & np.uint64(0xFF0000FF)
    x = (x * np.uint64(0x00000101)) & np.uint64(0x0F00F00F)
    x = (x * np.uint64(0x00000011)) & np.uint64(0xC30C30C3)
    x = (x * np.uint64(0x00000005)) & np.uint64(0x49249249)
    return int(x)


def test_morton_hand_values(oracle):
    """lo corner -> 0, hi corner -> 0x3FFFFFFF, centre -> 0x38000000;
    interleave matches the magic-number spreading (independent algorithm)."""
    pts = np.array([[-1, -1, -1], [1, 1, 1], [0, 0, 0]], np.float32)
    n = 3
    sc = synth.Scene(pts, np.tile(np.float32([1, 0, 0, 0]), (n, 1)), np.full((n, 3), 0.1, np.float32),
                     np.full(n, 5.0, np.float32), np.zeros((n, 1, 3), np.float32),
                     np.zeros((n, 0, 3), np.float32), np.zeros((n, 0), np.float32),
                     np.zeros((n, 0, 3), np.float32), 0, 0)
    b = oracle.BVH(sc, synth.RenderParams())
    assert list(b.codes) == [0, 0x3FFFFFFF, 0x38000000]
    rng = np.random.default_rng(5)
    sc = synth.random_scene(5, 500)
    b = oracle.BVH(sc, synth.RenderParams())
    lo, hi = sc.mean.min(0), sc.mean.max(0)
    for i in range(500):
        u = ((sc.mean[i] - lo) / (hi - lo)).astype(np.float32)
        qv = np.clip(np.floor(u * np.float32(1024)), 0, 1023).astype(int)
        code = (_morton_magic(qv[0]) << 2) | (_morton_magic(qv[1]) << 1) | _morton_magic(qv[2])
        assert code == b.codes[i]
        # the tie-break code (L34): the next 7 bits of each axis, same interleave
        q17 = np.clip(np.floor(u * np.float32(131072)), 0, 131071).astype(int)
        assert np.array_equal(q17 >> 7, qv)
        fv = q17 & 127
        assert b.fine[i] == (_morton_magic(fv[0]) << 2) | (_morton_magic(fv[1]) << 1) | _morton_magic(fv[2])


def test_sort_and_karras_structure(oracle):
    """order == stable argsort; Karras radix-tree invariants (each leaf once,
    contiguous ranges, split at the highest differing bit of the augmented key)."""
    for seed, n in [(6, 2), (7, 3), (8, 257), (9, 3000)]:
        sc = synth.random_scene(seed, n)
        if n == 3000:   # duplicate codes exercise the index tie-break
            sc.mean[1000:1200] = sc.mean[0]
        b = oracle.BVH(sc, synth.RenderParams())
        # stable sort by (code, fine code, index) (L34), via numpy's lexsort
        assert np.array_equal(b.order, np.lexsort((np.arange(n), b.fine, b.codes)))
        assert np.array_equal(b.sorted_codes, b.codes[b.order])
        keys = [(int(c) << 32) | i for i, c in enumerate(b.sorted_codes)]
        seen_leaf = np.zeros(n, int); seen_int = np.zeros(max(n - 1, 1), int)
        rng_of = {}

        def walk(node, a, bb):
            if node < 0:
                assert a == bb == ~node
                seen_leaf[~node] += 1
                return
            seen_int[node] += 1
            rng_of[node] = (a, bb)
            p = 64 - (keys[a] ^ keys[bb]).bit_length()        # common prefix length
            bit = 63 - p
            L, R = b.left[node], b.right[node]
            g = (~L) if L < 0 else None
            # split gamma: last index whose key has 0 at `bit`
            gam = max(i for i in range(a, bb + 1) if not (keys[i] >> bit) & 1)
            assert all(not (keys[i] >> bit) & 1 for i in range(a, gam + 1))
            assert all((keys[i] >> bit) & 1 for i in range(gam + 1, bb + 1))
            walk(L, a, gam)
            walk(R, gam + 1, bb)
        if n >= 2:
            walk(0, 0, n - 1)
            assert np.all(seen_leaf == 1) and np.all(seen_int == 1)


def test_refit_union(oracle):
    """Every node box == exact union of its children; root == union of all leaves."""
    sc = synth.random_scene(10, 777)
    b = oracle.BVH(sc, synth.RenderParams())

    def box(c):
        return b.leaf_boxes[~c] if c < 0 else b.node_boxes[c]
    for i in range(sc.n - 1):
        l, r = box(b.left[i]), box(b.right[i])
        u = np.concatenate([np.minimum(l[:3], r[:3]), np.maximum(l[3:], r[3:])])
        assert np.array_equal(u, b.node_boxes[i])
    allb = b.leaf_boxes
    assert np.array_equal(b.root, np.concatenate([allb[:, :3].min(0), allb[:, 3:].max(0)]))


def test_camera_rays(oracle):
    """Principal point ray = forward axis; unit directions; a pixel rect
    reproduces the corresponding sub-block (ray independence)."""
    cam = synth.orbit_camera(3.0, 30, 20, 64, 48, 50.0)
    o, d = oracle.camera_rays(cam)
    assert np.allclose(np.linalg.norm(d.astype(float), axis=1), 1, atol=1e-6)
    assert np.allclose(o, cam.c2w[:, 3])
    cam2 = synth.Camera(65, 49, 50.0, 50.0, 32.0, 24.0, cam.c2w)   # pixel 32-0.5.. no
    cam2.cx, cam2.cy = 32.5, 24.5
    o2, d2 = oracle.camera_rays(cam2)
    mid = d2.reshape(49, 65, 3)[24, 32]
    assert np.allclose(mid, cam.c2w[:, 2], atol=1e-7)
    camr = synth.Camera(64, 48, 50.0, 50.0, 32.0, 24.0, cam.c2w, rect=(10, 5, 30, 17))
    o3, d3 = oracle.camera_rays(camr)
    assert np.array_equal(d3.reshape(12, 20, 3), d.reshape(48, 64, 3)[5:17, 10:30])


def test_camera_rays_4x(oracle):
    """RayGauss4x rays: spp = 1 is the centre ray bit for bit; for
    the principal-point pixel the 4 subrays are mirror images about the forward
    axis, each at angle atan(0.25 sqrt(2) / f) from it (square pixels), and the
    rays of pixel p are 4p .. 4p+3"""
    cam = synth.orbit_camera(3.0, 30, 20, 16, 12, 50.0)
    o1, d1 = oracle.camera_rays(cam)
    o, d = oracle.camera_rays_spp(cam, 1)
    assert np.array_equal(d, d1) and np.array_equal(o, o1)
    c2 = synth.Camera(17, 13, 40.0, 40.0, 8.5, 6.5, cam.c2w)          # pixel (8, 6) centred
    o4, d4 = oracle.camera_rays_spp(c2, 4)
    assert d4.shape == (17 * 13 * 4, 3)
    sub = d4.reshape(13, 17, 4, 3)[6, 8].astype(np.float64)
    fwd, right, down = cam.c2w[:, 2], cam.c2w[:, 0], cam.c2w[:, 1]
    ang = np.arctan2(np.linalg.norm(np.cross(sub, fwd), axis=1), sub @ fwd)
    assert np.allclose(ang, np.arctan(0.25 * np.sqrt(2) / 40.0), rtol=1e-4)
    sx = np.sign(sub @ right); sy = np.sign(sub @ down)
    assert list(sx) == [-1, 1, -1, 1] and list(sy) == [-1, -1, 1, 1]   # s = sx + 2 sy
    assert np.allclose(sub.sum(0) / np.linalg.norm(sub.sum(0)), fwd, atol=1e-6)


def test_bbox_clip(oracle):
    ex = GOLD["bbox"][0]
    hit, t0, t1 = oracle.clip(ex["box"], ex["o"], ex["d"])
    assert hit and t0 == ex["t0"] and t1 == ex["t1"]
    hit, t0, t1 = oracle.clip(ex["box"], [0.5, 0.5, 0.5], [1, 0, 0])
    assert hit and t0 == 0.0 and t1 == 0.5                      # origin inside
    hit, *_ = oracle.clip(ex["box"], [-2, 2, 0.5], [1, 0, 0])  # parallel, outside
    assert not hit
    hit, *_ = oracle.clip([np.inf] * 3 + [-np.inf] * 3, [0, 0, 0], [1, 0, 0])
    assert not hit                                              # empty scene
