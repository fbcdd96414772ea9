"""Pins of the oracle's forward (fp64 values): SH/SG against textbook values and
scipy, compositing against SPEC worked examples and closed forms (single
Gaussian line integral with erf), brute force vs slab vs BVH, invariants
(slab-size, permutation, termination bound, conservation, background)."""
import json
import math
import os

import numpy as np
import pytest
from scipy.special import erf, sph_harm_y

from paper_2408_03356_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
Y00 = 0.28209479177387814


def fib_sphere(n):
    i = np.arange(n) + 0.5
    z = 1 - 2 * i / n
    r = np.sqrt(1 - z * z)
    ph = np.pi * (1 + 5 ** 0.5) * i
    return np.stack([r * np.cos(ph), r * np.sin(ph), z], 1)


def test_sh_constants_and_parity(oracle):
    assert abs(oracle.sh_basis(0, [0, 0, 1])[0] - GOLD["eval_sh"][0]["Y00"]) < 1e-6
    rng = np.random.default_rng(0)
    for _ in range(20):
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        a, b = oracle.sh_basis(3, d), oracle.sh_basis(3, -d)
        for l in range(4):                      # parity (-1)^l (S:180 for l=1)
            sl = slice(l * l, (l + 1) ** 2)
            assert np.allclose(b[sl], (-1) ** l * a[sl], atol=1e-14)


def test_sh_orthonormal(oracle):
    """int Y_i Y_j dOmega = delta_ij (Fibonacci-sphere quadrature)."""
    D = fib_sphere(20000)
    Y = np.stack([oracle.sh_basis(3, d) for d in D])
    G = Y.T @ Y * (4 * np.pi / len(D))
    assert np.allclose(G, np.eye(16), atol=2e-3)


def test_sh_matches_scipy_up_to_sign(oracle):
    """Each 3DGS basis function equals +-the standard real SH built from
    scipy's complex Y_l^m (sign is the convention of reading L10)."""
    D = fib_sphere(300)
    Y = np.stack([oracle.sh_basis(3, d) for d in D])
    theta = np.arccos(np.clip(D[:, 2], -1, 1)); phi = np.arctan2(D[:, 1], D[:, 0])
    col = 0
    for l in range(4):
        for m in range(-l, l + 1):
            if m == 0:
                ref = sph_harm_y(l, 0, theta, phi).real
            elif m > 0:
                ref = math.sqrt(2) * (-1) ** m * sph_harm_y(l, m, theta, phi).real
            else:
                ref = math.sqrt(2) * (-1) ** m * sph_harm_y(l, -m, theta, phi).imag
            ours = Y[:, col]
            s = np.sign(np.dot(ours, ref))
            assert np.allclose(ours, s * ref, atol=1e-12), (l, m)
            col += 1


@pytest.mark.parametrize("ex", GOLD["eval_sg"], ids=lambda e: e["cite"])
def test_sg_examples(oracle, ex):
    """c_high = sum k e^{lambda (d.p - 1)} (Eq. 15)."""
    d = np.array([1.0, 0, 0])
    p = np.array([ex["dot"], math.sqrt(max(0.0, 1 - ex["dot"] ** 2)), 0.0])
    sc = synth.Scene(np.zeros((1, 3), np.float32), np.float32([[1, 0, 0, 0]]), np.ones((1, 3), np.float32),
                     np.ones(1, np.float32), np.zeros((1, 1, 3), np.float32),
                     np.float32([[[1.0, 2.0, 3.0]]]), np.float32([[ex["lambda"]]]),
                     p.astype(np.float32)[None, None], 0, 1)
    c = oracle.color(sc, 0, d)
    f = c / np.array([1.0, 2.0, 3.0])
    assert np.allclose(f, ex["factor"], rtol=ex.get("rtol", 1e-6))


def iso_scene(mu_list, s, dens, dc, sh_degree=0):
    n = len(mu_list)
    nc = (sh_degree + 1) ** 2
    sh = np.zeros((n, nc, 3), np.float32)
    sh[:, 0, :] = np.asarray(dc, np.float32)
    return synth.Scene(np.asarray(mu_list, np.float32), np.tile(np.float32([1, 0, 0, 0]), (n, 1)),
                       np.full((n, 3), s, np.float32), np.full(n, dens, np.float32), sh,
                       np.zeros((n, 0, 3), np.float32), np.zeros((n, 0), np.float32),
                       np.zeros((n, 0, 3), np.float32), sh_degree, 0)


@pytest.mark.parametrize("ex", GOLD["compositing"], ids=lambda e: e["cite"])
def test_compositing_examples(oracle, ex):
    """sigma dt = ln 2 per sample: C = 0.5, T = 0.5; two samples 0.75 / 0.25
    (Eq. 4).  A very wide Gaussian makes sigma ~ sigma~
    constant over 1 or 2 samples of a support chord of (#samples) dt."""
    k = len(ex["sigma_dt"])
    dt = 0.01
    s = 1000.0
    chord = k * dt
    dens = math.log(2.0) / dt
    # support radius r with r s = chord/2 (k-sigma mode fixes r directly)
    sc = iso_scene([[0, 0, 0]], s, dens, [1 / Y00] * 3)
    p = synth.RenderParams(dt=dt, slab_samples=1, sigma_eps=0.1, t_eps=0.0, background=(0, 0, 0),
                           radius_mode=1, k_sigma=chord / (2 * s))
    o = np.float32([[-1, 0, 0]]); d = np.float32([[1, 0, 0]])
    r = oracle.render(sc, p, o, d, mode=1)
    assert r["counters"]["samples"] == k
    assert abs(r["rgb"][0, 0] - ex["C"]) < 1e-5 and abs(r["T"][0] - ex["T"]) < 1e-5


def closed_form_tau(sig_inv, mu, o, d, dens, r2):
    """int sigma~ exp(-q(t)/2) over the support chord, q(t) = (x-mu)^T Sigma^-1 (x-mu):
    = sigma~ e^{-qmin/2} sqrt(2 pi / A) erf(h sqrt(A/2)), h = sqrt((r^2-qmin)/A)."""
    v = o - mu
    A = d @ sig_inv @ d
    Bq = d @ sig_inv @ v
    tm = -Bq / A
    qmin = v @ sig_inv @ v - A * tm * tm
    h = math.sqrt(max(r2 - qmin, 0.0) / A)
    return dens * math.exp(-qmin / 2) * math.sqrt(2 * math.pi / A) * erf(h * math.sqrt(A / 2)), 2 * h


@pytest.mark.parametrize("aniso", [False, True])
def test_single_gaussian_closed_form(oracle, aniso):
    """Textbook line integral of one Gaussian: the oracle's
    T = e^{-tau_d} with |tau_d - tau| <= 2 sigma_eps dt + L dt^2 max|q''|..., and
    C = c(1 - T) + T bg exactly (telescoping)."""
    rng = np.random.default_rng(11 + aniso)
    for trial in range(20):
        dens = float(rng.uniform(5, 50)); s = 0.1
        if aniso:
            q = rng.normal(size=4); q /= np.linalg.norm(q)
            sv = s * np.exp(rng.uniform(-0.7, 0.7, 3))
        else:
            q = np.array([1.0, 0, 0, 0]); sv = np.full(3, s)
        sc = iso_scene([[0, 0, 0]], 1.0, dens, [0.7 / Y00, 0.2 / Y00, 0.4 / Y00])
        sc.quat[0] = q; sc.scale[0] = sv
        seps = 0.1
        dt = 1e-3
        p = synth.RenderParams(dt=dt, slab_samples=8, sigma_eps=seps, t_eps=0.0, background=(1, 1, 1))
        o = np.float32([[-2.0, rng.uniform(-0.05, 0.05), rng.uniform(-0.05, 0.05)]])
        dd = np.array([1.0, rng.uniform(-0.02, 0.02), rng.uniform(-0.02, 0.02)])
        d = (dd / np.linalg.norm(dd)).astype(np.float32)[None]
        r = oracle.render(sc, p, o, d, mode=1)
        T = r["T"][0]
        # independent Sigma from quaternion algebra (not the oracle's R)
        w, x, y, z = q
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                      [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                      [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
        Sig = R @ np.diag(np.float32(sv).astype(float) ** 2) @ R.T
        r2 = 2 * math.log(np.float32(dens) / np.float32(seps))
        tau, L = closed_form_tau(np.linalg.inv(Sig), np.zeros(3), o[0].astype(float),
                                 d[0].astype(float), float(np.float32(dens)), r2)
        tau_d = -math.log(T)
        A = d[0].astype(float) @ np.linalg.inv(Sig) @ d[0].astype(float)
        bound = 2 * seps * dt + L * dt * dt * dens * A / 24 * 2 + 1e-9
        assert abs(tau_d - tau) <= bound, (trial, tau_d, tau, bound)
        c = np.array([0.7, 0.2, 0.4])
        assert np.allclose(r["rgb"][0], c * (1 - T) + T, atol=1e-12)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_density_weighted_colour_colocated(oracle, mode):
    """Eq. 10-11: the colour of a sample is the DENSITY-weighted
    mean c_k = sum_l sigma_l(x) c_l / sum_l sigma_l(x).  Co-located Gaussians
    (same mu, q, s; k-sigma supports, so identical chords) have
    sigma_l(x) = sigma~_l G(x), hence c_k = sum sigma~_l c_l / sum sigma~_l at
    EVERY sample and, by telescoping Eq. 4, pixel = c_bar (1 - T) + T bg
    exactly.  Weighting by G alone (unweighted mean of the c_l), or by
    sigma~ twice, fails this."""
    rng = np.random.default_rng(31)
    dens = [7.0, 23.0, 2.5]
    cols = np.array([[0.9, 0.1, 0.3], [0.2, 0.8, 0.5], [0.05, 0.4, 0.95]])
    q = rng.normal(size=4); q /= np.linalg.norm(q)
    sv = np.float32([0.12, 0.07, 0.2])
    n = 3
    sc = synth.Scene(np.zeros((n, 3), np.float32) + np.float32([0.1, -0.05, 0.02]),
                     np.tile(np.float32(q), (n, 1)), np.tile(sv, (n, 1)),
                     np.float32(dens), (cols / Y00).astype(np.float32)[:, None, :],
                     np.zeros((n, 0, 3), np.float32), np.zeros((n, 0), np.float32),
                     np.zeros((n, 0, 3), np.float32), 0, 0)
    bg = (0.3, 0.6, 0.1)
    p = synth.RenderParams(dt=2e-3, slab_samples=8, sigma_eps=0.1, t_eps=0.0, background=bg,
                           radius_mode=1, k_sigma=3.0)
    o, d = synth.random_rays(32, 64, radius=2.0, jitter=0.15)
    r = oracle.render(sc, p, o, d, mode=mode)
    # c~ is stored in fp32: the colour the oracle sees is fp32(c/Y00) * Y00
    c_eff = (cols / Y00).astype(np.float32).astype(np.float64) * Y00
    w = np.float32(dens).astype(np.float64)
    cbar = (w[:, None] * c_eff).sum(0) / w.sum()
    T = r["T"][:, None]
    hit = r["T"] < 1.0
    assert hit.sum() >= 20
    bg32 = np.float32(bg).astype(np.float64)      # rg_config.background is fp32
    expect = cbar[None, :] * (1.0 - T) + T * bg32[None, :]
    assert np.abs(r["rgb"] - expect).max() <= 1e-12
    # the unweighted mean differs by far more than the tolerance on these rays
    wrong = c_eff.mean(0)[None, :] * (1.0 - T) + T * bg32[None, :]
    assert np.abs(r["rgb"][hit] - wrong[hit]).max() > 1e-2


def test_conservation_white_scene(oracle):
    """c == 1 everywhere, bg = 0: C + T = 1."""
    sc = synth.random_scene(20, 40, sh_degree=0)
    sc.sh[:, 0, :] = 1.0 / Y00
    cam = synth.orbit_camera(2.5, 10, 30, 24, 24, 30.0)
    o, d = oracle.camera_rays(cam)
    p = synth.RenderParams(dt=5e-3, t_eps=1e-4, background=(0, 0, 0))
    r = oracle.render(sc, p, o, d, mode=2)
    assert np.allclose(r["rgb"][:, 0] + r["T"], 1.0, atol=1e-9)


def dense_scene(seed, n=40, deg=1, sg=2):
    return synth.random_scene(seed, n, sh_degree=deg, sg_count=sg, density_range=(5, 40),
                              scale_range=(0.04, 0.15), extent=0.4)


@pytest.mark.parametrize("seed", range(6))
def test_modes_agree_bitexact(oracle, seed):
    """plain per-sample definition (mode 0) == Alg. 2 with brute-force slab sets
    (mode 1) == Alg. 2 with the oracle's BVH (mode 2), bit for bit, including
    per-slab hit sets and counters."""
    sc = dense_scene(100 + seed)
    cam = synth.orbit_camera(2.2, 40 * seed, 25, 16, 16, 18.0)
    o, d = oracle.camera_rays(cam)
    p = synth.RenderParams(dt=4e-3, slab_samples=[8, 4, 1, 16, 8, 3][seed], t_eps=1e-4,
                           background=(1, 1, 1))
    r0 = oracle.render(sc, p, o, d, mode=0)
    r1 = oracle.render(sc, p, o, d, mode=1, dump_cap=20000)
    r2 = oracle.render(sc, p, o, d, mode=2, dump_cap=20000)
    for r in (r1, r2):
        assert np.array_equal(r["rgb"], r0["rgb"]) and np.array_equal(r["T"], r0["T"])
        assert np.array_equal(r["s_term"], r0["s_term"])
        assert r["counters"] == r0["counters"]
    assert all(np.array_equal(a, b) for a, b in zip(r1["dump"], r2["dump"]))
    assert (r0["s_term"] >= 0).any()       # early termination exercised


def test_random_small_scenes_bvh_vs_brute(oracle):
    """50 random 20-primitive scenes, 16x16."""
    for seed in range(50):
        sc = synth.random_scene(200 + seed, 20, density_range=(1, 30))
        cam = synth.orbit_camera(2.5, 7 * seed, 10, 16, 16, 20.0)
        o, d = oracle.camera_rays(cam)
        p = synth.RenderParams(dt=1e-2, t_eps=1e-4)
        r1 = oracle.render(sc, p, o, d, mode=1, dump_cap=4000)
        r2 = oracle.render(sc, p, o, d, mode=2, dump_cap=4000)
        assert np.array_equal(r1["rgb"], r2["rgb"])
        assert all(np.array_equal(a, b) for a, b in zip(r1["dump"], r2["dump"]))


def test_overflow_keeps_k_smallest(oracle):
    """Hit-buffer overflow (Alg. 1, reading L7): each integrated slab
    set is the K smallest (t_entry, index) of the full per-slab set; BVH and
    brute force agree bit for bit."""
    sc = dense_scene(300, n=60, deg=0, sg=0)
    cam = synth.orbit_camera(2.2, 0, 20, 12, 12, 14.0)
    o, d = oracle.camera_rays(cam)
    K = 3
    p = synth.RenderParams(dt=4e-3, slab_samples=8, t_eps=1e-4, hit_capacity=K)
    r1 = oracle.render(sc, p, o, d, mode=1, dump_cap=20000)
    r2 = oracle.render(sc, p, o, d, mode=2, dump_cap=20000)
    assert r1["counters"]["overflows"] > 0
    assert np.array_equal(r1["rgb"], r2["rgb"])
    assert all(np.array_equal(a, b) for a, b in zip(r1["dump"], r2["dump"]))
    # independent check of the truncation rule on a few rays
    pfull = p.replace(hit_capacity=4096, t_eps=0.0)
    rf = oracle.render(sc, pfull, o, d, mode=1, dump_cap=20000)
    for ray in range(0, len(o), 7):
        full = {}
        for s, l in rf["dump"][ray]:
            full.setdefault(s, []).append(l)
        trunc = {}
        for s, l in r1["dump"][ray]:
            trunc.setdefault(s, []).append(l)
        for s, ids in trunc.items():
            assert ids == full[s][:K]


def test_slab_size_invariance(oracle):
    """B in {1,4,8,16} at fixed dt, T_eps = 0: identical output."""
    sc = dense_scene(400)
    cam = synth.orbit_camera(2.2, 70, 25, 12, 12, 14.0)
    o, d = oracle.camera_rays(cam)
    outs = [oracle.render(sc, synth.RenderParams(dt=4e-3, slab_samples=B, t_eps=0.0), o, d, mode=2)
            for B in (1, 4, 8, 16)]
    for r in outs[1:]:
        assert np.array_equal(r["rgb"], outs[0]["rgb"])


def test_ray_permutation(oracle):
    sc = dense_scene(401)
    cam = synth.orbit_camera(2.2, 10, 25, 12, 12, 14.0)
    o, d = oracle.camera_rays(cam)
    perm = np.random.default_rng(0).permutation(len(o))
    p = synth.RenderParams(dt=4e-3)
    a = oracle.render(sc, p, o, d, mode=2)
    b = oracle.render(sc, p, o[perm], d[perm], mode=2)
    assert np.array_equal(a["rgb"][perm], b["rgb"])


def test_early_termination_bound(oracle):
    """|render(T_eps) - render(0)| <= T_eps * max|c - bg|."""
    sc = dense_scene(402, deg=0, sg=0)
    cam = synth.orbit_camera(2.2, 10, 25, 16, 16, 18.0)
    o, d = oracle.camera_rays(cam)
    r0 = oracle.render(sc, synth.RenderParams(dt=4e-3, t_eps=0.0), o, d, mode=2)
    cmax = np.abs(sc.sh[:, 0, :] * Y00 - 1.0).max()
    for te in (1e-2, 1e-4):
        r = oracle.render(sc, synth.RenderParams(dt=4e-3, t_eps=te), o, d, mode=2)
        assert (r["s_term"] >= 0).any()
        assert np.abs(r["rgb"] - r0["rgb"]).max() <= te * cmax * (1 + 1e-9)


def test_empty_and_inactive_scene(oracle):
    """No active Gaussian -> background and T = 1."""
    sc = synth.random_scene(403, 10, density_range=(0.01, 0.09))
    cam = synth.orbit_camera(2.2, 10, 25, 8, 8, 10.0)
    o, d = oracle.camera_rays(cam)
    r = oracle.render(sc, synth.RenderParams(dt=4e-3, sigma_eps=0.1, background=(0.2, 0.3, 0.4)), o, d, mode=2)
    assert np.all(r["T"] == 1.0) and np.allclose(r["rgb"], [0.2, 0.3, 0.4])
    empty = sc.subset(np.arange(0))
    r = oracle.render(empty, synth.RenderParams(dt=4e-3), o, d, mode=1)
    assert np.all(r["T"] == 1.0)


def test_nonfinite_gaussian_ignored(oracle):
    sc = dense_scene(404, n=20)
    cam = synth.orbit_camera(2.2, 10, 25, 10, 10, 12.0)
    o, d = oracle.camera_rays(cam)
    p = synth.RenderParams(dt=4e-3)
    bad = sc.copy(); bad.mean[3] = np.nan; bad.sh[5, 0, 1] = np.inf
    keep = np.array([i for i in range(sc.n) if i not in (3, 5)])
    a = oracle.render(bad, p, o, d, mode=2)
    b = oracle.render(sc.subset(keep), p, o, d, mode=2)
    assert np.allclose(a["rgb"], b["rgb"], atol=1e-12)
