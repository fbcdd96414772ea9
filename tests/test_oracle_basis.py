"""Pins of the oracle's alternative basis functions (SURVEY §8(f) NEXT-3,
supplementary P:456-515): closed-form values of phi, psi = -2 sigma~ dphi/dq
against a numerical derivative, the support radius phi^-1(sigma_eps/sigma~)
(compact bases: the unit ball), line integrals of one
isotropic primitive through its centre against closed forms (or adaptive
quadrature for the Bump), and the backward against finite differences."""
import math

import numpy as np
import pytest
from scipy import integrate

from paper_2408_03356_b200 import synth
from test_oracle_grad import fd_scene, loss
from test_oracle_render import iso_scene, Y00

GROUPS = ("mean", "quat", "scale", "density", "sh", "sg_amp", "sg_sharp", "sg_axis")


def test_phi_closed_form_values(oracle):
    for b in range(6):
        assert oracle.basis_phi(b, 0.0) == pytest.approx(1.0, abs=1e-15)      # phi(0) = 1
    assert oracle.basis_phi(0, 2 * math.log(2)) == pytest.approx(0.5, rel=1e-14)
    assert oracle.basis_phi(1, 0.25) == pytest.approx(math.exp(-1 / 3), rel=1e-14)   # e^{1-1/(1-r^2)}
    assert oracle.basis_phi(2, 0.25) == pytest.approx(0.5 ** 4 * 3, rel=1e-14)       # (1-r)^4 (4r+1)
    assert oracle.basis_phi(3, 3.0) == pytest.approx(0.5, rel=1e-14)                 # 1/sqrt(1+r^2)
    assert oracle.basis_phi(4, 1.0) == pytest.approx(0.5, rel=1e-14)                 # 1/(1+r^2)
    assert oracle.basis_phi(5, math.log(2) ** 2) == pytest.approx(0.5, rel=1e-14)    # e^{-r}
    for b in (1, 2):                                                                  # compact
        assert oracle.basis_phi(b, 1.0) == 0.0 and oracle.basis_phi(b, 1.7) == 0.0
    for b in range(6):                                                                # decreasing
        v = [oracle.basis_phi(b, q) for q in np.linspace(0, 0.99, 50)]
        assert all(x > y for x, y in zip(v, v[1:]))


@pytest.mark.parametrize("b", range(6))
def test_psi_is_minus_two_sigma_dphi_dq(oracle, b):
    sig = 3.7
    for q in (0.01, 0.2, 0.55, 0.9, 2.5):
        if b in (1, 2) and q >= 1:
            continue
        h = 1e-6 * max(q, 1e-3)
        d = (oracle.basis_phi(b, q + h) - oracle.basis_phi(b, q - h)) / (2 * h)
        assert oracle.basis_psi(b, sig, q) == pytest.approx(-2 * sig * d, rel=1e-6), (b, q)


@pytest.mark.parametrize("b,r2", [(0, 2 * math.log(10)), (1, 1.0), (2, 1.0), (3, 99.0), (4, 9.0),
                                  (5, math.log(10) ** 2)])
def test_support_radius(oracle, b, r2):
    sc = iso_scene([[0, 0, 0]], 0.1, 1.0, [1, 1, 1])
    p = synth.RenderParams(sigma_eps=0.1, basis=b)
    got = oracle.prim_setup(sc, p, 0)[1]
    assert got == pytest.approx(r2, rel=2e-7)
    if b not in (1, 2):   # global bases: phi at the support boundary = sigma_eps / sigma~
        assert oracle.basis_phi(b, float(got)) == pytest.approx(0.1, rel=1e-6)


def _phi1(b, u):        # phi of |u| (1-D profile through the centre)
    return {1: lambda: math.exp(1 - 1 / (1 - u * u)) if abs(u) < 1 else 0.0,
            2: lambda: (1 - abs(u)) ** 4 * (4 * abs(u) + 1) if abs(u) <= 1 else 0.0}[b]()


@pytest.mark.parametrize("b", range(1, 6))
def test_single_primitive_line_integral(oracle, b):
    """tau = int sigma~ phi(|t|/s) dt over the support chord: closed forms
    (Wendland 2s/3, inverse quadratic 2s atan R, inverse multiquadric 2s asinh R,
    Matern 2s (1 - e^-R)) or adaptive quadrature (Bump); the oracle's midpoint
    sum within its error, and C = c (1 - T) + T bg exactly"""
    s, seps, dt = 0.1, 0.1, 1e-4
    dens = 0.3 if b == 3 else 8.0        # keep the global supports inside the ray segment
    sc = iso_scene([[0, 0, 0]], s, dens, [0.3 / Y00, 0.6 / Y00, 0.9 / Y00])
    p = synth.RenderParams(dt=dt, slab_samples=8, sigma_eps=seps, t_eps=0.0, background=(1, 1, 1),
                           basis=b)
    o = np.float32([[-2.0, 0, 0]]); d = np.float32([[1.0, 0, 0]])
    r = oracle.render(sc, p, o, d, mode=1)
    k = float(np.float32(dens)) / seps
    R = {1: 1.0, 2: 1.0, 3: math.sqrt(k * k - 1), 4: math.sqrt(k - 1), 5: math.log(k)}[b]
    closed = {2: 2 * s / 3, 4: 2 * s * math.atan(R), 3: 2 * s * math.asinh(R),
              5: 2 * s * (1 - math.exp(-R))}
    if b in closed:
        tau = dens * closed[b]
    else:
        tau = dens * s * integrate.quad(lambda u: _phi1(b, u), -1, 1, epsabs=1e-13, epsrel=1e-13)[0]
    tau_d = -math.log(r["T"][0])
    assert abs(tau_d - tau) <= 2e-4 * tau, (tau_d, tau)
    T = r["T"][0]
    assert np.allclose(r["rgb"][0], np.array([0.3, 0.6, 0.9]) * (1 - T) + T, atol=1e-12)


@pytest.mark.parametrize("b", range(1, 6))
def test_backward_matches_finite_differences_basis(oracle, b):
    sc = fd_scene(600 + b, deg=1, sg=1)
    cam = synth.orbit_camera(1.2, 45, 20, 8, 8, 8.0)
    o, d = oracle.camera_rays(cam)
    p = synth.RenderParams(dt=5e-3, slab_samples=4, t_eps=1e-3, background=(1.0, 0.5, 0.2), basis=b)
    rng = np.random.default_rng(b)
    g = rng.normal(size=(len(o), 3))
    base = sc.copy()
    r0 = oracle.render(sc, p, o, d, mode=1)
    st = r0["s_term"]
    an = oracle.backward(sc, p, o, d, g, mode=1)
    arrays = dict(zip(GROUPS, sc.arrays()))
    for name in ("mean", "quat", "scale", "density"):
        flat = arrays[name].reshape(-1)
        fd = np.zeros(flat.size)
        for i in range(flat.size):
            x0 = float(flat[i])
            h = 2e-4 * max(abs(x0), 0.05)
            xp, xm = np.float32(x0 + h), np.float32(x0 - h)
            flat[i] = xp
            lp = loss(oracle, sc, base, p, o, d, g, st)
            flat[i] = xm
            lm = loss(oracle, sc, base, p, o, d, g, st)
            flat[i] = np.float32(x0)
            fd[i] = (lp - lm) / (float(xp) - float(xm))
        a = an[name].reshape(-1)
        scale = max(np.abs(fd).max(), 1e-12)
        assert np.abs(a - fd).max() / scale < 5e-4, (name, np.abs(a - fd).max() / scale)
