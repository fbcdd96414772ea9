"""Pins of the oracle backward: central finite differences of the fp64 forward
with decisions frozen (contributor sets, bbox, termination held fixed -- the
function whose a.e. gradient the backward computes), plus the
zero-upstream and locality properties."""
import numpy as np
import pytest

from paper_2408_03356_b200 import synth

GROUPS = ("mean", "quat", "scale", "density", "sh", "sg_amp", "sg_sharp", "sg_axis")


def fd_scene(seed, n=4, deg=2, sg=2):
    sc = synth.random_scene(seed, n, sh_degree=deg, sg_count=sg, density_range=(5, 60),
                            scale_range=(0.08, 0.2), extent=0.15)
    return sc


def loss(oracle, sc, base, p, o, d, g, st):
    r = oracle.render(sc, p, o, d, mode=1, dec=base, force_s_term=st)
    return float(np.sum(r["rgb"] * g))


@pytest.mark.parametrize("seed,deg,sg,bg", [(0, 2, 2, 1.0), (1, 3, 1, 0.0), (2, 1, 0, 1.0)])
def test_backward_matches_finite_differences(oracle, seed, deg, sg, bg):
    sc = fd_scene(500 + seed, deg=deg, sg=sg)
    cam = synth.orbit_camera(1.2, 30 * seed, 20, 8, 8, 8.0)
    o, d = oracle.camera_rays(cam)
    p = synth.RenderParams(dt=5e-3, slab_samples=4, t_eps=1e-3, background=(bg, bg * 0.5, bg))
    rng = np.random.default_rng(seed)
    g = rng.normal(size=(len(o), 3))
    base = sc.copy()
    r0 = oracle.render(sc, p, o, d, mode=1)
    st = r0["s_term"]
    an = oracle.backward(sc, p, o, d, g, mode=1)
    arrays = dict(zip(GROUPS, sc.arrays()))
    for name in GROUPS:
        arr = arrays[name]
        if arr.size == 0:
            continue
        flat = arr.reshape(-1)
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
        err = np.abs(a - fd).max() / scale
        assert err < 2e-5, (name, err, scale)


def test_zero_upstream_gives_zero(oracle):
    sc = fd_scene(600)
    cam = synth.orbit_camera(1.2, 0, 20, 8, 8, 8.0)
    o, d = oracle.camera_rays(cam)
    an = oracle.backward(sc, synth.RenderParams(dt=5e-3), o, d, np.zeros((len(o), 3)), mode=2)
    assert all(np.all(v == 0) for v in an.values())


def test_locality(oracle):
    """Two disjoint Gaussians, rays through only one: the other's gradients
    are exactly zero."""
    sc = fd_scene(601, n=2)
    sc.mean[0] = [0.0, 0.0, 0.0]
    sc.mean[1] = [5.0, 5.0, 5.0]
    o = np.float32([[-1, 0.01 * i, 0.0] for i in range(5)])
    d = np.float32([[1, 0, 0]] * 5)
    an = oracle.backward(sc, synth.RenderParams(dt=5e-3), o, d, np.ones((5, 3)), mode=2)
    assert np.abs(an["mean"][0]).max() > 0
    for k, v in an.items():
        assert np.all(v[1] == 0), k
