"""Pins of oracle/train.py (Adam, schedule, unlock, activations) against what
the paper and the mathematics fix, independent of the oracle's own formulas."""
import numpy as np
import pytest
import torch

from oracle import train as T


def _raw(rng, n=7, nc=9, G=3):
    return dict(mean=rng.normal(size=(n, 3)), quat=rng.normal(size=(n, 4)),
                scale=rng.normal(-4, 0.3, size=(n, 3)), density=rng.normal(1, 1, size=n),
                sh=rng.normal(size=(n, nc, 3)), sg_amp=rng.normal(size=(n, G, 3)),
                sg_sharp=rng.uniform(1, 30, size=(n, G)), sg_axis=rng.normal(size=(n, G, 3)))


def _zeros(d):
    return {k: np.zeros_like(v) for k, v in d.items()}


def test_mean_lr_schedule_endpoints():
    """1.5e-5 at the start, 2.5e-6 after 30,000 iterations; exponential
    decay = the geometric mean half way; Mip density 0.5 -> 0.01"""
    lr0, lr1 = T.LR_BLENDER["mean"]
    assert (lr0, lr1) == (1.5e-5, 2.5e-6)
    assert T.expon_lr(lr0, lr1, 0) == pytest.approx(1.5e-5, rel=1e-12)
    assert T.expon_lr(lr0, lr1, 30_000) == pytest.approx(2.5e-6, rel=1e-12)
    assert T.expon_lr(lr0, lr1, 15_000) == pytest.approx(np.sqrt(1.5e-5 * 2.5e-6), rel=1e-12)
    assert T.expon_lr(lr0, lr1, 45_000) == pytest.approx(2.5e-6, rel=1e-12)
    assert T.group_lr(T.LR_MIP, 30_000)["density"] == pytest.approx(0.01, rel=1e-12)
    assert T.group_lr(T.LR_MIP, 0)["density"] == pytest.approx(0.5, rel=1e-12)
    lrs = T.group_lr(T.LR_BLENDER, 123)
    assert (lrs["density"], lrs["sh_dc"], lrs["sh_rest"], lrs["sg_amp"], lrs["sg_sharp"],
            lrs["sg_axis"], lrs["scale"], lrs["quat"]) == (1.5e-1, 1.3e-3, 1.1e-4, 6.0e-4, 1.0e-1,
                                                            2.0e-3, 1.2e-2, 3.0e-4)


def test_unlock_schedule():
    """degrees 0, 1, 2, then the 7 SG, every 1000 iterations: 16
    colour functions in the end (P:680's 27 SH + 21 SG coefficients)"""
    assert T.unlocked(0, max_deg=2) == (0, 0)
    assert T.unlocked(999, max_deg=2) == (0, 0)
    assert T.unlocked(1000, max_deg=2) == (1, 0)
    assert T.unlocked(2000, max_deg=2) == (2, 0)
    deg, lobes = T.unlocked(3000, max_deg=2)
    assert (deg + 1) ** 2 + lobes == 16
    assert 3 + 3 + 4 + 1 + 3 * (deg + 1) ** 2 + 3 * lobes + lobes + 3 * lobes == 87


def test_first_adam_step_is_lr_sign():
    """Kingma & Ba: with m0 = v0 = 0 the bias-corrected first step is
    -lr * g / (|g| + eps) = -lr * sign(g) for |g| >> eps"""
    rng = np.random.default_rng(0)
    raw = _raw(rng)
    g = {k: rng.normal(size=v.shape) for k, v in raw.items()}
    # identity-activation groups: raw gradient = activated gradient
    r2, m2, v2, _ = T.adam_step(raw, _zeros(raw), _zeros(raw), g, 0)
    lrs = T.group_lr(T.LR_BLENDER, 0)
    assert np.allclose(r2["mean"] - raw["mean"], -lrs["mean"] * np.sign(g["mean"]), rtol=1e-9, atol=0)
    assert np.allclose(r2["sg_sharp"] - raw["sg_sharp"], -lrs["sg_sharp"] * np.sign(g["sg_sharp"]),
                       rtol=1e-9, atol=0)
    dc = r2["sh"][:, 0] - raw["sh"][:, 0]
    assert np.allclose(dc, -lrs["sh_dc"] * np.sign(g["sh"][:, 0]), rtol=1e-9, atol=0)


def test_constant_gradient_moves_lr_per_step():
    """constant gradient: bias correction makes mhat = g and vhat = g^2 at every
    step, so each step moves exactly lr * sign(g)"""
    rng = np.random.default_rng(1)
    raw = _raw(rng, n=3)
    g = {k: rng.normal(size=v.shape) for k, v in raw.items()}
    m, v, r = _zeros(raw), _zeros(raw), raw
    for it in range(25):
        r, m, v, _ = T.adam_step(r, m, v, g, it, lrs=dict(T.LR_BLENDER, mean=1e-3))
    assert np.allclose(r["mean"] - raw["mean"], -25e-3 * np.sign(g["mean"]), rtol=1e-9, atol=1e-15)


def test_adam_matches_torch_optim():
    """the library's Adam (torch.optim.Adam, fp64) on the raw parameters with
    the chain-ruled gradients, over a random gradient sequence"""
    rng = np.random.default_rng(2)
    raw = _raw(rng, n=5, nc=4, G=2)
    const = dict(T.LR_BLENDER, mean=1.5e-5)          # constant: torch's lr is fixed
    lrs = T.group_lr(const, 0)
    lr = T.lr_per_element(raw, lrs, 4, 2)
    m, v, r = _zeros(raw), _zeros(raw), raw
    tp = {k: torch.tensor(raw[k], dtype=torch.float64, requires_grad=True) for k in T.GROUPS}
    # torch needs one param group per distinct lr: split by element via masks -> use
    # one optimiser per (group, lr value) on masked copies
    opts = []
    for k in T.GROUPS:
        for val in np.unique(lr[k]):
            if val == 0:
                continue
            opts.append((k, val, torch.optim.Adam([tp[k]], lr=float(val), betas=(0.9, 0.999), eps=1e-15)))
    for it in range(6):
        ga = {k: rng.normal(size=raw[k].shape) for k in T.GROUPS}
        graw = T.raw_grad({k: tp[k].detach().numpy() for k in T.GROUPS}, ga)
        new = {k: tp[k].detach().clone() for k in T.GROUPS}
        for k, val, opt in opts:
            p = tp[k]
            saved = p.detach().clone()
            p.grad = torch.tensor(graw[k])
            opt.step()
            mask = torch.tensor(lr[k] == val)
            new[k][mask] = p.detach()[mask]
            with torch.no_grad():
                p.copy_(saved)
        # element-wise optimisers share the gradient history, so state per element is
        # that of its own optimiser: emulate by stepping all and keeping the masked part
        with torch.no_grad():
            for k in T.GROUPS:
                tp[k].copy_(new[k])
        r, m, v, _ = T.adam_step(r, m, v, ga, it, lrs=const, sh_active=4, sg_active=2)
    for k in T.GROUPS:
        assert np.allclose(r[k], tp[k].detach().numpy(), rtol=1e-12, atol=1e-15), k


def test_raw_grad_matches_finite_differences():
    rng = np.random.default_rng(3)
    raw = _raw(rng, n=2, nc=1, G=2)
    ga = {k: rng.normal(size=v.shape) for k, v in raw.items()}
    g = T.raw_grad(raw, ga)
    h = 1e-6
    for k in T.GROUPS:
        flat = np.asarray(raw[k], np.float64).reshape(-1)
        for i in range(min(flat.size, 12)):
            rp = {kk: np.array(vv, np.float64) for kk, vv in raw.items()}
            rm = {kk: np.array(vv, np.float64) for kk, vv in raw.items()}
            rp[k].reshape(-1)[i] += h
            rm[k].reshape(-1)[i] -= h
            fp = sum(np.sum(T.activate(rp)[kk] * ga[kk]) for kk in T.GROUPS)
            fm = sum(np.sum(T.activate(rm)[kk] * ga[kk]) for kk in T.GROUPS)
            assert (fp - fm) / (2 * h) == pytest.approx(g[k].reshape(-1)[i], rel=1e-6, abs=1e-8), (k, i)


def test_locked_coefficients_do_not_move():
    rng = np.random.default_rng(4)
    raw = _raw(rng, n=4, nc=9, G=3)
    g = {k: rng.normal(size=v.shape) for k, v in raw.items()}
    r2, m2, v2, a2 = T.adam_step(raw, _zeros(raw), _zeros(raw), g, 0, sh_active=4, sg_active=1)
    assert np.array_equal(r2["sh"][:, 4:], raw["sh"][:, 4:])
    assert not np.any(m2["sh"][:, 4:]) and not np.any(v2["sh"][:, 4:])
    for k in ("sg_amp", "sg_sharp", "sg_axis"):
        assert np.array_equal(r2[k][:, 1:], raw[k][:, 1:])
        assert not np.array_equal(r2[k][:, :1], raw[k][:, :1])
    assert np.allclose(np.linalg.norm(a2["quat"], axis=-1), 1.0)
    assert np.all(a2["scale"] > 0) and np.all(a2["density"] > 0)


# ---------------------------------------------------------------------------
# L1 + DSSIM loss oracle
# ---------------------------------------------------------------------------

def test_gaussian_window():
    g = T.gaussian_window()
    assert len(g) == 11 and g.sum() == pytest.approx(1.0, abs=1e-15)
    assert np.array_equal(g, g[::-1]) and np.argmax(g) == 5
    # variance of the taps ~ sigma^2 (truncated at +-5 = 3.33 sigma)
    k = np.arange(11) - 5
    assert np.sum(g * k * k) == pytest.approx(1.5 ** 2, rel=0.01)


def test_ssim_identical_images_is_one():
    rng = np.random.default_rng(5)
    x = rng.uniform(size=(20, 17, 3))
    import torch
    s = T.ssim_map(torch.tensor(x), torch.tensor(x)).numpy()
    assert np.allclose(s, 1.0, atol=1e-12)
    loss, g = T.l1_dssim_loss_grad(x, x)
    assert loss == pytest.approx(0.0, abs=1e-12)
    assert np.abs(g).max() < 1e-9        # L1 subgradient sign(0) = 0, SSIM at its maximum


def test_ssim_constant_images_closed_form():
    """interior of constant images a, b: sigma = 0, SSIM = (2ab + C1) / (a^2 + b^2 + C1)"""
    import torch
    a, b = 0.3, 0.7
    x = np.full((30, 30, 3), a); y = np.full((30, 30, 3), b)
    s = T.ssim_map(torch.tensor(x), torch.tensor(y)).numpy()
    inner = s[5:-5, 5:-5]
    ref = (2 * a * b + 0.01 ** 2) / (a * a + b * b + 0.01 ** 2)
    assert np.allclose(inner, ref, rtol=1e-12)


def test_ssim_matches_direct_windowed_statistics():
    """a few pixels of the SSIM map recomputed by explicit weighted sums over the
    zero-padded 11x11 neighbourhood (no convolution routine)"""
    import torch
    rng = np.random.default_rng(6)
    x = rng.uniform(size=(16, 13, 3)); y = rng.uniform(size=(16, 13, 3))
    s = T.ssim_map(torch.tensor(x), torch.tensor(y)).numpy()
    g = T.gaussian_window()
    for (i, j, c) in [(0, 0, 0), (7, 6, 1), (15, 12, 2), (3, 11, 0)]:
        mx = my = exx = eyy = exy = 0.0
        for di in range(-5, 6):
            for dj in range(-5, 6):
                ii, jj = i + di, j + dj
                if 0 <= ii < 16 and 0 <= jj < 13:
                    w = g[di + 5] * g[dj + 5]
                    xv, yv = x[ii, jj, c], y[ii, jj, c]
                    mx += w * xv; my += w * yv
                    exx += w * xv * xv; eyy += w * yv * yv; exy += w * xv * yv
        sxx, syy, sxy = exx - mx * mx, eyy - my * my, exy - mx * my
        ref = ((2 * mx * my + 1e-4) * (2 * sxy + 9e-4)) / ((mx * mx + my * my + 1e-4) * (sxx + syy + 9e-4))
        assert s[i, j, c] == pytest.approx(ref, rel=1e-12)


def test_l1_dssim_gradient_finite_differences():
    rng = np.random.default_rng(7)
    x = rng.uniform(size=(12, 14, 3)); y = rng.uniform(size=(12, 14, 3))
    loss, g = T.l1_dssim_loss_grad(x, y)
    h = 1e-6
    for (i, j, c) in [(0, 0, 0), (5, 7, 1), (11, 13, 2), (6, 0, 2)]:
        xp = x.copy(); xp[i, j, c] += h
        xm = x.copy(); xm[i, j, c] -= h
        fd = (T.l1_dssim_loss_grad(xp, y)[0] - T.l1_dssim_loss_grad(xm, y)[0]) / (2 * h)
        assert fd == pytest.approx(g[i, j, c], rel=1e-5, abs=1e-10)
    # lambda = 0 reduces to the mean L1 with its sign gradient
    l0, g0 = T.l1_dssim_loss_grad(x, y, lam=0.0)
    assert l0 == pytest.approx(np.mean(np.abs(x - y)), rel=1e-12)
    assert np.allclose(g0, np.sign(x - y) / x.size, rtol=1e-12)


# ---------------------------------------------------------------------------
# adaptive density control oracle
# ---------------------------------------------------------------------------

def _act_scene(rng, n):
    q = rng.normal(size=(n, 4))
    return dict(mean=rng.normal(size=(n, 3)).astype(np.float32),
                quat=(q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32),
                scale=np.exp(rng.normal(-4, 1, size=(n, 3))).astype(np.float32),
                density=np.exp(rng.normal(0, 1.5, size=n)).astype(np.float32),
                sh=rng.normal(size=(n, 4, 3)).astype(np.float32),
                sg_amp=rng.normal(size=(n, 1, 3)).astype(np.float32),
                sg_sharp=rng.uniform(1, 9, size=(n, 1)).astype(np.float32),
                sg_axis=rng.normal(size=(n, 1, 3)).astype(np.float32))


def test_densify_statistic_and_decisions():
    acc = np.zeros(4, np.float32); cnt = np.zeros(4, np.int32)
    acc, cnt = T.densify_accumulate(acc, cnt, [[3, 4, 0], [0, 0, 0], [1e-5, 0, 0], [0, 0, 1]])
    acc, cnt = T.densify_accumulate(acc, cnt, [[0, 0, 0], [0, 0, 0], [3e-5, 0, 0], [0, 0, 1]])
    assert list(acc) == [5.0, 0.0, np.float32(np.float32(1e-5) + np.float32(3e-5)), 2.0]
    assert list(cnt) == [1, 0, 2, 2]                     # invisible iterations do not count
    sc = dict(scale=np.array([[0.001] * 3, [0.5] * 3, [0.02, 0.001, 0.001], [0.05] * 3], np.float32),
              density=np.array([1.0, 1.0, 1.0, 0.05], np.float32))
    act = T.densify_plan(sc, acc, cnt, grad_eps=2e-5, extent=1.5, sigma_eps=0.1)
    # avg 5 -> clone (0.001 <= 0.015); never seen -> keep; avg 2e-5 >= 2e-5 and
    # max scale 0.02 > 0.015 -> split; low density -> prune (overrides densify)
    assert list(act) == [1, 0, 2, 3]


def test_densify_apply_order_and_split_geometry():
    rng = np.random.default_rng(8)
    sc = _act_scene(rng, 6)
    action = np.array([0, 1, 2, 3, 1, 2])
    z = rng.normal(size=(6, 2, 3))
    out, src = T.densify_apply(sc, action, z)
    assert list(src) == [0, 1, 4, 1, 4, 2, 2, 5, 5]      # survivors, clones, split children
    assert out["mean"].shape == (9, 3)
    for k in sc:                                          # clones are exact copies
        assert np.array_equal(out[k][3], np.asarray(sc[k][1], np.float64))
    # split children: mean + R diag(s) z, i.e. the child offset in the Gaussian's own
    # frame is s * z (invert with R^T), scale / 1.6, everything else copied
    for j, (p, k) in enumerate([(2, 0), (2, 1), (5, 0), (5, 1)]):
        row = 5 + j
        R = T.rotation64(sc["quat"][p:p + 1])[0]
        local = R.T @ (out["mean"][row] - sc["mean"][p])
        assert np.allclose(local, sc["scale"][p] * z[p, k], rtol=1e-9, atol=1e-12)
        assert np.allclose(out["scale"][row], sc["scale"][p] / 1.6, rtol=1e-12)
        assert np.array_equal(out["sh"][row], sc["sh"][p].astype(np.float64))
    # the split offsets have the Gaussian's covariance: E[(x-mu)(x-mu)^T] = R S^2 R^T
    zz = rng.normal(size=(1, 200000, 3))
    sc1 = {k: v[2:3] for k, v in sc.items()}
    R = T.rotation64(sc1["quat"])[0]
    offs = np.einsum("ab,nb->na", R, sc1["scale"][0].astype(np.float64) * zz[0])
    cov = offs.T @ offs / len(offs)
    ref = R @ np.diag(sc1["scale"][0].astype(np.float64) ** 2) @ R.T
    assert np.allclose(cov, ref, rtol=0.05, atol=0.02 * ref.max())


def test_rotation64_closed_forms():
    c = np.cos(np.pi / 4); s = np.sin(np.pi / 4)
    R = T.rotation64(np.array([[c, 0, 0, s], [1, 0, 0, 0], [c, s, 0, 0]]))
    assert np.allclose(R[0], [[0, -1, 0], [1, 0, 0], [0, 0, 1]], atol=1e-15)   # 90 deg about z
    assert np.allclose(R[1], np.eye(3), atol=1e-15)
    assert np.allclose(R[2], [[1, 0, 0], [0, 0, -1], [0, 1, 0]], atol=1e-15)   # 90 deg about x
