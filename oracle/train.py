"""Oracle of the training-step neighbours of the hot path (SURVEY.md §8(f)
NEXT-1): the Adam update with the paper's per-group learning rates, schedule
and colour unlock, and the parameter activations.  Plain NumPy in float64,
one step of the algorithm per line, no fusion.

TEST INFRASTRUCTURE ONLY: imported by tests/ (and nothing in the product
package).  Pinned by tests/test_oracle_train.py.

Citations: P:n = /root/reference/PAPER.md line n.
  * Adam: Kingma & Ba 2014, Algorithm 1 (cited at P:639): with gradient g_t,
        m_t = b1 m_{t-1} + (1 - b1) g_t
        v_t = b2 v_{t-1} + (1 - b2) g_t^2
        mhat = m_t / (1 - b1^t),  vhat = v_t / (1 - b2^t)
        theta_t = theta_{t-1} - lr * mhat / (sqrt(vhat) + eps)
  * learning rates (Blender): density 1.5e-1, constant colour (SH DC)
    1.3e-3, SH 1.1e-4, SG coefficients 6.0e-4, lobe sharpness 1.0e-1, lobe
    direction 2.0e-3, scale 1.2e-2, quaternion 3.0e-4, mean exponential decay
    1.5e-5 -> 2.5e-6 over 30,000 iterations; Mip-NeRF360: density
    exponential decay 0.5 -> 0.01 over 30,000 iterations.
  * unlock: SH degrees 0, 1, 2, then the 7 SG, every 1000
    iterations; a locked coefficient is not updated.
Readings where the paper is silent (L23-L27): the optimiser holds
raw parameters; scale = exp(raw), density = exp(raw), quaternion and lobe
axis = raw / |raw|, everything else the identity; eps = 1e-15, b1 = 0.9,
b2 = 0.999 (the 3D Gaussian Splatting practice P:224 follows); exponential
decay is log-linear in the iteration, constant after the last iteration.
"""
from __future__ import annotations

import numpy as np

GROUPS = ("mean", "quat", "scale", "density", "sh", "sg_amp", "sg_sharp", "sg_axis")

LR_BLENDER = dict(mean=(1.5e-5, 2.5e-6), quat=3.0e-4, scale=1.2e-2, density=1.5e-1,
                  sh_dc=1.3e-3, sh_rest=1.1e-4, sg_amp=6.0e-4, sg_sharp=1.0e-1, sg_axis=2.0e-3)
LR_MIP = dict(LR_BLENDER, density=(0.5, 0.01))
DECAY_STEPS = 30_000


def expon_lr(lr0: float, lr1: float, it: int, steps: int = DECAY_STEPS) -> float:
    """exponential decay from lr0 at iteration 0 to lr1 at `steps`,
    log-linear interpolation, constant afterwards"""
    t = min(max(it / steps, 0.0), 1.0)
    return float(np.exp(np.log(lr0) * (1.0 - t) + np.log(lr1) * t))


def group_lr(lrs: dict, it: int) -> dict:
    out = {}
    for k, v in lrs.items():
        out[k] = expon_lr(v[0], v[1], it) if isinstance(v, tuple) else float(v)
    return out


def unlocked(it: int, every: int = 1000, max_deg: int = 3, max_lobes: int = 7):
    """(active SH degree, active SG lobes) at iteration `it`: degree 0
    from the start, one more SH degree every `every` iterations up to 2, then
    the SG (and the last SH degree if the scene has it)"""
    stage = it // every
    deg = min(stage, min(max_deg, 2))
    lobes = max_lobes if stage >= 3 else 0
    if stage >= 3 and max_deg == 3:
        deg = 3
    return deg, lobes


def activate(raw: dict) -> dict:
    """activated parameters from raw ones (readings L23-L25)"""
    a = {k: np.asarray(v, np.float64) for k, v in raw.items()}
    a["scale"] = np.exp(a["scale"])
    a["density"] = np.exp(a["density"])
    a["quat"] = a["quat"] / np.linalg.norm(a["quat"], axis=-1, keepdims=True)
    a["sg_axis"] = a["sg_axis"] / np.linalg.norm(a["sg_axis"], axis=-1, keepdims=True)
    return a


def raw_grad(raw: dict, grad_act: dict) -> dict:
    """chain rule of `activate`: dL/draw from dL/dactivated"""
    g = {k: np.asarray(v, np.float64).copy() for k, v in grad_act.items()}
    g["scale"] = grad_act["scale"] * np.exp(np.asarray(raw["scale"], np.float64))
    g["density"] = grad_act["density"] * np.exp(np.asarray(raw["density"], np.float64))
    for k in ("quat", "sg_axis"):
        r = np.asarray(raw[k], np.float64)
        nr = np.linalg.norm(r, axis=-1, keepdims=True)
        u = r / nr
        ga = np.asarray(grad_act[k], np.float64)
        g[k] = (ga - u * np.sum(u * ga, axis=-1, keepdims=True)) / nr   # (I - u u^T) g / |r|
    return g


def lr_per_element(raw: dict, lrs: dict, sh_active: int, sg_active: int) -> dict:
    """learning rate of every raw element (0 for locked colour coefficients)"""
    out = {}
    for k in GROUPS:
        shape = np.asarray(raw[k]).shape
        if k == "sh":
            lr = np.full(shape, lrs["sh_rest"])
            lr[:, 0, :] = lrs["sh_dc"]
            lr[:, sh_active:, :] = 0.0
        elif k in ("sg_amp", "sg_sharp", "sg_axis"):
            lr = np.full(shape, lrs[k])
            lr[:, sg_active:, ...] = 0.0
        else:
            lr = np.full(shape, lrs[k])
        out[k] = lr
    return out


def adam_step(raw: dict, m: dict, v: dict, grad_act: dict, it: int, *, lrs=LR_BLENDER,
              sh_active=16, sg_active=7, b1=0.9, b2=0.999, eps=1e-15):
    """one Adam step (Kingma & Ba Alg. 1) at iteration `it` (t = it + 1) on the
    raw parameters; returns (raw', m', v', activated')"""
    t = it + 1
    g = raw_grad(raw, grad_act)
    lr = lr_per_element(raw, group_lr(lrs, it), sh_active, sg_active)
    raw2, m2, v2 = {}, {}, {}
    for k in GROUPS:
        th = np.asarray(raw[k], np.float64)
        live = lr[k] > 0.0                               # locked: no update at all
        mk = b1 * np.asarray(m[k], np.float64) + (1.0 - b1) * g[k]
        vk = b2 * np.asarray(v[k], np.float64) + (1.0 - b2) * g[k] * g[k]
        mhat = mk / (1.0 - b1 ** t)
        vhat = vk / (1.0 - b2 ** t)
        upd = th - lr[k] * mhat / (np.sqrt(vhat) + eps)
        raw2[k] = np.where(live, upd, th)
        m2[k] = np.where(live, mk, m[k])
        v2[k] = np.where(live, vk, v[k])
    return raw2, m2, v2, activate(raw2)


# ---------------------------------------------------------------------------
# loss: L = (1 - lambda) L1 + lambda DSSIM, following 3D Gaussian
# Splatting practice: SSIM of Wang et al. 2004 with an 11x11 Gaussian
# window (sigma 1.5), zero padding ("same" size), C1 = 0.01^2, C2 = 0.03^2,
# per channel, averaged over pixels and channels; DSSIM = 1 - SSIM;
# lambda = 0.2 (readings L26-L27).  Images are [H, W, 3] (the ray order of
# rg_render_forward's camera mode, row-major).
# ---------------------------------------------------------------------------

SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2
SSIM_WIN = 11
SSIM_SIGMA = 1.5
LAMBDA_DSSIM = 0.2


def gaussian_window(size=SSIM_WIN, sigma=SSIM_SIGMA):
    """normalised 1-D Gaussian taps g_k ~ exp(-(k - size//2)^2 / (2 sigma^2))"""
    k = np.arange(size, dtype=np.float64) - size // 2
    g = np.exp(-(k * k) / (2.0 * sigma * sigma))
    return g / g.sum()


def _filter(img, g):
    """zero-padded 'same' correlation of each channel of img [H,W,C] with the
    separable window g (x) g (the window is symmetric: = convolution)"""
    import torch
    t = torch.as_tensor(img, dtype=torch.float64).permute(2, 0, 1).unsqueeze(1)   # [C,1,H,W]
    w = torch.as_tensor(np.outer(g, g), dtype=torch.float64)[None, None]
    out = torch.nn.functional.conv2d(t, w, padding=len(g) // 2)
    return out.squeeze(1).permute(1, 2, 0)


def ssim_map(x, y):
    """per-pixel, per-channel SSIM (Wang et al. 2004 Eq. 13) of torch fp64 [H,W,3]"""
    import torch
    g = gaussian_window()
    mx, my = _filter(x, g), _filter(y, g)
    sxx = _filter(x * x, g) - mx * mx
    syy = _filter(y * y, g) - my * my
    sxy = _filter(x * y, g) - mx * my
    return ((2 * mx * my + SSIM_C1) * (2 * sxy + SSIM_C2)) / (
        (mx * mx + my * my + SSIM_C1) * (sxx + syy + SSIM_C2))


def l1_dssim_loss_grad(rgb, target, lam=LAMBDA_DSSIM):
    """(loss, dL/drgb) of L = (1 - lam) mean|rgb - target| + lam (1 - mean SSIM),
    rgb/target [H,W,3]; the gradient by fp64 autograd of the plain definition"""
    import torch
    x = torch.tensor(np.asarray(rgb, np.float64), requires_grad=True)
    y = torch.tensor(np.asarray(target, np.float64))
    l1 = torch.mean(torch.abs(x - y))
    loss = (1.0 - lam) * l1 + lam * (1.0 - torch.mean(ssim_map(x, y)))
    loss.backward()
    return float(loss.detach()), x.grad.numpy()


# ---------------------------------------------------------------------------
# adaptive density control (Alg. 3): the 3D Gaussian
# Splatting heuristic the paper follows, with the mean-gradient criterion
# grad_mu > grad_eps and pruning of sigma~ < sigma_eps.  Readings L30-L32:
#   * statistic: per Gaussian, the mean over iterations of ||dL/dmu|| (fp32
#     accumulation acc += ||g||, cnt += (||g|| > 0), average acc / cnt);
#   * densify if avg >= grad_eps (cnt > 0): CLONE (copy) when
#     max(scale) <= percent_dense * extent, else SPLIT into 2 children at
#     mu + R(q) (s * z_k), z_k ~ N(0, I) (passed in), scale s / 1.6, other
#     parameters copied, parent removed; PRUNE sigma~ < sigma_eps (a pruned
#     Gaussian is neither cloned nor split);
#   * output order: surviving originals (index order), then clones (index
#     order), then split children (parent index order, child 0 then 1).
# Decisions are taken in fp32 (the kernel's precision); the split positions and
# scales are computed in fp64.
# ---------------------------------------------------------------------------

PERCENT_DENSE = 0.01
SPLIT_N = 2
SPLIT_SCALE = 1.6          # 0.8 * N


def densify_accumulate(acc, cnt, grad_mean):
    """acc += ||g|| (fp32), cnt += (||g|| > 0) for one iteration's dL/dmu [n,3]"""
    g = np.asarray(grad_mean, np.float32)
    nrm = np.sqrt((g[:, 0] * g[:, 0] + g[:, 1] * g[:, 1]) + g[:, 2] * g[:, 2]).astype(np.float32)
    return (np.asarray(acc, np.float32) + nrm).astype(np.float32), \
        np.asarray(cnt, np.int32) + (nrm > 0).astype(np.int32)


def densify_plan(scene_act, acc, cnt, grad_eps, extent, sigma_eps, percent_dense=PERCENT_DENSE):
    """per Gaussian action: 0 keep, 1 clone, 2 split, 3 prune (fp32 decisions)"""
    acc = np.asarray(acc, np.float32); cnt = np.asarray(cnt, np.int32)
    avg = np.where(cnt > 0, acc / np.maximum(cnt, 1).astype(np.float32), np.float32(0)).astype(np.float32)
    dens = avg >= np.float32(grad_eps)
    smax = np.max(np.asarray(scene_act["scale"], np.float32), axis=1)
    small = smax <= np.float32(np.float32(percent_dense) * np.float32(extent))
    prune = np.asarray(scene_act["density"], np.float32) < np.float32(sigma_eps)
    act = np.zeros(len(acc), np.int32)
    act[dens & small] = 1
    act[dens & ~small] = 2
    act[prune] = 3
    return act


def rotation64(q):
    """R(q) of unit-normalised (w,x,y,z) quaternions, fp64 (Hamilton)"""
    q = np.asarray(q, np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.empty((len(q), 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z); R[:, 0, 1] = 2 * (x * y - w * z); R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z); R[:, 1, 1] = 1 - 2 * (x * x + z * z); R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y); R[:, 2, 1] = 2 * (y * z + w * x); R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def densify_apply(scene_act, action, z):
    """new activated parameter arrays (dict) in the output order above;
    z [n, 2, 3] standard normal draws (only split rows are used)"""
    action = np.asarray(action)
    keep = np.nonzero((action == 0) | (action == 1))[0]
    clone = np.nonzero(action == 1)[0]
    split = np.nonzero(action == 2)[0]
    src = np.concatenate([keep, clone, np.repeat(split, SPLIT_N)]).astype(np.int64)
    out = {k: np.asarray(v)[src].astype(np.float64) for k, v in scene_act.items()}
    ns = len(split)
    if ns:
        mu = np.asarray(scene_act["mean"], np.float64)[split]
        s = np.asarray(scene_act["scale"], np.float64)[split]
        R = rotation64(np.asarray(scene_act["quat"])[split])
        zz = np.asarray(z, np.float64)[split]                       # [ns, 2, 3]
        child_mu = mu[:, None, :] + np.einsum("nab,nkb->nka", R, s[:, None, :] * zz)
        base = len(keep) + len(clone)
        out["mean"][base:] = child_mu.reshape(-1, 3)
        out["scale"][base:] = np.repeat(s / SPLIT_SCALE, SPLIT_N, axis=0)
    return out, src
