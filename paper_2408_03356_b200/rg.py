"""Thin ctypes binding of the C-ABI in include/rg.h (libraygauss.so).

Argument marshalling only: torch tensors provide device memory and the current
CUDA stream; every step of the path runs in the library's sm_100a kernels.
There is no CPU fallback: if the library cannot be loaded, or CUDA is not
available, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

from . import build as _build

__all__ = ["RGError", "Config", "Gaussians", "BVH", "lib", "build_bvh", "camera_rays",
           "render_forward", "render_backward", "l1_loss_grad", "camera_struct", "STAT_KEYS"]

STAT_KEYS = ("rays", "rays_hit", "slabs", "pairs", "evals", "samples", "overflows", "fetches",
             "node_visits", "stack_overflows", "nonfinite_grads", "restarts")


class RGError(RuntimeError):
    pass


class _Gaussians(C.Structure):
    _fields_ = [("n", C.c_int32), ("sh_degree", C.c_int32), ("sg_count", C.c_int32),
                ("pad_", C.c_int32)] + [(k, C.c_void_p) for k in
                                        ("mean", "quat", "scale", "density", "sh", "sg_amp",
                                         "sg_sharp", "sg_axis")]


class _Grads(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("mean", "quat", "scale", "density", "sh", "sg_amp",
                                          "sg_sharp", "sg_axis")]


class _Config(C.Structure):
    _fields_ = [("dt", C.c_float), ("slab_samples", C.c_int32), ("sigma_eps", C.c_float),
                ("t_eps", C.c_float), ("hit_capacity", C.c_int32), ("radius_mode", C.c_int32),
                ("k_sigma", C.c_float), ("t_near", C.c_float), ("background", C.c_float * 3),
                ("basis", C.c_int32), ("list_capacity", C.c_int32)]


class _AdamConfig(C.Structure):
    _fields_ = [("n", C.c_int32), ("sh_degree", C.c_int32), ("sg_count", C.c_int32),
                ("step", C.c_int32), ("lr", C.c_float * 9), ("beta1", C.c_float),
                ("beta2", C.c_float), ("eps", C.c_float), ("sh_active", C.c_int32),
                ("sg_active", C.c_int32)]


class _Rays(C.Structure):
    _fields_ = [("n", C.c_int32), ("pad_", C.c_int32), ("origin", C.c_void_p), ("dir", C.c_void_p)]


class _Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("x0", C.c_int32), ("y0", C.c_int32),
                ("x1", C.c_int32), ("y1", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("c2w", C.c_float * 12),
                ("spp", C.c_int32), ("tile", C.c_int32), ("shard", C.c_int32),
                ("shards", C.c_int32), ("pad_", C.c_int32)]


class _BVH(C.Structure):
    _fields_ = [("n", C.c_int32), ("sh_degree", C.c_int32), ("sg_count", C.c_int32),
                ("app_stride", C.c_int32)] + [(k, C.c_void_p) for k in
                                              ("geom", "app", "nodes", "wide", "wide_info",
                                               "leaf_box", "root_box", "codes", "sorted_codes",
                                               "order")]


EXPORTS = ("rg_status_string", "rg_version", "rg_kernel_launches", "rg_bvh_workspace_bytes", "rg_build_bvh",
           "rg_refit_bvh", "rg_adam_step", "rg_dssim_workspace_bytes", "rg_l1_dssim_loss_grad",
           "rg_supersample_resolve", "rg_supersample_spread", "rg_densify_accumulate",
           "rg_densify_workspace_bytes", "rg_densify_plan", "rg_densify_apply",
           "rg_camera_ray_count", "rg_camera_rays", "rg_render_forward", "rg_backward_workspace_bytes",
           "rg_render_backward", "rg_l1_loss_grad", "rg_fetch_log_bytes")

_lib = None


def lib(load_only: bool = False):
    """Load libraygauss.so (building it in-tree with nvcc if missing/stale)."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    if _build.stale():
        try:
            _build.build()
        except Exception as e:  # noqa: BLE001
            if not os.path.exists(path):
                raise RGError(f"libraygauss.so missing and build failed: {e}") from e
    try:
        L = C.CDLL(path)
    except OSError as e:
        raise RGError(f"cannot load {path}: {e}") from e
    P, I32, SZ = C.c_void_p, C.c_int32, C.c_size_t
    L.rg_status_string.restype = C.c_char_p
    L.rg_status_string.argtypes = [C.c_int]
    L.rg_version.restype = C.c_char_p
    L.rg_kernel_launches.restype = C.c_ulonglong
    L.rg_bvh_workspace_bytes.restype = SZ
    L.rg_bvh_workspace_bytes.argtypes = [I32, I32, I32]
    L.rg_build_bvh.restype = C.c_int
    L.rg_build_bvh.argtypes = [P, P, P, SZ, P, P]
    L.rg_refit_bvh.restype = C.c_int
    L.rg_refit_bvh.argtypes = [P, P, P, SZ, P, P]
    L.rg_adam_step.restype = C.c_int
    L.rg_adam_step.argtypes = [P, P, P, P, P, P, P]
    L.rg_dssim_workspace_bytes.restype = SZ
    L.rg_dssim_workspace_bytes.argtypes = [I32, I32]
    L.rg_l1_dssim_loss_grad.restype = C.c_int
    L.rg_l1_dssim_loss_grad.argtypes = [P, P, I32, I32, C.c_float, P, P, P, SZ, P]
    L.rg_supersample_resolve.restype = C.c_int
    L.rg_supersample_resolve.argtypes = [P, C.c_int64, I32, P, P]
    L.rg_supersample_spread.restype = C.c_int
    L.rg_supersample_spread.argtypes = [P, C.c_int64, I32, P, P]
    L.rg_densify_accumulate.restype = C.c_int
    L.rg_densify_accumulate.argtypes = [P, I32, P, P, P]
    L.rg_densify_workspace_bytes.restype = SZ
    L.rg_densify_workspace_bytes.argtypes = [I32]
    L.rg_densify_plan.restype = C.c_int
    L.rg_densify_plan.argtypes = [P, P, P, C.c_float, C.c_float, C.c_float, C.c_float, P, P, SZ, P, P]
    L.rg_densify_apply.restype = C.c_int
    L.rg_densify_apply.argtypes = [P, P, P, P, P, P, I32, P, P]
    L.rg_camera_ray_count.restype = C.c_int64
    L.rg_camera_ray_count.argtypes = [P]
    L.rg_camera_rays.restype = C.c_int
    L.rg_camera_rays.argtypes = [P, P, P, P]
    L.rg_render_forward.restype = C.c_int
    L.rg_render_forward.argtypes = [P, P, P, P, P, P, P, P, P, SZ, P, I32, I32, P, P, P]
    L.rg_fetch_log_bytes.restype = SZ
    L.rg_fetch_log_bytes.argtypes = [I32, I32]
    L.rg_backward_workspace_bytes.restype = SZ
    L.rg_backward_workspace_bytes.argtypes = [I32, I32, I32]
    L.rg_render_backward.restype = C.c_int
    L.rg_render_backward.argtypes = [P, P, P, P, P, P, P, P, P, SZ, P, P, P, P, SZ, P]
    L.rg_l1_loss_grad.restype = C.c_int
    L.rg_l1_loss_grad.argtypes = [P, P, C.c_int64, C.c_float, P, P, P]
    _lib = L
    return L


def _check(status: int, what: str):
    if status != 0:
        msg = lib().rg_status_string(status).decode()
        raise RGError(f"{what}: {msg} ({status})")


def _require_cuda():
    if not torch.cuda.is_available():
        raise RGError("CUDA device required: libraygauss has no CPU path")


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr()) if t.numel() > 0 else None


@dataclass
class Config:
    dt: float = 2.5e-4
    slab_samples: int = 8
    sigma_eps: float = 0.1
    t_eps: float = 1e-4
    hit_capacity: int = 512
    radius_mode: int = 0
    k_sigma: float = 3.0
    t_near: float = 0.0
    background: tuple = (1.0, 1.0, 1.0)
    basis: int = 0            # RG_BASIS_*: 0 Gaussian, 1 Bump, 2 Wendland, 3 inverse
                              # multiquadric, 4 inverse quadratic, 5 C0-Matern
    list_capacity: int = 0    # forward kernel-variant hint (rg.h): > 64 = large active list

    @classmethod
    def of(cls, p) -> "Config":
        return cls(p.dt, p.slab_samples, p.sigma_eps, p.t_eps, p.hit_capacity, p.radius_mode,
                   p.k_sigma, p.t_near, tuple(p.background), getattr(p, "basis", 0),
                   getattr(p, "list_capacity", 0))

    def struct(self) -> _Config:
        c = _Config()
        c.dt, c.slab_samples, c.sigma_eps, c.t_eps = self.dt, self.slab_samples, self.sigma_eps, self.t_eps
        c.hit_capacity, c.radius_mode, c.k_sigma, c.t_near = (self.hit_capacity, self.radius_mode,
                                                              self.k_sigma, self.t_near)
        for i in range(3):
            c.background[i] = self.background[i]
        c.basis = self.basis
        c.list_capacity = self.list_capacity
        return c


GROUPS = ("mean", "quat", "scale", "density", "sh", "sg_amp", "sg_sharp", "sg_axis")


class Gaussians:
    """Activated parameters as contiguous fp32 CUDA tensors (caller layout of rg.h)."""

    def __init__(self, mean, quat, scale, density, sh, sg_amp=None, sg_sharp=None, sg_axis=None,
                 *, sh_degree=None, sg_count=None):
        n = mean.shape[0]
        self.sh_degree = int(sh_degree if sh_degree is not None else round(sh.shape[1] ** 0.5) - 1)
        self.sg_count = int(sg_count if sg_count is not None else
                            (0 if sg_amp is None else sg_amp.shape[1]))
        dev = mean.device
        z = lambda *s: torch.zeros(*s, dtype=torch.float32, device=dev)  # noqa: E731
        self.mean, self.quat, self.scale, self.density, self.sh = [
            t.contiguous().float() for t in (mean, quat, scale, density, sh)]
        self.sg_amp = (sg_amp if sg_amp is not None else z(n, 0, 3)).contiguous().float()
        self.sg_sharp = (sg_sharp if sg_sharp is not None else z(n, 0)).contiguous().float()
        self.sg_axis = (sg_axis if sg_axis is not None else z(n, 0, 3)).contiguous().float()

    @classmethod
    def from_scene(cls, sc, device="cuda"):
        t = lambda a: torch.from_numpy(a).to(device)  # noqa: E731
        return cls(*[t(a) for a in sc.arrays()], sh_degree=sc.sh_degree, sg_count=sc.sg_count)

    @property
    def n(self):
        return int(self.mean.shape[0])

    def tensors(self):
        return [getattr(self, k) for k in GROUPS]

    def struct(self) -> _Gaussians:
        s = _Gaussians()
        s.n, s.sh_degree, s.sg_count = self.n, self.sh_degree, self.sg_count
        for k in GROUPS:
            setattr(s, k, _ptr(getattr(self, k)))
        return s

    def zeros_like_grads(self):
        return {k: torch.zeros_like(getattr(self, k)) for k in GROUPS}


class BVH:
    def __init__(self, ws, handle: _BVH, scene: Gaussians):
        self.ws = ws
        self.h = handle
        self.scene = scene   # keep parameters alive

    def check(self):
        """Raise if the build's 32-wide collapse flagged an error (synchronises)."""
        if self.h.n > 1 and int(self.debug_views()["wide_info"][3].item()) != 0:
            raise RGError("rg_build_bvh: 32-wide collapse error (rg_bvh.wide_info[3])")
        return self

    def debug_views(self):
        """Device arrays of the build for parity tests."""
        n = self.h.n
        dev = self.ws.device

        def view(addr, count, dtype, itemsize):
            if count <= 0:
                return torch.zeros(0, dtype=dtype, device=dev)
            base = self.ws.data_ptr()
            off = addr - base
            assert off % itemsize == 0
            flat = self.ws.view(torch.uint8)[off:off + count * itemsize]
            return flat.view(dtype)
        return dict(
            codes=view(self.h.codes, n, torch.int32, 4),
            sorted_codes=view(self.h.sorted_codes, n, torch.int32, 4),
            order=view(self.h.order, n, torch.int32, 4),
            nodes=view(self.h.nodes, 16 * max(n - 1, 0), torch.float32, 4).reshape(-1, 16),
            leaf_box=view(self.h.leaf_box, 6 * n, torch.float32, 4).reshape(-1, 6),
            root_box=view(self.h.root_box, 6, torch.float32, 4),
            geom=view(self.h.geom, 16 * n, torch.float32, 4).reshape(-1, 16),
            wide_info=view(self.h.wide_info, 4, torch.int32, 4),
        )

    def wide_nodes(self):
        """[count, 7, 32] view of the 32-wide nodes (6 box planes + child ids; a
        negative id is a leaf range ~((first << 3) | (count - 1)), include/rg.h)."""
        info = self.debug_views()["wide_info"].cpu()
        cnt = int(info[0])
        base = self.h.wide - self.ws.data_ptr()
        raw = self.ws.view(torch.uint8)[base:base + cnt * 896]
        return raw.view(torch.float32).reshape(cnt, 7, 32), raw.view(torch.int32).reshape(cnt, 7, 32)


def bvh_workspace(scene: Gaussians):
    nbytes = int(lib().rg_bvh_workspace_bytes(scene.n, scene.sh_degree, scene.sg_count))
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=scene.mean.device)


def build_bvh(scene: Gaussians, cfg: Config, ws=None, check=False) -> BVH:
    """Full LBVH rebuild (UpdateBVH).  `ws` (from bvh_workspace) may be
    reused across calls; the returned BVH is valid until ws is rebuilt.
    check=True synchronises and raises if the 32-wide collapse reported an
    error (rg_bvh.wide_info[3])."""
    _require_cuda()
    L = lib()
    nbytes = int(L.rg_bvh_workspace_bytes(scene.n, scene.sh_degree, scene.sg_count))
    if ws is None:
        ws = bvh_workspace(scene)
    if ws.numel() < nbytes:
        raise RGError("bvh workspace too small")
    h = _BVH()
    gs, cs = scene.struct(), cfg.struct()
    _check(L.rg_build_bvh(C.byref(gs), C.byref(cs), _ptr(ws), nbytes, C.byref(h), _stream()),
           "rg_build_bvh")
    b = BVH(ws, h, scene)
    if check:
        b.check()
    return b


def refit_bvh(bvh: BVH, scene: Gaussians, cfg: Config) -> BVH:
    """UpdateBVH by refit (rg_refit_bvh): new parameter values of a scene with
    the same n / sh_degree / sg_count, topology of the last build kept."""
    _require_cuda()
    L = lib()
    gs, cs = scene.struct(), cfg.struct()
    _check(L.rg_refit_bvh(C.byref(gs), C.byref(cs), _ptr(bvh.ws), bvh.ws.numel(), C.byref(bvh.h),
                          _stream()), "rg_refit_bvh")
    bvh.scene = scene
    return bvh


def camera_struct(cam) -> _Camera:
    s = _Camera()
    x0, y0, x1, y1 = cam.x0y0x1y1
    s.width, s.height, s.x0, s.y0, s.x1, s.y1 = cam.width, cam.height, x0, y0, x1, y1
    s.fx, s.fy, s.cx, s.cy = cam.fx, cam.fy, cam.cx, cam.cy
    flat = [float(v) for v in cam.c2w.reshape(-1)]
    for i in range(12):
        s.c2w[i] = flat[i]
    s.spp = int(getattr(cam, "spp", 1))
    s.tile = int(getattr(cam, "tile", 0))
    s.shard = int(getattr(cam, "shard", 0))
    s.shards = int(getattr(cam, "shards", 1))
    return s


def camera_ray_count(cam) -> int:
    """ray slots of a camera (rg_camera_ray_count; 0 if the camera is invalid)"""
    cs = camera_struct(cam)
    return int(lib().rg_camera_ray_count(C.byref(cs)))


def camera_rays(cam, device="cuda"):
    _require_cuda()
    n = cam.n_rays
    o = torch.empty(n, 3, dtype=torch.float32, device=device)
    d = torch.empty(n, 3, dtype=torch.float32, device=device)
    cs = camera_struct(cam)
    _check(lib().rg_camera_rays(C.byref(cs), _ptr(o), _ptr(d), _stream()), "rg_camera_rays")
    return o, d


def _device_f32(t, shape, what, device):
    """Validated contiguous fp32 device tensor for a raw pointer argument: the
    returned tensor must be kept alive until the launch has been enqueued."""
    if not isinstance(t, torch.Tensor):
        raise RGError(f"{what}: expected a torch tensor")
    if t.device != torch.device(device):
        raise RGError(f"{what}: on {t.device}, expected {device}")
    if tuple(t.shape) != tuple(shape):
        raise RGError(f"{what}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    return t.contiguous().float()


def _ray_args(rays, camera, device):
    if (rays is None) == (camera is None):
        raise RGError("pass exactly one of rays=(origin, dir) or camera=")
    if rays is not None:
        o, d = rays
        n = int(o.shape[0]) if isinstance(o, torch.Tensor) and o.dim() == 2 else -1
        o = _device_f32(o, (n, 3), "ray origins", device)
        d = _device_f32(d, (n, 3), "ray directions", device)
        r = _Rays()
        r.n = n
        r.origin, r.dir = _ptr(o), _ptr(d)
        return C.byref(r), None, r.n, (r, o, d)
    cs = camera_struct(camera)
    n = int(lib().rg_camera_ray_count(C.byref(cs)))
    if n != camera.n_rays:
        raise RGError(f"invalid camera (ray slots {n} vs {camera.n_rays})")
    return None, C.byref(cs), n, (cs,)


def check_stats(stats, what="render"):
    """Data errors the C-ABI only counts (rg.h: rg_stats) become exceptions here
    (non-finite gradients must be reported): synchronises on the
    stats tensor.  Traversal-stack overflow drops subtrees, so it is an error too."""
    s = stats_dict(stats)
    if s["nonfinite_grads"]:
        raise RGError(f"{what}: {s['nonfinite_grads']} non-finite gradient values")
    if s["stack_overflows"]:
        raise RGError(f"{what}: {s['stack_overflows']} BVH traversal stack overflows")


def new_log(n_rays, device="cuda", pairs_per_ray=0):
    """Fetch-log buffer for a training forward (rg_fetch_log_bytes)."""
    nbytes = int(lib().rg_fetch_log_bytes(int(n_rays), int(pairs_per_ray)))
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


def render_forward(scene: Gaussians, bvh: BVH, cfg: Config, *, rays=None, camera=None,
                   stats=None, debug=None, out=None, log=None, check=True):
    """Returns dict(rgb [R,3], T [R], replay [R]) (+ debug counts/records).
    `log` (from new_log) records the BVH query results for render_backward.
    With `stats` and check=True the counters are read back (a synchronisation)
    and a traversal-stack overflow raises RGError."""
    _require_cuda()
    dev = scene.mean.device
    rp, cp, n, keep = _ray_args(rays, camera, dev)
    if out is None:
        out = dict(rgb=torch.empty(n, 3, dtype=torch.float32, device=dev),
                   T=torch.empty(n, dtype=torch.float32, device=dev),
                   replay=torch.empty(n, dtype=torch.int32, device=dev))
    dbg_n, dbg_cap, dc, dr = 0, 0, None, None
    if debug is not None:
        dbg_n, dbg_cap = debug
        dc = torch.zeros(dbg_n, dtype=torch.int32, device=dev)
        dr = torch.full((dbg_n, dbg_cap, 2), -1, dtype=torch.int32, device=dev)
        out["debug_counts"], out["debug_records"] = dc, dr
    gs, cs = scene.struct(), cfg.struct()
    lw = int(log.numel()) if log is not None else 0
    _check(lib().rg_render_forward(C.byref(gs), C.byref(bvh.h), C.byref(cs), rp, cp,
                                   _ptr(out["rgb"]), _ptr(out["T"]), _ptr(out["replay"]),
                                   _ptr(log), lw, _ptr(stats), dbg_n, dbg_cap, _ptr(dc), _ptr(dr),
                                   _stream()),
           "rg_render_forward")
    out["log"] = log
    del keep
    if stats is not None and check:
        check_stats(stats, "rg_render_forward")
    return out


def backward_workspace(scene: Gaussians):
    nbytes = int(lib().rg_backward_workspace_bytes(scene.n, scene.sh_degree, scene.sg_count))
    return torch.empty(max(nbytes // 4, 4), dtype=torch.float32, device=scene.mean.device)


def render_backward(scene: Gaussians, bvh: BVH, cfg: Config, fwd: dict, d_rgb, *, rays=None,
                    camera=None, grads=None, stats=None, ws=None, check=True):
    """Accumulates dL/dparams for L = sum <d_rgb, rgb> into `grads` (dict of tensors).
    With `stats` and check=True the counters are read back (a synchronisation)
    and non-finite gradients or a traversal-stack overflow raise RGError."""
    _require_cuda()
    dev = scene.mean.device
    rp, cp, n, keep = _ray_args(rays, camera, dev)
    if grads is None:
        grads = scene.zeros_like_grads()
    if ws is None:
        ws = backward_workspace(scene)
    g = _Grads()
    for k in GROUPS:
        t = grads[k]
        ref = getattr(scene, k)
        if (t.dtype != torch.float32 or not t.is_contiguous() or t.device != dev
                or t.shape != ref.shape):
            raise RGError(f"grads[{k!r}]: need a contiguous fp32 tensor of shape "
                          f"{tuple(ref.shape)} on {dev}")
        setattr(g, k, _ptr(t))
    gs, cs = scene.struct(), cfg.struct()
    d_rgb = _device_f32(d_rgb, (n, 3), "d_rgb", dev)
    log = fwd.get("log")
    lw = int(log.numel()) if log is not None else 0
    _check(lib().rg_render_backward(C.byref(gs), C.byref(bvh.h), C.byref(cs), rp, cp,
                                    _ptr(fwd["rgb"]), _ptr(fwd["T"]), _ptr(fwd["replay"]),
                                    _ptr(log), lw, _ptr(d_rgb), C.byref(g), _ptr(stats), _ptr(ws),
                                    ws.numel() * 4, _stream()), "rg_render_backward")
    del keep
    if stats is not None and check:
        check_stats(stats, "rg_render_backward")
    return grads


def l1_loss_grad(rgb, target, scale, d_rgb=None, loss=None):
    _require_cuda()
    if d_rgb is None:
        d_rgb = torch.empty_like(rgb)
    if loss is None:
        loss = torch.zeros(1, dtype=torch.float32, device=rgb.device)
    _check(lib().rg_l1_loss_grad(_ptr(rgb), _ptr(target), rgb.numel(), float(scale), _ptr(d_rgb),
                                 _ptr(loss), _stream()), "rg_l1_loss_grad")
    return d_rgb, loss


def kernel_launches() -> int:
    return int(lib().rg_kernel_launches())


def new_stats(device="cuda"):
    return torch.zeros(16, dtype=torch.int64, device=device)


def stats_dict(t):
    v = t.cpu().tolist()
    return {k: int(v[i]) for i, k in enumerate(STAT_KEYS)}


# ---------------------------------------------------------------------------
# training-step neighbours
# ---------------------------------------------------------------------------

LR_SLOTS = ("mean", "quat", "scale", "density", "sh_dc", "sh_rest", "sg_amp", "sg_sharp", "sg_axis")
# P:642 (Blender); tuples are exponential decays (start, end) over 30,000 iterations
LR_BLENDER = dict(mean=(1.5e-5, 2.5e-6), quat=3.0e-4, scale=1.2e-2, density=1.5e-1,
                  sh_dc=1.3e-3, sh_rest=1.1e-4, sg_amp=6.0e-4, sg_sharp=1.0e-1, sg_axis=2.0e-3)
LR_MIP = dict(LR_BLENDER, density=(0.5, 0.01))


def learning_rates(it: int, table=LR_BLENDER, decay_steps: int = 30_000):
    """per-slot learning rates at iteration `it` (exponential decay, log-linear)"""
    import math
    f = min(max(it / decay_steps, 0.0), 1.0)
    out = []
    for k in LR_SLOTS:
        x = table[k]
        out.append(math.exp(math.log(x[0]) * (1 - f) + math.log(x[1]) * f) if isinstance(x, tuple)
                   else float(x))
    return out


def _arrays(d) -> _Grads:
    a = _Grads()
    for k in GROUPS:
        setattr(a, k, _ptr(d[k]))
    return a


class Adam:
    """Optimiser state of Alg. 3 (raw parameters + moments, caller layout) and
    the fused rg_adam_step.  Built from ACTIVATED parameters (inverse of the
    activations of DESIGN.md L23-L25); `step` writes the activated parameters
    back into `scene` for the next render."""

    def __init__(self, scene: Gaussians, betas=(0.9, 0.999), eps=1e-15, table=LR_BLENDER):
        self.scene, self.betas, self.eps, self.table = scene, betas, eps, table
        self.raw = {k: getattr(scene, k).clone() for k in GROUPS}
        self.raw["scale"] = torch.log(self.raw["scale"])
        self.raw["density"] = torch.log(self.raw["density"])
        self.m = {k: torch.zeros_like(v) for k, v in self.raw.items()}
        self.v = {k: torch.zeros_like(v) for k, v in self.raw.items()}
        self.t = 0

    def step(self, grads: dict, it: int = None, lrs=None, sh_active=None, sg_active=None):
        _require_cuda()
        sc = self.scene
        self.t += 1
        c = _AdamConfig()
        c.n, c.sh_degree, c.sg_count, c.step = sc.n, sc.sh_degree, sc.sg_count, self.t
        lr = lrs if lrs is not None else learning_rates(self.t - 1 if it is None else it, self.table)
        for i in range(9):
            c.lr[i] = lr[i]
        c.beta1, c.beta2, c.eps = self.betas[0], self.betas[1], self.eps
        c.sh_active = (sc.sh_degree + 1) ** 2 if sh_active is None else sh_active
        c.sg_active = sc.sg_count if sg_active is None else sg_active
        act = {k: getattr(sc, k) for k in GROUPS}
        _check(lib().rg_adam_step(C.byref(c), C.byref(_arrays(grads)), C.byref(_arrays(self.raw)),
                                  C.byref(_arrays(self.m)), C.byref(_arrays(self.v)),
                                  C.byref(_arrays(act)), _stream()), "rg_adam_step")


def l1_dssim_loss_grad(rgb, target, width: int, height: int, lam: float = 0.2, d_rgb=None,
                       loss=None, ws=None):
    """fused L = (1-lam) L1 + lam DSSIM and dL/drgb (rg_l1_dssim_loss_grad);
    rgb/target [height*width, 3] (camera-mode order).  Returns (d_rgb, loss)."""
    _require_cuda()
    L = lib()
    rgb, target = rgb.contiguous(), target.contiguous()
    if d_rgb is None:
        d_rgb = torch.empty_like(rgb)
    if loss is None:
        loss = torch.zeros(1, dtype=torch.float32, device=rgb.device)
    nb = int(L.rg_dssim_workspace_bytes(width, height))
    if ws is None:
        ws = torch.empty(max(nb // 4, 1), dtype=torch.float32, device=rgb.device)
    _check(L.rg_l1_dssim_loss_grad(_ptr(rgb), _ptr(target), width, height, lam, _ptr(d_rgb),
                                   _ptr(loss), _ptr(ws), ws.numel() * 4, _stream()),
           "rg_l1_dssim_loss_grad")
    return d_rgb, loss


def supersample_resolve(rgb_rays, spp: int, out=None):
    """RayGauss4x: [n_px*spp, 3] ray colours -> [n_px, 3] pixels (box-filter mean)"""
    _require_cuda()
    n = rgb_rays.shape[0] // spp
    out = torch.empty(n, 3, dtype=torch.float32, device=rgb_rays.device) if out is None else out
    _check(lib().rg_supersample_resolve(_ptr(rgb_rays.contiguous()), n, spp, _ptr(out), _stream()),
           "rg_supersample_resolve")
    return out


def supersample_spread(d_px, spp: int, out=None):
    """adjoint of supersample_resolve: d_rays = d_px / spp per subsample"""
    _require_cuda()
    n = d_px.shape[0]
    out = torch.empty(n * spp, 3, dtype=torch.float32, device=d_px.device) if out is None else out
    _check(lib().rg_supersample_spread(_ptr(d_px.contiguous()), n, spp, _ptr(out), _stream()),
           "rg_supersample_spread")
    return out


# ---------------------------------------------------------------------------
# adaptive density control (Alg. 3)
# ---------------------------------------------------------------------------

class DensityStats:
    """per-Gaussian accumulated ||dL/dmu|| and visible-iteration count"""

    def __init__(self, n, device="cuda"):
        self.acc = torch.zeros(n, dtype=torch.float32, device=device)
        self.cnt = torch.zeros(n, dtype=torch.int32, device=device)

    def accumulate(self, grad_mean):
        _check(lib().rg_densify_accumulate(_ptr(grad_mean.contiguous()), self.acc.numel(),
                                           _ptr(self.acc), _ptr(self.cnt), _stream()),
               "rg_densify_accumulate")


def densify(scene: Gaussians, stats: DensityStats, grad_eps: float, extent: float,
            sigma_eps: float, percent_dense: float = 0.01, z=None, adam: "Adam" = None,
            generator=None):
    """One adaptive-density-control step: returns (new Gaussians, action tensor);
    if `adam` is given its raw parameters and moments are carried over in place
    (new rows: moments zero).  z: [n,2,3] normal draws (sampled if None)."""
    _require_cuda()
    L = lib()
    n, dev = scene.n, scene.mean.device
    if z is None:
        z = torch.randn(n, 2, 3, device=dev, generator=generator)
    ws = torch.empty(max(int(L.rg_densify_workspace_bytes(n)), 16), dtype=torch.uint8, device=dev)
    action = torch.empty(n, dtype=torch.int32, device=dev)
    counts = torch.zeros(4, dtype=torch.int32, device=dev)
    gs = scene.struct()
    _check(L.rg_densify_plan(C.byref(gs), _ptr(stats.acc), _ptr(stats.cnt), grad_eps, extent,
                             sigma_eps, percent_dense, _ptr(action), _ptr(ws), ws.numel(),
                             _ptr(counts), _stream()), "rg_densify_plan")
    n_out = int(counts[3].item())

    def alloc():
        return {k: torch.empty((n_out,) + tuple(getattr(scene, k).shape[1:]), dtype=torch.float32,
                               device=dev) for k in GROUPS}

    def apply(src, mode):
        out = alloc()
        if n_out > 0:
            _check(L.rg_densify_apply(C.byref(gs), None if src is None else C.byref(_arrays(src)),
                                      _ptr(action), _ptr(ws), _ptr(counts), _ptr(z.contiguous()),
                                      mode, C.byref(_arrays(out)), _stream()), "rg_densify_apply")
        return out
    new = apply(None, 0)
    if adam is not None:
        adam.raw = apply(adam.raw, 1)
        adam.m = apply(adam.m, 2)
        adam.v = apply(adam.v, 2)
    g2 = Gaussians(*[new[k] for k in GROUPS], sh_degree=scene.sh_degree, sg_count=scene.sg_count)
    if adam is not None:
        adam.scene = g2
    return g2, action
