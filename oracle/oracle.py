"""ctypes wrapper of the C oracle (oracle/rg_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2408_03356_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rg_oracle.c")
_HDR = os.path.join(_HERE, "rg_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    stale = (not os.path.exists(_LIB) or
             os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class OgGaussians(C.Structure):
    _fields_ = [("n", C.c_int32), ("sh_degree", C.c_int32), ("sg_count", C.c_int32),
                ("pad_", C.c_int32)] + [(k, C.c_void_p) for k in
                                        ("mean", "quat", "scale", "density", "sh", "sg_amp",
                                         "sg_sharp", "sg_axis")]


class OgConfig(C.Structure):
    _fields_ = [("dt", C.c_float), ("slab_samples", C.c_int32), ("sigma_eps", C.c_float),
                ("t_eps", C.c_float), ("hit_capacity", C.c_int32), ("radius_mode", C.c_int32),
                ("k_sigma", C.c_float), ("t_near", C.c_float), ("background", C.c_float * 3),
                ("basis", C.c_int32)]


class OgCounters(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("slabs", "pairs", "evals", "samples", "overflows", "rays_hit")]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        _lib.og_build.restype = P
        _lib.og_build.argtypes = [P, P]
        _lib.og_free.argtypes = [P]
        _lib.og_bvh_views.argtypes = [P] + [P] * 11
        _lib.og_render.restype = C.c_int32
        _lib.og_render.argtypes = [P, P, P, C.c_int32, P, C.c_int32, P, P, P, P, P, P, P,
                                   C.c_int32, P, P]
        _lib.og_backward.restype = C.c_int32
        _lib.og_backward.argtypes = [P, P, C.c_int32, P, C.c_int32, P, P, P] + [P] * 8
        _lib.og_prim_setup.argtypes = [P, P, C.c_int32, P, P, P, P]
        _lib.og_isect.restype = C.c_int32
        _lib.og_isect.argtypes = [P, C.c_float, P, P, P, P, P]
        _lib.og_rotation_f32.argtypes = [P, P]
        _lib.og_morton.argtypes = [P, P, P, P, P, P]
        _lib.og_sort.argtypes = [C.c_int32, P, P, P, P]
        _lib.og_camera_rays.argtypes = [C.c_int32, C.c_int32, C.c_float, C.c_float, C.c_float,
                                        C.c_float, P, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, P, P]
        _lib.og_camera_rays_spp.argtypes = [C.c_int32, C.c_int32, C.c_float, C.c_float, C.c_float,
                                            C.c_float, P, C.c_int32, C.c_int32, C.c_int32,
                                            C.c_int32, C.c_int32, P, P]
        _lib.og_basis_phi.restype = C.c_double
        _lib.og_basis_phi.argtypes = [C.c_int32, C.c_double]
        _lib.og_basis_psi.restype = C.c_double
        _lib.og_basis_psi.argtypes = [C.c_int32, C.c_double, C.c_double]
        _lib.og_clip.restype = C.c_int32
        _lib.og_clip.argtypes = [P, P, P, C.c_float, P, P]
        _lib.og_color.argtypes = [P, C.c_int32, P, P]
        _lib.og_sh_basis.argtypes = [C.c_int32, P, P]
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


class _SceneRef:
    """Keeps contiguous copies alive while the C struct points at them."""

    def __init__(self, scene):
        self.arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in scene.arrays()]
        if self.arrs[4].size == 0:
            self.arrs[4] = np.zeros((scene.n, 1, 3), np.float32)
        self.s = OgGaussians(scene.n, scene.sh_degree, scene.sg_count, 0,
                             *[a.ctypes.data if a.size else None for a in self.arrs])

    @property
    def ptr(self):
        return C.byref(self.s)


def config(params) -> OgConfig:
    c = OgConfig()
    c.dt = params.dt; c.slab_samples = params.slab_samples; c.sigma_eps = params.sigma_eps
    c.t_eps = params.t_eps; c.hit_capacity = params.hit_capacity
    c.radius_mode = params.radius_mode; c.k_sigma = params.k_sigma; c.t_near = params.t_near
    c.basis = getattr(params, "basis", 0)
    for i in range(3):
        c.background[i] = params.background[i]
    return c


def rotation(q):
    q = np.ascontiguousarray(q, np.float32)
    R = np.zeros(9, np.float32)
    lib().og_rotation_f32(_p(q), _p(R))
    return R.reshape(3, 3)


def prim_setup(scene, params, i):
    sr = _SceneRef(scene)
    cfg = config(params)
    M = np.zeros(9, np.float32); r2 = np.zeros(1, np.float32)
    box = np.zeros(6, np.float32); fl = np.zeros(1, np.int32)
    lib().og_prim_setup(sr.ptr, C.byref(cfg), i, _p(M), _p(r2), _p(box), _p(fl))
    return M.reshape(3, 3), float(r2[0]), box, int(fl[0])


def isect(M, r2, mu, o, d):
    M = np.ascontiguousarray(M, np.float32).reshape(9)
    mu, o, d = [np.ascontiguousarray(x, np.float32) for x in (mu, o, d)]
    te = np.zeros(1, np.float32); tx = np.zeros(1, np.float32)
    hit = lib().og_isect(_p(M), C.c_float(r2), _p(mu), _p(o), _p(d), _p(te), _p(tx))
    return bool(hit), float(te[0]), float(tx[0])


def clip(box, o, d, t_near=0.0):
    box, o, d = [np.ascontiguousarray(x, np.float32) for x in (box, o, d)]
    t0 = np.zeros(1, np.float32); t1 = np.zeros(1, np.float32)
    hit = lib().og_clip(_p(box), _p(o), _p(d), C.c_float(t_near), _p(t0), _p(t1))
    return bool(hit), float(t0[0]), float(t1[0])


def camera_rays(cam):
    if getattr(cam, "spp", 1) != 1:
        return camera_rays_spp(cam, cam.spp)
    x0, y0, x1, y1 = cam.x0y0x1y1
    n = (x1 - x0) * (y1 - y0)
    o = np.zeros((n, 3), np.float32); d = np.zeros((n, 3), np.float32)
    c2w = np.ascontiguousarray(cam.c2w, np.float32)
    lib().og_camera_rays(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, _p(c2w),
                         x0, y0, x1, y1, _p(o), _p(d))
    return o, d


def camera_rays_spp(cam, spp):
    """RayGauss4x rays: spp per pixel, pixel-major (og_camera_rays_spp)"""
    x0, y0, x1, y1 = cam.x0y0x1y1
    n = (x1 - x0) * (y1 - y0) * spp
    o = np.zeros((n, 3), np.float32); d = np.zeros((n, 3), np.float32)
    c2w = np.ascontiguousarray(cam.c2w, np.float32)
    lib().og_camera_rays_spp(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, _p(c2w),
                             x0, y0, x1, y1, spp, _p(o), _p(d))
    return o, d


BASES = ("gaussian", "bump", "wendland", "inv_multiquadric", "inv_quadratic", "matern_c0")


def basis_phi(basis, q):
    return lib().og_basis_phi(basis, float(q))


def basis_psi(basis, sigma, q):
    return lib().og_basis_psi(basis, float(sigma), float(q))


def sh_basis(degree, d):
    d = np.ascontiguousarray(d, np.float64)
    out = np.zeros(16, np.float64)
    lib().og_sh_basis(degree, _p(d), _p(out))
    return out[:(degree + 1) ** 2]


def color(scene, i, d):
    sr = _SceneRef(scene)
    d = np.ascontiguousarray(d, np.float64)
    out = np.zeros(3, np.float64)
    lib().og_color(sr.ptr, i, _p(d), _p(out))
    return out


class BVH:
    def __init__(self, scene, params):
        self._sr = _SceneRef(scene)
        self._cfg = config(params)
        self.n = scene.n
        self.h = lib().og_build(self._sr.ptr, C.byref(self._cfg))
        ptrs = [C.c_void_p() for _ in range(11)]
        lib().og_bvh_views(self.h, *[C.byref(p) for p in ptrs])
        n = self.n

        def view(p, count, dt):
            if count <= 0 or not p.value:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(np.ctypeslib.as_ctypes_type(dt))),
                                         shape=(count,)).copy()
        self.codes = view(ptrs[0], n, np.uint32)
        self.sorted_codes = view(ptrs[1], n, np.uint32)
        self.order = view(ptrs[2], n, np.uint32)
        self.left = view(ptrs[3], n - 1, np.int32)
        self.right = view(ptrs[4], n - 1, np.int32)
        self.leaf_boxes = view(ptrs[5], 6 * n, np.float32).reshape(-1, 6)
        self.node_boxes = view(ptrs[6], 6 * (n - 1), np.float32).reshape(-1, 6)
        self.root = view(ptrs[7], 6, np.float32)
        self.mean_lo = view(ptrs[8], 3, np.float32)
        self.mean_hi = view(ptrs[9], 3, np.float32)
        self.fine = view(ptrs[10], n, np.uint32)

    def __del__(self):
        if getattr(self, "h", None):
            lib().og_free(self.h)
            self.h = None


def render(scene, params, ray_o, ray_d, *, mode=2, bvh=None, dec=None, force_s_term=None,
           dump_cap=0):
    """Forward (fp64 values).  Returns dict(rgb, T, s_term, counters, dump?)."""
    sr = _SceneRef(scene)
    dr = _SceneRef(dec) if dec is not None else None
    cfg = config(params)
    ray_o = np.ascontiguousarray(ray_o, np.float32)
    ray_d = np.ascontiguousarray(ray_d, np.float32)
    n = ray_o.shape[0]
    if mode == 2 and bvh is None:
        bvh = BVH(scene, params)
    rgb = np.zeros((n, 3), np.float64); T = np.zeros(n, np.float64)
    st = np.zeros(n, np.int32)
    cnt = OgCounters()
    fs = np.ascontiguousarray(force_s_term, np.int32) if force_s_term is not None else None
    dcnt = np.zeros(n, np.int32) if dump_cap else None
    dump = np.zeros((n, dump_cap, 2), np.int32) if dump_cap else None
    rc = lib().og_render(sr.ptr, dr.ptr if dr else None, C.byref(cfg), mode,
                         bvh.h if (bvh is not None and mode == 2) else None, n, _p(ray_o),
                         _p(ray_d), _p(fs) if fs is not None else None, _p(rgb), _p(T), _p(st),
                         C.byref(cnt), dump_cap, _p(dcnt) if dump_cap else None,
                         _p(dump) if dump_cap else None)
    if rc != 0:
        raise RuntimeError(f"og_render failed ({rc})")
    out = dict(rgb=rgb, T=T, s_term=st, counters=cnt.as_dict())
    if dump_cap:
        out["dump"] = [dump[r, :dcnt[r]].copy() for r in range(n)]
    return out


def backward(scene, params, ray_o, ray_d, d_rgb, *, mode=2, bvh=None):
    """fp64 gradients of sum_r <d_rgb_r, rgb_r> w.r.t. the activated parameters."""
    sr = _SceneRef(scene)
    cfg = config(params)
    ray_o = np.ascontiguousarray(ray_o, np.float32)
    ray_d = np.ascontiguousarray(ray_d, np.float32)
    d_rgb = np.ascontiguousarray(d_rgb, np.float64)
    n = ray_o.shape[0]
    if mode == 2 and bvh is None:
        bvh = BVH(scene, params)
    N, nc, G = scene.n, (scene.sh_degree + 1) ** 2, scene.sg_count
    g = dict(mean=np.zeros((N, 3)), quat=np.zeros((N, 4)), scale=np.zeros((N, 3)),
             density=np.zeros(N), sh=np.zeros((N, nc, 3)), sg_amp=np.zeros((N, G, 3)),
             sg_sharp=np.zeros((N, G)), sg_axis=np.zeros((N, G, 3)))
    rc = lib().og_backward(sr.ptr, C.byref(cfg), mode, bvh.h if mode == 2 else None, n,
                           _p(ray_o), _p(ray_d), _p(d_rgb),
                           *[_p(g[k]) for k in ("mean", "quat", "scale", "density", "sh",
                                                "sg_amp", "sg_sharp", "sg_axis")])
    if rc != 0:
        raise RuntimeError(f"og_backward failed ({rc})")
    return g
