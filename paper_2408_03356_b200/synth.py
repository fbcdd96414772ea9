"""Seeded synthetic workloads shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the RayGauss method: it only draws scene
parameters (already "activated": unit quaternions, positive scales, positive
densities), pinhole cameras (intrinsics + camera-to-world pose) and render
parameters, with the shapes and value distributions SURVEY.md §8(d) fixes for
the five configurations C0..C4 (BASELINE.json `configs`).  Rotation matrices,
covariances, rays, supports, colours, compositing: none of that is here; the
oracle (oracle/) and the CUDA library (csrc/) each implement it on their own.

Conventions (inputs only):
  * quaternion (w, x, y, z), unit norm (PAPER.md P:183 leaves the convention
    open; reading L11);
  * SH coefficients [n, (deg+1)^2, 3] coefficient-major, RGB-minor;
  * SG amplitudes [n, G, 3], sharpness [n, G], axes [n, G, 3] unit;
  * camera: c2w is 3x4 [right | down | forward | eye] (OpenCV-style axes),
    pixel (px, py) looks through its centre ("one ray per pixel").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Scene", "Camera", "RenderParams", "Workload",
    "random_scene", "scene_tiny", "scene_blender", "scene_mip", "scene_stress",
    "look_at", "orbit_camera", "workload", "WORKLOADS", "random_rays",
]


@dataclass
class Scene:
    mean: np.ndarray      # [n,3] f32
    quat: np.ndarray      # [n,4] f32 (w,x,y,z), unit
    scale: np.ndarray     # [n,3] f32 > 0
    density: np.ndarray   # [n]   f32 > 0  (sigma-tilde)
    sh: np.ndarray        # [n,(deg+1)^2,3] f32
    sg_amp: np.ndarray    # [n,G,3] f32
    sg_sharp: np.ndarray  # [n,G] f32 >= 0
    sg_axis: np.ndarray   # [n,G,3] f32 unit
    sh_degree: int
    sg_count: int

    @property
    def n(self) -> int:
        return int(self.mean.shape[0])

    def arrays(self):
        return (self.mean, self.quat, self.scale, self.density, self.sh,
                self.sg_amp, self.sg_sharp, self.sg_axis)

    def copy(self) -> "Scene":
        return Scene(*[a.copy() for a in self.arrays()], self.sh_degree, self.sg_count)

    def subset(self, idx) -> "Scene":
        return Scene(*[np.ascontiguousarray(a[idx]) for a in self.arrays()],
                     self.sh_degree, self.sg_count)


@dataclass
class Camera:
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    c2w: np.ndarray                 # [3,4] f32
    rect: tuple | None = None       # (x0, y0, x1, y1) pixel rectangle, default full
    spp: int = 1                    # rays per pixel: 1, or 4 (RayGauss4x)
    tile: int = 0                   # > 0: interleaved tile sharding (rg.h rg_camera): this
    shard: int = 0                  #   camera covers the tile x tile squares k of the
    shards: int = 1                 #   rectangle with k % shards == shard

    @property
    def x0y0x1y1(self):
        return self.rect if self.rect is not None else (0, 0, self.width, self.height)

    def owned_squares(self):
        """(kx, ky) of the squares a tile-sharded camera covers, in ray order"""
        x0, y0, x1, y1 = self.x0y0x1y1
        nsx = -(-(x1 - x0) // self.tile)
        nsy = -(-(y1 - y0) // self.tile)
        return [(k % nsx, k // nsx) for k in range(self.shard, nsx * nsy, self.shards)]

    @property
    def n_rays(self) -> int:
        x0, y0, x1, y1 = self.x0y0x1y1
        if self.tile > 0:
            return len(self.owned_squares()) * self.tile * self.tile
        return (x1 - x0) * (y1 - y0) * self.spp

    def slot_pixels(self):
        """tile sharding: rectangle-relative row-major pixel index of every ray slot,
        -1 for slots of ragged squares outside the rectangle (index bookkeeping only)"""
        x0, y0, x1, y1 = self.x0y0x1y1
        w, h, t = x1 - x0, y1 - y0, self.tile
        out = []
        for kx, ky in self.owned_squares():
            ly, lx = np.meshgrid(np.arange(t), np.arange(t), indexing="ij")
            px, py = kx * t + lx.reshape(-1), ky * t + ly.reshape(-1)
            out.append(np.where((px < w) & (py < h), py * w + px, -1))
        return np.concatenate(out) if out else np.zeros(0, np.int64)


@dataclass
class RenderParams:
    dt: float = 2.5e-4          # Delta t (Table 5 grey row P:715)
    slab_samples: int = 8       # B ("8 samples per slab")
    sigma_eps: float = 0.1      # sigma_eps
    t_eps: float = 1e-4         # T_eps (never stated; L5)
    hit_capacity: int = 512     # n_max
    radius_mode: int = 0        # 0 = paper support radius, 1 = k-sigma
    k_sigma: float = 3.0
    t_near: float = 0.0
    background: tuple = (1.0, 1.0, 1.0)
    basis: int = 0              # basis function: 0 Gaussian, 1 Bump, 2 Wendland,
                                # 3 inverse multiquadric, 4 inverse quadratic, 5 C0-Matern
    list_capacity: int = 0      # CUDA kernel-variant hint (rg.h rg_config); no effect on results

    def replace(self, **kw) -> "RenderParams":
        d = dict(self.__dict__)
        d.update(kw)
        return RenderParams(**d)


@dataclass
class Workload:
    name: str
    scene: Scene
    cameras: list
    params: RenderParams
    notes: str = ""


# ----------------------------------------------------------------------------
# elementary draws (input construction only)
# ----------------------------------------------------------------------------

def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _random_unit_quat(rng, n):
    return _unit(rng.normal(size=(n, 4))).astype(np.float32)


def _random_dirs(rng, n):
    return _unit(rng.normal(size=(n, 3)))


def _loguniform(rng, lo, hi, size):
    return np.exp(rng.uniform(math.log(lo), math.log(hi), size=size))


def _qmul(a, b):
    """Hamilton product of quaternion arrays (w,x,y,z) -- used only to draw
    oriented inputs (align local z with a surface normal, then twist)."""
    aw, ax, ay, az = a[..., 0], a[..., 1], a[..., 2], a[..., 3]
    bw, bx, by, bz = b[..., 0], b[..., 1], b[..., 2], b[..., 3]
    return np.stack([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw], axis=-1)


def _quat_z_to(n, twist):
    """Unit quaternion whose rotation takes +z to unit normal n, composed with
    a twist about local z (input drawing only)."""
    z = np.array([0.0, 0.0, 1.0])
    c = n @ z
    axis = np.cross(np.broadcast_to(z, n.shape), n)
    q = np.concatenate([(1.0 + c)[:, None], axis], axis=1)
    bad = (1.0 + c) < 1e-9           # n == -z: rotate pi about x
    q[bad] = np.array([0.0, 1.0, 0.0, 0.0])
    q = _unit(q)
    qt = np.stack([np.cos(twist / 2), np.zeros_like(twist), np.zeros_like(twist),
                   np.sin(twist / 2)], axis=1)
    return _unit(_qmul(q, qt))


def _appearance(rng, n, sh_degree, sg_count, dc_lo=0.18, dc_hi=3.37):
    """SH + SG coefficients (SURVEY.md §8(d) C1 recipe): DC ~ U(dc_lo, dc_hi)
    (an albedo in ~[0.05,0.95] after the band-0 basis), band j ~ N(0, 0.1/j);
    SG amplitudes N(0, 0.1), sharpness U(2, 60), axes uniform."""
    nc = (sh_degree + 1) ** 2
    sh = np.zeros((n, nc, 3), np.float32)
    sh[:, 0, :] = rng.uniform(dc_lo, dc_hi, size=(n, 3))
    for j in range(1, sh_degree + 1):
        sh[:, j * j:(j + 1) * (j + 1), :] = rng.normal(0.0, 0.1 / j, size=(n, 2 * j + 1, 3))
    sg_amp = rng.normal(0.0, 0.1, size=(n, sg_count, 3)).astype(np.float32)
    sg_sharp = rng.uniform(2.0, 60.0, size=(n, sg_count)).astype(np.float32)
    sg_axis = _random_dirs(rng, n * sg_count).reshape(n, sg_count, 3).astype(np.float32)
    # re-normalise in f32 so the stored axes are unit to f32 rounding
    sg_axis = (sg_axis / np.linalg.norm(sg_axis, axis=-1, keepdims=True)).astype(np.float32)
    return sh, sg_amp, sg_sharp, sg_axis


def _f32(*arrs):
    return [np.ascontiguousarray(a, dtype=np.float32) for a in arrs]


# ----------------------------------------------------------------------------
# scenes
# ----------------------------------------------------------------------------

def random_scene(seed, n, *, sh_degree=0, sg_count=0, extent=0.6,
                 scale_range=(0.05, 0.2), density_range=(0.5, 5.0),
                 anisotropic=True, dc_range=(0.0, 3.54)):
    """Uniform random cloud (C0 recipe): mu ~ U[-e,e]^3,
    s = exp U(ln lo, ln hi), q uniform, sigma ~ U(density_range)."""
    rng = np.random.default_rng(seed)
    mean = rng.uniform(-extent, extent, size=(n, 3))
    if anisotropic:
        scale = _loguniform(rng, scale_range[0], scale_range[1], (n, 3))
    else:
        scale = np.repeat(_loguniform(rng, scale_range[0], scale_range[1], (n, 1)), 3, axis=1)
    quat = _random_unit_quat(rng, n)
    density = rng.uniform(density_range[0], density_range[1], size=n)
    sh, sg_amp, sg_sharp, sg_axis = _appearance(rng, n, sh_degree, sg_count,
                                                dc_range[0], dc_range[1])
    mean, scale, density = _f32(mean, scale, density)
    return Scene(mean, quat, scale, density, sh, sg_amp, sg_sharp, sg_axis, sh_degree, sg_count)


def scene_tiny(seed=1000):
    """C0: 64 Gaussians, SH degree 0, no SG."""
    return random_scene(seed, 64, sh_degree=0, sg_count=0)


def _surface_points(rng, n):
    """Area-sampled points + normals on four analytic shapes inside [-1.2,1.2]^3
    (sphere, torus, box shell, ground patch) -- a NeRF-synthetic-like object."""
    sph_c, sph_r = np.array([-0.45, 0.35, 0.0]), 0.45
    tor_c, tor_R, tor_r = np.array([0.5, -0.1, 0.25]), 0.40, 0.12
    box_c, box_h = np.array([0.05, -0.55, -0.45]), 0.30
    gz, g_half = -0.9, 1.1
    areas = np.array([4 * np.pi * sph_r ** 2, 4 * np.pi ** 2 * tor_R * tor_r,
                      6 * (2 * box_h) ** 2, (2 * g_half) ** 2])
    counts = rng.multinomial(n, areas / areas.sum())
    pts, nrm = [], []
    # sphere
    d = _random_dirs(rng, counts[0])
    pts.append(sph_c + sph_r * d); nrm.append(d)
    # torus (rejection sampling for area uniformity), axis = z
    m = counts[1]
    th_l, ph_l = [], []
    while sum(len(x) for x in th_l) < m:
        th = rng.uniform(0, 2 * np.pi, 2 * m)
        ph = rng.uniform(0, 2 * np.pi, 2 * m)
        keep = rng.uniform(0, 1, 2 * m) < (tor_R + tor_r * np.cos(ph)) / (tor_R + tor_r)
        th_l.append(th[keep]); ph_l.append(ph[keep])
    th = np.concatenate(th_l)[:m]; ph = np.concatenate(ph_l)[:m]
    ring = np.stack([np.cos(th), np.sin(th), np.zeros_like(th)], 1)
    tn = np.cos(ph)[:, None] * ring + np.sin(ph)[:, None] * np.array([0, 0, 1.0])
    pts.append(tor_c + tor_R * ring + tor_r * tn); nrm.append(tn)
    # box shell
    m = counts[2]
    face = rng.integers(0, 6, m)
    uv = rng.uniform(-box_h, box_h, size=(m, 2))
    axis = face // 2
    sign = np.where(face % 2 == 0, 1.0, -1.0)
    p = np.zeros((m, 3)); nb = np.zeros((m, 3))
    for a in range(3):
        sel = axis == a
        others = [b for b in range(3) if b != a]
        p[sel, a] = sign[sel] * box_h
        p[sel, others[0]] = uv[sel, 0]
        p[sel, others[1]] = uv[sel, 1]
        nb[sel, a] = sign[sel]
    pts.append(box_c + p); nrm.append(nb)
    # ground patch
    m = counts[3]
    g = np.stack([rng.uniform(-g_half, g_half, m), rng.uniform(-g_half, g_half, m),
                  np.full(m, gz)], 1)
    pts.append(g); nrm.append(np.tile([0.0, 0.0, 1.0], (m, 1)))
    return np.concatenate(pts), np.concatenate(nrm)


def _surface_gaussians(rng, pts, nrm, st_med, sigma_lo, sigma_hi, jitter):
    n = pts.shape[0]
    mean = pts + nrm * rng.normal(0.0, jitter, size=(n, 1))
    s_t = st_med * np.exp(rng.normal(0.0, 0.35, size=n)) if np.isscalar(st_med) \
        else st_med * np.exp(rng.normal(0.0, 0.35, size=n))
    scale = np.stack([s_t, s_t * rng.uniform(0.6, 1.0, n), s_t * rng.uniform(0.15, 0.5, n)], 1)
    quat = _quat_z_to(nrm, rng.uniform(0, 2 * np.pi, n))
    density = _loguniform(rng, sigma_lo, sigma_hi, n)
    return mean, quat, scale, density


def scene_blender(seed=1001, n=300_000, sh_degree=3, sg_count=7):
    """C1/C2: 300k surface-concentrated Gaussians, SH deg 3 + 7 SG lobes,
    sigma ~ LogU(20, 2000)."""
    rng = np.random.default_rng(seed)
    pts, nrm = _surface_points(rng, n)
    mean, quat, scale, density = _surface_gaussians(rng, pts, nrm, 0.006, 20.0, 2000.0, 0.002)
    sh, sg_amp, sg_sharp, sg_axis = _appearance(rng, n, sh_degree, sg_count)
    mean, quat, scale, density = _f32(mean, quat, scale, density)
    return Scene(mean, quat, scale, density, sh, sg_amp, sg_sharp, sg_axis, sh_degree, sg_count)


def scene_mip(seed=1003, n=2_000_000, sh_degree=3, sg_count=7):
    """C3: unbounded Mip-NeRF360-like scene: 60% central object (x1.25),
    15% ground disc z=-1 (rho in [1.5,15]), 25% background shell r~U(8,40);
    sigma ~ LogU(5, 500)."""
    rng = np.random.default_rng(seed)
    n_obj = int(n * 0.6); n_gnd = int(n * 0.15); n_bg = n - n_obj - n_gnd
    pts, nrm = _surface_points(rng, n_obj)
    m1, q1, s1, d1 = _surface_gaussians(rng, pts * 1.25, nrm, 0.0075, 5.0, 500.0, 0.0025)
    rho = np.sqrt(rng.uniform(1.5 ** 2, 15.0 ** 2, n_gnd))
    th = rng.uniform(0, 2 * np.pi, n_gnd)
    gp = np.stack([rho * np.cos(th), rho * np.sin(th), np.full(n_gnd, -1.0)], 1)
    gn = np.tile([0.0, 0.0, 1.0], (n_gnd, 1))
    m2, q2, s2, d2 = _surface_gaussians(rng, gp, gn, 0.01 * (1 + rho), 5.0, 500.0, 0.003)
    rad = rng.uniform(8.0, 40.0, n_bg)
    bd = _random_dirs(rng, n_bg)
    m3, q3, s3, d3 = _surface_gaussians(rng, bd * rad[:, None], -bd, 0.004 * rad, 5.0, 500.0, 0.01)
    s3[:, 2] = 0.3 * s3[:, 0]
    mean = np.concatenate([m1, m2, m3]); quat = np.concatenate([q1, q2, q3])
    scale = np.concatenate([s1, s2, s3]); density = np.concatenate([d1, d2, d3])
    sh, sg_amp, sg_sharp, sg_axis = _appearance(rng, n, sh_degree, sg_count)
    mean, quat, scale, density = _f32(mean, quat, scale, density)
    return Scene(mean, quat, scale, density, sh, sg_amp, sg_sharp, sg_axis, sh_degree, sg_count)


def scene_stress(seed=1004, n=5_000_000, sh_degree=3, sg_count=7):
    """C4: 5M heavily overlapping Gaussians in [-1,1]^3, s ~ LogU(0.07, 0.14)
    with anisotropy <= 2x, sigma ~ LogU(0.012, 0.05) (sigma_eps = 0.01).
    Oracle calibration (SURVEY §8(d) rule; tools/calibrate_c4.py) on 1,000 evenly
    spaced rays of the 1920x1080 view: mean per-slab set before truncation 982
    (96% of 2K; median 391), median termination depth 1.14 (>= 0.2); 31% of the
    rays do not terminate.  Scales +3% moved the mean only to 991 (denser supports
    also terminate rays earlier), so the recipe is kept."""
    rng = np.random.default_rng(seed)
    mean = rng.uniform(-1.0, 1.0, size=(n, 3))
    s0 = _loguniform(rng, 0.07, 0.14, n)
    scale = s0[:, None] * rng.uniform(0.5, 1.0, size=(n, 3))
    quat = _random_unit_quat(rng, n)
    density = _loguniform(rng, 0.012, 0.05, n)
    sh, sg_amp, sg_sharp, sg_axis = _appearance(rng, n, sh_degree, sg_count)
    mean, scale, density = _f32(mean, scale, density)
    return Scene(mean, quat, scale, density, sh, sg_amp, sg_sharp, sg_axis, sh_degree, sg_count)


# ----------------------------------------------------------------------------
# cameras
# ----------------------------------------------------------------------------

def look_at(eye, target=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0)):
    """c2w [right | down | forward | eye] (3x4, f32)."""
    eye = np.asarray(eye, np.float64)
    f = np.asarray(target, np.float64) - eye
    f /= np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, np.float64))
    if np.linalg.norm(r) < 1e-9:
        r = np.cross(f, np.array([0.0, 1.0, 0.0]))
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    return np.stack([r, d, f, eye], axis=1).astype(np.float32)


def orbit_camera(radius, azimuth_deg, elevation_deg, width, height, fx, fy=None,
                 target=(0.0, 0.0, 0.0), height_offset=0.0):
    az, el = math.radians(azimuth_deg), math.radians(elevation_deg)
    eye = (radius * math.cos(el) * math.cos(az), radius * math.cos(el) * math.sin(az),
           radius * math.sin(el) + height_offset)
    return Camera(width, height, float(fx), float(fy if fy is not None else fx),
                  width / 2.0, height / 2.0, look_at(eye, target))


def random_rays(seed, n, *, radius=2.5, jitter=0.6):
    """Explicit uncorrelated rays: origins on a sphere, directions
    towards random points near the centre, normalised in f32."""
    rng = np.random.default_rng(seed)
    o = _random_dirs(rng, n) * radius
    tgt = rng.uniform(-jitter, jitter, size=(n, 3))
    d = _unit(tgt - o)
    o = o.astype(np.float32)
    d = d.astype(np.float32)
    d = (d / np.linalg.norm(d.astype(np.float64), axis=1, keepdims=True)).astype(np.float32)
    return o, d


# ----------------------------------------------------------------------------
# the five workloads (BASELINE.json configs)
# ----------------------------------------------------------------------------

BLENDER_FX = 400.0 / math.tan(0.6911112070083618 / 2.0)   # camera_angle_x of NeRF-synthetic


def workload(name: str, *, n=None, views=None) -> Workload:
    if name == "tiny":
        sc = scene_tiny()
        cams = [orbit_camera(2.5, 30.0, 20.0, 64, 64, 87.92)]
        p = RenderParams(dt=5e-3, slab_samples=8, sigma_eps=0.1, t_eps=1e-4,
                         hit_capacity=512, background=(1.0, 1.0, 1.0))
        return Workload(name, sc, cams, p, "C0: 64 Gaussians, SH deg 0, 64x64, B=8")
    if name in ("blender", "blender_train"):
        sc = scene_blender(n=n or 300_000)
        nv = views or (1 if name == "blender" else 8)
        cams = [orbit_camera(4.0311, 45.0 * v + 15.0, 30.0, 800, 800, BLENDER_FX) for v in range(nv)]
        p = RenderParams(dt=2.5e-4, slab_samples=8, sigma_eps=0.1, t_eps=1e-4,
                         hit_capacity=512, background=(1.0, 1.0, 1.0))
        return Workload(name, sc, cams, p, "C1/C2: 300k Gaussians SH3+7SG, 800x800")
    if name == "mip":
        sc = scene_mip(n=n or 2_000_000)
        cams = [orbit_camera(3.0, 45.0 * v + 10.0, 0.0, 1245, 825, 1078.2, height_offset=0.6)
                for v in range(views or 1)]
        p = RenderParams(dt=2.5e-4, slab_samples=8, sigma_eps=0.01, t_eps=1e-4,
                         hit_capacity=512, background=(0.0, 0.0, 0.0), list_capacity=128)
        return Workload(name, sc, cams, p, "C3: 2M Gaussians unbounded, 1245x825")
    if name == "stress":
        sc = scene_stress(n=n or 5_000_000)
        cams = [orbit_camera(3.5, 20.0, 15.0, 1920, 1080, 960.0 / math.tan(math.radians(25.0)))]
        p = RenderParams(dt=2.5e-4, slab_samples=8, sigma_eps=0.01, t_eps=1e-4,
                         hit_capacity=512, background=(0.0, 0.0, 0.0), list_capacity=520)
        return Workload(name, sc, cams, p, "C4: 5M overlapping Gaussians, 1920x1080")
    raise KeyError(name)


WORKLOADS = ("tiny", "blender", "blender_train", "mip", "stress")
