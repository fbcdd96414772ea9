/*
 * rg.h -- C-ABI of the B200-native RayGauss hot path (arXiv 2408.03356):
 * differentiable volume ray casting of anisotropic 3D Gaussians, slab by slab
 * through a BVH (Alg. 1-2, Eq. 4, Eq. 10-16
 * P:163-237, supplementary P:500-564).  Implemented by libraygauss.so
 * (paper_2408_03356_b200/csrc, hand-written sm_100a CUDA).
 *
 * Conventions for every entry point
 *   - Pointers are DEVICE pointers owned by the caller unless stated "host".
 *   - Every call is asynchronous on `stream` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream).  The library never allocates, frees or
 *     synchronises; scratch memory is the caller's workspace.
 *   - Argument validation happens before anything is enqueued; on error nothing
 *     is launched and a status != RG_OK is returned.  A failed launch returns
 *     RG_ERR_CUDA (cudaGetLastError after the launch).
 *   - Data errors never fail a call: non-finite Gaussians are inactive; hit-buffer
 *     overflow is truncated deterministically (L7); both are counted
 *     in the optional device-side rg_stats.
 *   - Parameters are ACTIVATED values (activations live with the caller):
 *     unit quaternion (w,x,y,z), scale > 0, density sigma~ > 0, SG axes unit.
 *     The quaternion/axes are consumed as given (no internal normalisation) and
 *     gradients are w.r.t. exactly these tensors.
 *   - Layouts are row-major, caller (original) Gaussian order:
 *       mean [n,3], quat [n,4], scale [n,3], density [n],
 *       sh [n,(sh_degree+1)^2,3], sg_amp [n,sg_count,3], sg_sharp [n,sg_count],
 *       sg_axis [n,sg_count,3]; rays / images [R,3] row-major, R = ray count.
 *   - Thread safety: calls on different streams with different workspaces are
 *     independent; the only global state is the diagnostic launch counter and a
 *     mutex-guarded cache of instantiated CUDA graphs of rg_build_bvh (keyed by
 *     parameters, config, workspace and device; RG_NO_GRAPH=1 disables it).
 */
#ifndef RAYGAUSS_RG_H
#define RAYGAUSS_RG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RG_ABI_VERSION 1

typedef enum {
  RG_OK = 0,
  RG_ERR_INVALID_ARG = 1,
  RG_ERR_WORKSPACE_TOO_SMALL = 2,
  RG_ERR_CUDA = 3,
  RG_ERR_NOT_IMPLEMENTED = 4
} rg_status;

/* Scene parameters P = {(sigma~, c~, mu, q, s)}. */
typedef struct {
  int32_t n;          /* number of Gaussians, >= 0 */
  int32_t sh_degree;  /* L1 of Eq. 14, 0..3 */
  int32_t sg_count;   /* number of SG lobes (Eq. 15), 0..7 */
  int32_t pad_;
  const float *mean, *quat, *scale, *density;
  const float *sh, *sg_amp, *sg_sharp, *sg_axis;   /* sg_* may be NULL if sg_count == 0 */
} rg_gaussians;

/* Gradients w.r.t. the same tensors, same layouts.  ACCUMULATED (+=): the
   caller zeroes them.  Any pointer may be NULL to skip that group. */
typedef struct {
  float *mean, *quat, *scale, *density, *sh, *sg_amp, *sg_sharp, *sg_axis;
} rg_gaussian_grads;

typedef struct {
  float dt;              /* Delta t, world units along unit d > 0 */
  int32_t slab_samples;  /* B, samples per slab, 1..32 */
  float sigma_eps;       /* truncation threshold (Eq. 16) > 0 */
  float t_eps;           /* early-termination threshold, [0,1) */
  int32_t hit_capacity;  /* K = n_max of Alg. 1, 1..4096 */
  int32_t radius_mode;   /* 0: r = phi^-1(sigma_eps/sigma~); 1: r = k_sigma */
  float k_sigma;         /* support radius in radius_mode 1 (north star "3-sigma") */
  float t_near;          /* t0 = max(bbox entry, t_near) (L13), usually 0 */
  float background[3];   /* pixel = C + T_end * background (L12) */
  int32_t basis;         /* basis function phi (supplementary P:456-515, L33):
                            RG_BASIS_* below; non-Gaussian bases need radius_mode 0 and
                            slab_samples >= 5 (else RG_ERR_NOT_IMPLEMENTED) */
  int32_t list_capacity; /* forward kernel-variant hint, results identical either way:
                            0 = the 64-slot per-ray active list; 65..128 = a 128-slot list;
                            > 128 = a 520-slot list (hit_capacity < 520) that holds whole
                            truncated slab sets (K-saturated scenes such as C4); the larger
                            lists apply to the Gaussian basis with slab_samples >= 5 and
                            avoid re-querying the BVH for slab sets above 64 */
} rg_config;

enum { RG_BASIS_GAUSSIAN = 0, RG_BASIS_BUMP = 1, RG_BASIS_WENDLAND = 2,
       RG_BASIS_INV_MULTIQUADRIC = 3, RG_BASIS_INV_QUADRATIC = 4, RG_BASIS_MATERN_C0 = 5 };

/* Explicit, possibly uncorrelated rays: device [n,3] origins and
   unit directions. */
typedef struct {
  int32_t n, pad_;
  const float *origin, *dir;
} rg_rays;

/* Pinhole camera: one ray through each pixel centre of the
   rectangle [x0,x1) x [y0,y1); rays are numbered row-major inside the
   rectangle.  c2w is HOST data (passed by value to the kernel): 3x4 row-major
   [right | down | forward | eye].
   Interleaved tile sharding (rays are independent):
   tile > 0 cuts the rectangle into tile x tile squares numbered row-major
   (ragged squares at the right and bottom edges) and this call renders only
   the squares k with k % shards == shard.  Rays are then numbered
   i * tile^2 + ly * tile + lx for the i-th owned square and the pixel (lx, ly)
   inside it; slots of a ragged square outside the rectangle are rendered as
   misses (rgb = background, T = 1, replay = -1) and get no gradient.
   rg_camera_ray_count gives the number of ray slots. */
typedef struct {
  int32_t width, height, x0, y0, x1, y1;
  float fx, fy, cx, cy;
  float c2w[12];
  int32_t spp;           /* rays per pixel: 1 (the pixel centre) or 4 (RayGauss4x, P:775:
                            a 2x2 grid at offsets 1/4, 3/4; L29).  Rays are
                            numbered pixel * spp + (sx + 2 sy); rg_supersample_resolve /
                            rg_supersample_spread map between rays and pixels. */
  int32_t tile;          /* 0: the whole rectangle; else the square size (even, 2..256;
                            spp must be 1) of the interleaved tile sharding above */
  int32_t shard, shards; /* owned squares: k % shards == shard (0 <= shard < shards) */
  int32_t pad_;
} rg_camera;

/* Number of rays (ray slots) rg_render_forward / rg_camera_rays produce for cam
   (host; 0 for an invalid camera). */
int64_t rg_camera_ray_count(const rg_camera* cam);

/* BVH handle filled by rg_build_bvh: device pointers into the caller's
   workspace.  Valid until the workspace is reused or the parameters change
   (the paper rebuilds after every optimiser step). Read-only for callers. */
typedef struct {
  int32_t n, sh_degree, sg_count, app_stride;
  const void* geom;        /* [n] 64-B records, Morton order */
  const float* app;        /* [n, app_stride] appearance, Morton order */
  const void* nodes;       /* [n-1] 64-B internal nodes (child boxes, child ids, the
                              node's first and last leaf in Morton order) */
  const void* wide;        /* 32-wide collapse of the Karras tree (traversal structure):
                              896-B nodes, 6 SoA box planes + 32 child ids; id >= 0 a
                              wide node, 0x7FFFFFFF empty, < 0 a leaf range
                              ~((first << 3) | (count - 1)) of 1..8 consecutive
                              Morton-order Gaussians (so n < 2^28) */
  const int32_t* wide_info;/* device [4]: wide node count, -, -, rounds left unfinished */
  const float* leaf_box;   /* [n,6] padded AABBs, Morton order */
  const float* root_box;   /* [6] scene bbox = union of active AABBs */
  const uint32_t* codes;   /* [n] Morton codes, caller order */
  const uint32_t* sorted_codes; /* [n] */
  const uint32_t* order;   /* [n] order[pos] = caller index */
} rg_bvh;

/* Device-side counters, ACCUMULATED with atomics (caller zeroes). */
typedef struct {
  unsigned long long rays;           /* rays launched */
  unsigned long long rays_hit;       /* rays with t0 < t1 */
  unsigned long long slabs;          /* non-empty slabs integrated */
  unsigned long long pairs;          /* (ray, Gaussian) pair set-ups */
  unsigned long long evals;          /* (sample, Gaussian) contributions */
  unsigned long long samples;        /* composited samples (sigma > 0) */
  unsigned long long overflows;      /* slabs truncated to K */
  unsigned long long fetches;        /* BVH traversals */
  unsigned long long node_visits;    /* internal nodes visited */
  unsigned long long stack_overflows; /* restart-query stack overflows (subtrees dropped) */
  unsigned long long nonfinite_grads;
  unsigned long long restarts;       /* persistent-traversal restarts after a frontier or
                                        candidate overflow (exact: no key is lost) */
  unsigned long long pad_[4];
} rg_stats;

/* static string for a status code (host) */
const char* rg_status_string(rg_status s);
/* library build string (host) */
const char* rg_version(void);
/* diagnostic: kernels enqueued by this library since load (host; the only
   process-wide state, a relaxed atomic counter) */
unsigned long long rg_kernel_launches(void);

/* ---- BVH build -------------------------------- */
/* Workspace bytes for rg_build_bvh on n Gaussians with the given appearance
   sizes (0 for invalid sizes).  The workspace must be 256-B aligned. */
size_t rg_bvh_workspace_bytes(int32_t n, int32_t sh_degree, int32_t sg_count);

/* Preprocess (R(q), M = S^-1 R^T, support radius, padded tight AABB: P:176-183,
   P:529-558), 30-bit Morton codes of the means, stable CUB-free LSD radix sort,
   Karras hierarchy, bottom-up refit, 32-wide collapse with leaf ranges.
   Errors: RG_ERR_INVALID_ARG for NULL pointers, n < 0 or n >= 2^28, sh_degree
   not in 0..3, sg_count not in 0..7, bad config; RG_ERR_WORKSPACE_TOO_SMALL. */
rg_status rg_build_bvh(const rg_gaussians* g, const rg_config* cfg, void* ws, size_t ws_bytes,
                       rg_bvh* out, void* stream);

/* UpdateBVH by refit (the paper rebuilds after each
   optimiser step): recomputes every record, AABB and box for new
   parameter VALUES while keeping the topology (Morton order, Karras tree,
   32-wide collapse) of the rg_build_bvh call that filled `bvh` on this same
   workspace.  Rendering results are identical to a rebuild (traversal is exact
   against conservative boxes); only traversal efficiency degrades as the means
   drift from their Morton order, so callers rebuild periodically.  `bvh` keeps
   its pointers.  Errors: RG_ERR_INVALID_ARG as rg_build_bvh, or when n,
   sh_degree, sg_count or the workspace differ from the build's;
   RG_ERR_WORKSPACE_TOO_SMALL. */
rg_status rg_refit_bvh(const rg_gaussians* g, const rg_config* cfg, void* ws, size_t ws_bytes,
                       rg_bvh* bvh, void* stream);

/* ---- rays -------------------------------------------------------------- */
/* Writes the camera's rays (ARITH-7) to device o/d [R,3], R = rg_camera_ray_count
   (ray slots outside the rectangle of a tile-sharded camera get o = d = 0). */
rg_status rg_camera_rays(const rg_camera* cam, float* origin, float* dir, void* stream);

/* ---- forward (a6-a10) ---------------------------------------------------- */
/* Renders either `rays` or `cam` (exactly one non-NULL).  Outputs (device):
     rgb [R,3]  = C + T_end * background,
     T   [R]    = final transmittance,
     replay [R] = index of the slab after which the ray terminated early
                  (T <= t_eps), or -1; consumed by rg_render_backward.
   fetch_log: optional device buffer of log_bytes bytes (training), at least
   rg_fetch_log_bytes(R, 0): the forward records each ray's BVH query results
   and set-up pair data so that rg_render_backward can replay the march without
   traversing or re-evaluating colours.  A ray whose record does not fit is
   marked and recomputed by the backward (results are identical either way).
   stats: optional device rg_stats.  debug: if debug_records != NULL, the first
   debug_rays rays append up to debug_cap (slab, caller index) pairs per ray of
   their integrated per-slab hit sets (in order) to debug_records
   [debug_rays, debug_cap, 2] and their record count to debug_counts. */
rg_status rg_render_forward(const rg_gaussians* g, const rg_bvh* bvh, const rg_config* cfg,
                            const rg_rays* rays, const rg_camera* cam, float* rgb, float* T,
                            int32_t* replay, void* fetch_log, size_t log_bytes,
                            rg_stats* stats, int32_t debug_rays, int32_t debug_cap,
                            int32_t* debug_counts, int32_t* debug_records, void* stream);

/* Bytes of a fetch log for n_rays rays with room for pairs_per_ray set-up
   pairs per ray on average (pairs_per_ray <= 0: a default of 48) and, for the
   4-slab windows, 2 * pairs_per_ray stored per-sample sums per ray on average
   (the backward reloads them instead of re-evaluating; windows that do not fit
   are recomputed, results identical either way). */
size_t rg_fetch_log_bytes(int32_t n_rays, int32_t pairs_per_ray);

/* ---- backward (a11-a12) ------------------------------------------------- */
/* Workspace for rg_render_backward: the Morton-ordered gradient accumulator. */
size_t rg_backward_workspace_bytes(int32_t n, int32_t sh_degree, int32_t sg_count);

/* Exact gradient (a.e., decisions held fixed) of sum_r <d_rgb_r, rgb_r> w.r.t.
   the activated parameters, by replaying the forward (same rays/camera, same
   bvh and cfg, forward outputs rgb/T/replay and, if it was recorded, the same
   fetch_log / log_words).  Gradients are ACCUMULATED into
   `grads` (caller order).  Non-finite gradient values are counted in stats. */
rg_status rg_render_backward(const rg_gaussians* g, const rg_bvh* bvh, const rg_config* cfg,
                             const rg_rays* rays, const rg_camera* cam, const float* rgb,
                             const float* T, const int32_t* replay, const void* fetch_log,
                             size_t log_bytes, const float* d_rgb,
                             const rg_gaussian_grads* grads, rg_stats* stats, void* ws,
                             size_t ws_bytes, void* stream);

/* ---- training-step neighbours ---------------------- */
/* Mutable fp32 arrays in the rg_gaussians layouts (raw parameters, Adam moments,
   activated outputs). */
typedef rg_gaussian_grads rg_param_arrays;

/* learning-rate slots of rg_adam_config.lr */
enum { RG_LR_MEAN = 0, RG_LR_QUAT, RG_LR_SCALE, RG_LR_DENSITY, RG_LR_SH_DC, RG_LR_SH_REST,
       RG_LR_SG_AMP, RG_LR_SG_SHARP, RG_LR_SG_AXIS, RG_LR_COUNT };

typedef struct {
  int32_t n, sh_degree, sg_count;
  int32_t step;          /* t >= 1 of Kingma & Ba Alg. 1 (bias corrections 1 - beta^t) */
  float lr[RG_LR_COUNT]; /* this iteration's learning rates (schedules are the caller's) */
  float beta1, beta2, eps;   /* in [0,1), [0,1), > 0 */
  int32_t sh_active;     /* SH coefficients per channel being optimised, 1..(sh_degree+1)^2;
                            the rest are locked (colour unlock) */
  int32_t sg_active;     /* SG lobes being optimised, 0..sg_count */
} rg_adam_config;

/* One fused Adam step over every parameter group (Alg. 3 AdamOptim):
     g_raw = J_act^T grad_act (activations: scale = exp(raw), density = exp(raw),
             quat and sg_axis = raw/|raw|, identity otherwise -- DESIGN.md L23-L25);
     m = b1 m + (1-b1) g_raw;  v = b2 v + (1-b2) g_raw^2;
     raw -= lr * (m/(1-b1^t)) / (sqrt(v/(1-b2^t)) + eps)      (Kingma & Ba Alg. 1);
     act_out = act(raw) for every element (locked ones too).
   raw, m, v are updated in place; grad_act is read (the gradient w.r.t. the
   activated parameters, e.g. from rg_render_backward); act_out may alias the
   arrays of the rg_gaussians the next render reads.  Locked colour coefficients
   keep raw, m and v.  Errors: RG_ERR_INVALID_ARG for NULL arrays (sg_* may be
   NULL when sg_count == 0), bad sizes, step < 1, out-of-range betas/eps/active
   counts. */
rg_status rg_adam_step(const rg_adam_config* cfg, const rg_gaussian_grads* grad_act,
                       const rg_param_arrays* raw, const rg_param_arrays* m,
                       const rg_param_arrays* v, const rg_param_arrays* act_out, void* stream);

/* Workspace bytes of rg_l1_dssim_loss_grad for a width x height image (0 if invalid). */
size_t rg_dssim_workspace_bytes(int32_t width, int32_t height);

/* Training loss of the paper (3D Gaussian Splatting practice;
   DESIGN.md L26-L27) and its gradient, fused:
     L = (1 - lambda) mean|rgb - target| + lambda (1 - mean SSIM(rgb, target)),
   SSIM (Wang et al. 2004) per pixel and channel from 11x11 Gaussian-window
   (sigma 1.5) local moments with zero padding, C1 = 0.01^2, C2 = 0.03^2; means
   over all pixels and the 3 channels.  rgb, target: device [height, width, 3]
   row-major (rg_render_forward's camera-mode ray order); d_rgb (device, same
   shape) is WRITTEN with dL/drgb (sign(0) = 0 for the L1 term); *loss (device)
   is ACCUMULATED with L (may be NULL).  Errors: RG_ERR_INVALID_ARG for NULL
   images, width/height < 0, lambda outside [0,1]; RG_ERR_WORKSPACE_TOO_SMALL. */
rg_status rg_l1_dssim_loss_grad(const float* rgb, const float* target, int32_t width,
                                int32_t height, float lambda, float* d_rgb, float* loss, void* ws,
                                size_t ws_bytes, void* stream);

/* RayGauss4x pixel <-> ray maps for spp rays per pixel (device, [n_pixels*spp,3]
   rays, [n_pixels,3] pixels): resolve writes rgb_px = mean of the pixel's spp ray
   colours (box filter); spread writes d_rays = d_px / spp (its adjoint).  Errors:
   RG_ERR_INVALID_ARG for NULL pointers with n_pixels > 0, spp < 1. */
rg_status rg_supersample_resolve(const float* rgb_rays, int64_t n_pixels, int32_t spp,
                                 float* rgb_px, void* stream);
rg_status rg_supersample_spread(const float* d_px, int64_t n_pixels, int32_t spp, float* d_rays,
                                void* stream);

/* ---- adaptive density control (Alg. 3; L30-L32) -- */
/* Statistic: acc[i] += ||grad_mean[i]||, cnt[i] += (||grad_mean[i]|| > 0) (device, fp32 /
   int32, [n]); call once per iteration with the step's dL/dmu [n,3]. */
rg_status rg_densify_accumulate(const float* grad_mean, int32_t n, float* acc, int32_t* cnt,
                                void* stream);
/* Workspace bytes of rg_densify_plan / _apply for n Gaussians. */
size_t rg_densify_workspace_bytes(int32_t n);
/* Decisions (fp32): avg = acc/cnt (0 if cnt = 0); PRUNE if density < sigma_eps; else
   if avg >= grad_eps: CLONE if max(scale) <= percent_dense * extent, else SPLIT; else
   KEEP.  Writes action[i] (0 keep, 1 clone, 2 split, 3 prune), the output order into
   ws, and device counts[4] = {survivors (keep + clone originals), clones, splits,
   n_out = survivors + clones + 2 splits}.  Output order: survivors (index order),
   clones (index order), split children (parent order, child 0 then 1). */
rg_status rg_densify_plan(const rg_gaussians* g, const float* acc, const int32_t* cnt,
                          float grad_eps, float extent, float sigma_eps, float percent_dense,
                          int32_t* action, void* ws, size_t ws_bytes, int32_t* counts,
                          void* stream);
/* Writes the n_out output rows of one array set (device, caller layouts, out sized
   counts[3] rows).  mode 0: the activated parameters of `g` (in = NULL or g's
   arrays): split children get mean + R(q) (scale * z_k) and scale / 1.6;
   mode 1: raw optimiser parameters `in` (rg_adam_step's raw): split children get the
   same child mean and raw scale - ln 1.6; mode 2: Adam moments `in`: new rows
   (clones, children) are zero.  z: device [n, 2, 3] standard normal draws. */
rg_status rg_densify_apply(const rg_gaussians* g, const rg_param_arrays* in,
                           const int32_t* action, const void* ws, const int32_t* counts,
                           const float* z, int32_t mode, const rg_param_arrays* out, void* stream);

/* ---- loss helper (for benchmarks; loss itself is outside the paper's path) -- */
/* L1 loss: loss += scale * sum |rgb - target|, d_rgb = scale * sign(rgb - target)
   over n_values floats (device; loss is one device float, accumulated). */
rg_status rg_l1_loss_grad(const float* rgb, const float* target, int64_t n_values, float scale,
                          float* d_rgb, float* loss, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RAYGAUSS_RG_H */
