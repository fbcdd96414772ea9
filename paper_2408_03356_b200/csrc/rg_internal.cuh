// rg_internal.cuh -- device-side building blocks of libraygauss (sm_100a).
//
// The fp32 "decision" sequences below follow DESIGN.md ARITH-1..9 with every
// operation explicitly rounded (__f*_rn) so nvcc cannot contract or reorder
// them; they decide Morton codes, hit sets, sample positions and must agree
// bit for bit with the oracle, which implements the same contract on its own
// (oracle/rg_oracle.c; no code is shared).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rg.h"

// Device-side invariant checks (compute-sanitizer is closed on this GPU pool): a
// build with -DRG_CHECKS (RG_DEFINES=RG_CHECKS python paper_2408_03356_b200/build.py)
// traps on any shared-memory slot, stack, queue, log-word, arena or gradient-row
// index outside its buffer; the GPU test suite is run against that build.
#ifdef RG_CHECKS
#include <cstdio>
#define RG_CHECK(c)                                                                    \
  do {                                                                                 \
    if (!(c)) {                                                                        \
      printf("RG_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);                  \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define RG_CHECK(c) \
  do {              \
  } while (0)
#endif

namespace rg {

// ---------------------------------------------------------------------------
// constants / layouts
// ---------------------------------------------------------------------------
constexpr int kMaxDeg = 3;
constexpr int kMaxLobes = 7;
constexpr int kMaxApp = 3 * 16 + 7 * 7;          // 97 floats
constexpr int kStack = 64;                        // traversal stack entries
constexpr int kACap = 32;                         // active-list capacity per ray
constexpr int kGroup = 8;                         // samples per register group
constexpr float kLog2e = 1.4426950408889634f;

// appearance record: SH region fixed at 16 coefficients x 3 (zero past the
// degree) so that the SG lobes (7 floats each) always start at float 48
constexpr int kShFloats = 48;
__host__ __device__ inline int app_floats(int deg, int lobes) {
  (void)deg;
  return kShFloats + 7 * lobes;
}
__host__ __device__ inline int app_stride(int deg, int lobes) {
  return (app_floats(deg, lobes) + 3) & ~3;
}
// Morton-ordered gradient row (floats): [0..2] v = sum (Sw x' + Sw1 d), [3] dL/dsigma~,
// [4..9] the symmetric S = sum (Sw x'x'^T + Sw1 (x'd^T + dx'^T) + Sw2 dd^T) as
// (S00, S01, S02, S11, S12, S22) -- k_finalize forms dL/dmu = M^T M v and
// dL/dM = -M S -- [10..15] pad, then SH grads channel-major [3][ncp]
// (ncp = (deg+1)^2 rounded up to 4), then SG grads lobe-major [G][8]
// (k0,k1,k2,lambda | p0,p1,p2,-), so that every float4 of the appearance part
// is one SH channel x 4 coefficients or one half of one lobe.
__host__ __device__ inline int sh_pad(int deg) { return (((deg + 1) * (deg + 1)) + 3) & ~3; }
__host__ __device__ inline int grad_stride(int deg, int lobes) {
  return 16 + 3 * sh_pad(deg) + 8 * lobes;
}

// geometry record, 64 B, Morton order:
//  g0 = {mu.x, mu.y, mu.z, sigma~}   g1 = {M0, M1, M2, M3}
//  g2 = {M4, M5, M6, M7}             g3 = {M8, r2 (<0: inactive), idx bits, 0}
// node record, 64 B: n0 = {L.lo.xyz, L.hi.x} n1 = {L.hi.yz, R.lo.xy}
//                    n2 = {R.lo.z, R.hi.xyz} n3 = {left, right (int bits), first, last}
// child id >= 0: internal node, < 0: leaf ~pos; [first, last]: the node's leaf
// range in Morton order (Karras: its split gamma is left or ~left).

// 32-wide BVH node (collapse of the Karras tree, one child per warp lane):
// SoA child boxes and child ids; child >= 0: wide node, < 0: a leaf RANGE
// ~((first << 3) | (count - 1)) of 1..kLeafRange consecutive Morton-order
// Gaussians (a binary subtree of <= kLeafRange leaves is not made a wide node
// of its own: its leaves are queued for the exact test directly, and its box is
// the union of theirs), kWideEmpty: unused slot (its box is empty).
constexpr int kWide = 32;
constexpr int kWideEmpty = 0x7FFFFFFF;
// leaf ranges of up to RG_LEAF_RANGE Gaussians: measured (medians of 9, C1):
// R = 1 forward 6.33 / backward 4.83 ms, R = 2 6.80 / 5.33, R = 4 6.72 / 5.34,
// R = 8 9.52 / 5.58 -- R = 4 cuts node visits by 20% (C1) and 45% (C3) but the
// extra exact tests cost more (C3 forward +23%): single leaves by default
#ifndef RG_LEAF_RANGE
#define RG_LEAF_RANGE 1
#endif
constexpr int kLeafRange = RG_LEAF_RANGE;
static_assert(kLeafRange >= 1 && kLeafRange <= 8, "leaf ranges: 3-bit count");
constexpr int kMaxLeafPos = 1 << 28;   // n limit of the range encoding
__host__ __device__ __forceinline__ int leaf_range_enc(int first, int count) {
  return ~((first << 3) | (count - 1));
}
__host__ __device__ __forceinline__ int leaf_range_first(int child) {
  return (int)((unsigned)~child >> 3);
}
__host__ __device__ __forceinline__ int leaf_range_count(int child) { return (~child & 7) + 1; }
struct WideNode {
  float lox[kWide], loy[kWide], loz[kWide], hix[kWide], hiy[kWide], hiz[kWide];
  int child[kWide];
};
// Upper bound on the wide-node count of the greedy collapse: a wide node with
// fewer than 32 entries holds only single leaves (>= 2 of them: it was made
// for a subtree of > kLeafRange >= 1 leaves, or is the root), so there are at most
// n/2 such nodes; every other node has 32 entries, and entries = (W - 1) + n,
// which bounds the full ones by (n - 1 - W_partial)/31.  Hence
// W <= n/2 + (n/2)/31 + 1 (a balanced grid scene reaches 33825 of 33827 at
// n = 65536).
__host__ __device__ constexpr size_t wide_capacity(int n) {
  return (size_t)(n / 2 + n / 62 + 4);
}

struct SceneView {
  const float4* geom;
  const float* app;
  const float4* nodes;
  const WideNode* wide;
  const float* root_box;
  int n, deg, lobes, app_stride;
};

// ---------------------------------------------------------------------------
// exact fp32 helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float div_(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }
// (a0*b0 + a1*b1) + a2*b2, each op rounded
__device__ __forceinline__ float dot3_(float a0, float a1, float a2, float b0, float b1, float b2) {
  return add_(add_(mul_(a0, b0), mul_(a1, b1)), mul_(a2, b2));
}

__device__ __forceinline__ uint32_t fkey(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(b);
}

__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// ARITH-1: R(q), q = (w,x,y,z)
__device__ __forceinline__ void rot_exact(float w, float x, float y, float z, float R[9]) {
  const float xx = mul_(x, x), yy = mul_(y, y), zz = mul_(z, z);
  const float xy = mul_(x, y), xz = mul_(x, z), yz = mul_(y, z);
  const float wx = mul_(w, x), wy = mul_(w, y), wz = mul_(w, z);
  R[0] = sub_(1.0f, mul_(2.0f, add_(yy, zz)));
  R[1] = mul_(2.0f, sub_(xy, wz));
  R[2] = mul_(2.0f, add_(xz, wy));
  R[3] = mul_(2.0f, add_(xy, wz));
  R[4] = sub_(1.0f, mul_(2.0f, add_(xx, zz)));
  R[5] = mul_(2.0f, sub_(yz, wx));
  R[6] = mul_(2.0f, sub_(xz, wy));
  R[7] = mul_(2.0f, add_(yz, wx));
  R[8] = sub_(1.0f, mul_(2.0f, add_(xx, yy)));
}

// ARITH-5: support interval of the ray against the ellipsoid of a geometry
// record.  Returns false on miss.  Also returns d_l = M d and A = |d_l|^2.
struct PairGeom {
  float te, tx, tm, A;
  float dl0, dl1, dl2;
};
__device__ __forceinline__ bool isect_exact(const float4& g0, const float4& g1, const float4& g2,
                                            const float4& g3, const float3& o, const float3& d,
                                            PairGeom& pg) {
  const float r2 = g3.y;
  const float v0 = sub_(o.x, g0.x), v1 = sub_(o.y, g0.y), v2 = sub_(o.z, g0.z);
  const float ol0 = dot3_(g1.x, g1.y, g1.z, v0, v1, v2);
  const float ol1 = dot3_(g1.w, g2.x, g2.y, v0, v1, v2);
  const float ol2 = dot3_(g2.z, g2.w, g3.x, v0, v1, v2);
  const float dl0 = dot3_(g1.x, g1.y, g1.z, d.x, d.y, d.z);
  const float dl1 = dot3_(g1.w, g2.x, g2.y, d.x, d.y, d.z);
  const float dl2 = dot3_(g2.z, g2.w, g3.x, d.x, d.y, d.z);
  const float A = dot3_(dl0, dl1, dl2, dl0, dl1, dl2);
  const float B = dot3_(ol0, ol1, ol2, dl0, dl1, dl2);
  const float tm = -div_(B, A);
  const float u0 = add_(ol0, mul_(tm, dl0));
  const float u1 = add_(ol1, mul_(tm, dl1));
  const float u2 = add_(ol2, mul_(tm, dl2));
  const float qmin = dot3_(u0, u1, u2, u0, u1, u2);
  if (!(qmin <= r2)) return false;
  const float h = sqrt_(div_(sub_(r2, qmin), A));
  pg.te = sub_(tm, h);
  pg.tx = add_(tm, h);
  pg.tm = tm;
  pg.A = A;
  pg.dl0 = dl0; pg.dl1 = dl1; pg.dl2 = dl2;
  return true;
}

// Compensated x' = (o - mu) + tm * d (TwoSum / fma TwoProduct): the world
// offset of the ray point at t_mid from the Gaussian centre, accurate to a few
// ulp of |x'| although |o - mu| >> |x'|.  Value path only (never a decision).
__device__ __forceinline__ float two_sum_err(float a, float b, float s) {
  const float bb = sub_(s, a);
  return add_(sub_(a, sub_(s, bb)), sub_(b, bb));
}
__device__ __forceinline__ float offset_at(float o, float mu, float tm, float d) {
  const float v = sub_(o, mu);
  const float ve = two_sum_err(o, -mu, v);
  const float p = mul_(tm, d);
  const float pe = fma_(tm, d, -p);
  const float s = add_(v, p);
  const float se = two_sum_err(v, p, s);
  return add_(s, add_(se, add_(ve, pe)));
}

// ARITH-8: scene bbox clip
__device__ __forceinline__ bool clip_exact(const float* box, const float3& o, const float3& d,
                                           float t_near, float& t0, float& t1) {
  if (!(box[0] <= box[3]) || !(box[1] <= box[4]) || !(box[2] <= box[5])) return false;
  const float ix = div_(1.0f, d.x), iy = div_(1.0f, d.y), iz = div_(1.0f, d.z);
  const float ax = mul_(sub_(box[0], o.x), ix), bx = mul_(sub_(box[3], o.x), ix);
  const float ay = mul_(sub_(box[1], o.y), iy), by = mul_(sub_(box[4], o.y), iy);
  const float az = mul_(sub_(box[2], o.z), iz), bz = mul_(sub_(box[5], o.z), iz);
  t0 = fmaxf(fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fminf(az, bz)), t_near);
  t1 = fminf(fminf(fmaxf(ax, bx), fmaxf(ay, by)), fmaxf(az, bz));
  return t0 < t1;
}

// ARITH-7: pinhole ray through pixel centre
// subsample s of a pixel: the centre for spp = 1, the 2x2 grid at 1/4, 3/4 for spp = 4
__device__ __forceinline__ float sub_off(int spp, int s_axis) {
  return spp == 1 ? 0.5f : 0.25f + 0.5f * (float)s_axis;
}
__device__ __forceinline__ void camera_ray(const rg_camera& cam, int px, int py, float ox, float oy,
                                           float3& o, float3& d) {
  const float xc = div_(sub_(add_((float)px, ox), cam.cx), cam.fx);
  const float yc = div_(sub_(add_((float)py, oy), cam.cy), cam.fy);
  const float* M = cam.c2w;
  const float dw0 = add_(add_(mul_(M[0], xc), mul_(M[1], yc)), M[2]);
  const float dw1 = add_(add_(mul_(M[4], xc), mul_(M[5], yc)), M[6]);
  const float dw2 = add_(add_(mul_(M[8], xc), mul_(M[9], yc)), M[10]);
  const float nrm = sqrt_(dot3_(dw0, dw1, dw2, dw0, dw1, dw2));
  d = make_float3(div_(dw0, nrm), div_(dw1, nrm), div_(dw2, nrm));
  o = make_float3(M[3], M[7], M[11]);
}

// camera ray slots (rg.h): the rectangle x spp, or the owned squares x tile^2
__host__ __device__ inline int64_t camera_squares_x(const rg_camera& c) {
  return c.tile > 0 ? ((int64_t)(c.x1 - c.x0) + c.tile - 1) / c.tile : 0;
}
__host__ __device__ inline int64_t camera_owned_squares(const rg_camera& c) {
  if (c.tile <= 0) return 0;
  const int64_t nsq = camera_squares_x(c) * (((int64_t)(c.y1 - c.y0) + c.tile - 1) / c.tile);
  return c.shard < nsq ? (nsq - c.shard + c.shards - 1) / c.shards : 0;
}
__host__ __device__ inline int64_t camera_ray_slots(const rg_camera& c) {
  if (c.tile > 0) return camera_owned_squares(c) * c.tile * c.tile;
  return (int64_t)(c.x1 - c.x0) * (c.y1 - c.y0) * c.spp;
}
// tile-sharded slot -> pixel of the rectangle (false: outside, a miss)
__host__ __device__ inline bool camera_tile_pixel(const rg_camera& c, int64_t slot, int& px, int& py) {
  const int64_t t2 = (int64_t)c.tile * c.tile;
  const int64_t i = slot / t2, r = slot - i * t2;
  const int64_t k = c.shard + i * c.shards;
  const int64_t nsx = camera_squares_x(c);
  px = (int)((k % nsx) * c.tile + r % c.tile);
  py = (int)((k / nsx) * c.tile + r / c.tile);
  return px < c.x1 - c.x0 && py < c.y1 - c.y0;
}

// ARITH-9
__device__ __forceinline__ float sample_t(int k, float dt, float t0) {
  return fma_(add_((float)k, 0.5f), dt, t0);
}

// ---------------------------------------------------------------------------
// colour c_l(d) (Eq. 14-15): 3DGS real SH basis (L10) + SG lobes
// ---------------------------------------------------------------------------
__device__ __forceinline__ void sh_basis(int deg, float x, float y, float z, float Y[16]) {
  Y[0] = 0.28209479177387814f;
  if (deg < 1) return;
  Y[1] = -0.4886025119029199f * y;
  Y[2] = 0.4886025119029199f * z;
  Y[3] = -0.4886025119029199f * x;
  if (deg < 2) return;
  const float xx = x * x, yy = y * y, zz = z * z;
  Y[4] = 1.0925484305920792f * x * y;
  Y[5] = -1.0925484305920792f * y * z;
  Y[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
  Y[7] = -1.0925484305920792f * x * z;
  Y[8] = 0.5462742152960396f * (xx - yy);
  if (deg < 3) return;
  Y[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
  Y[10] = 2.890611442640554f * x * y * z;
  Y[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
  Y[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
  Y[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
  Y[14] = 1.445305721320277f * z * (xx - yy);
  Y[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
}

// ---------------------------------------------------------------------------
// host-side launchers (defined in the .cu files)
// ---------------------------------------------------------------------------
// fetch log (training): [0, 256) pair-arena counter (u64 @0) and sample-arena
// counter (u64 @8); then per-ray records of kLogWords int32 ([0] = fetch words
// used | stored windows << 16, or -1; then (count, arena entry offset) per fetch
// from the front and one window-slot index per stored 4-slab window from the
// back); then the arena of 48-B pair slots (3 float4 each: per-ray blocks of 32
// slots, then a shared overflow region bump-allocated through the counter); then the sample
// arena (one float4 (sigma, sigma c) per lane of a stored window).  Split of the
// space after the records: rest / 80 pair slots, the remainder float4 samples.
constexpr int kLogWords = 128;
__host__ __device__ inline size_t fetch_log_header_bytes(int n_rays) {
  return 256 + ((4 * (size_t)kLogWords * (size_t)(n_rays > 0 ? n_rays : 1) + 255) & ~(size_t)255);
}

struct BvhLayout {
  size_t geom, app, nodes, leaf_box, root_box, codes, keys_a, keys_b, vals_a, vals_b,
      box_orig, flags, parent_int, parent_leaf, refit_cnt, bounds, hist, wide, wq_a, wide_src,
      wcounts, total;
  int tiles;
};
BvhLayout bvh_layout(int n, int deg, int lobes);
cudaError_t launch_build(const rg_gaussians& g, const rg_config& c, char* ws, const BvhLayout& L,
                         cudaStream_t st);
cudaError_t launch_refit(const rg_gaussians& g, const rg_config& c, char* ws, const BvhLayout& L,
                         cudaStream_t st);
cudaError_t launch_adam(const rg_adam_config& c, const rg_gaussian_grads& g,
                        const rg_gaussian_grads& raw, const rg_gaussian_grads& m,
                        const rg_gaussian_grads& v, const rg_gaussian_grads& act, cudaStream_t st);
size_t dssim_workspace_bytes(int H, int W);
cudaError_t launch_l1_dssim(const float* x, const float* y, int H, int W, float lam, float* d,
                            float* loss, float* ws, cudaStream_t st);
cudaError_t launch_ss_resolve(const float* r, int64_t n, int spp, float* px, cudaStream_t st);
cudaError_t launch_ss_spread(const float* dpx, int64_t n, int spp, float* dr, cudaStream_t st);
size_t densify_workspace_bytes(int n);
cudaError_t launch_dens_acc(const float* g, int n, float* acc, int* cnt, cudaStream_t st);
cudaError_t launch_dens_plan(const rg_gaussians& g, const float* acc, const int* cnt, float grad_eps,
                             float extent, float sigma_eps, float percent_dense, int* action,
                             char* ws, int* counts, cudaStream_t st);
cudaError_t launch_dens_apply(const rg_gaussians& g, const rg_gaussian_grads& in,
                              const rg_gaussian_grads& out, const int* action, const char* ws,
                              const int* counts, const float* z, int mode, cudaStream_t st);
cudaError_t launch_camera_rays(const rg_camera& cam, float* o, float* d, cudaStream_t st);
cudaError_t launch_forward(const rg_gaussians& g, const rg_bvh& b, const rg_config& c,
                           const rg_rays* rays, const rg_camera* cam, float* rgb, float* T,
                           int32_t* replay, void* log, size_t log_bytes, rg_stats* stats,
                           int dbg_rays, int dbg_cap,
                           int32_t* dbg_counts, int32_t* dbg_rec, cudaStream_t st);
cudaError_t launch_backward(const rg_gaussians& g, const rg_bvh& b, const rg_config& c,
                            const rg_rays* rays, const rg_camera* cam, const float* rgb,
                            const float* T, const int32_t* replay, const void* log,
                            size_t log_bytes, const float* d_rgb,
                            const rg_gaussian_grads& grads, rg_stats* stats, float* gbuf,
                            cudaStream_t st);
void count_launches(unsigned n);
cudaError_t launch_l1(const float* rgb, const float* target, int64_t n, float scale, float* d_rgb,
                      float* loss, cudaStream_t st);

}  // namespace rg
