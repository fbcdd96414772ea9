// Training-step neighbours of the hot path.
//
// k_adam: ONE launch updates every parameter group of Alg. 3's AdamOptim
// -- chain rule from the gradient w.r.t. the activated parameters (what
// rg_render_backward produces) to the raw ones, the Adam update of Kingma &
// Ba Alg. 1 (cited at P:639) with the per-group learning rates of P:642 and
// the colour unlock of P:644 (locked coefficients are not touched), and the
// activated parameters the next render consumes.  HBM-streaming: per element
// read raw, m, v, grad (16 B) and write raw, m, v, activated (16 B).
// Activations (L23-L25, the paper is silent): scale = exp(raw),
// density = exp(raw), quaternion / lobe axis = raw / |raw|, identity otherwise.
#include "rg_internal.cuh"

namespace rg {

namespace {

struct AdamArgs {
  int64_t n;
  int nc, G, sh_active, sg_active;
  float lr[9];
  float b1, b2, eps, bc1, bc2;
  rg_gaussian_grads g, raw, m, v, act;
  int64_t seg[9];   // cumulative item counts of the 8 segments
};

__device__ __forceinline__ float adam1(float th, float& m, float& v, float g, float lr,
                                       const AdamArgs& A) {
  m = A.b1 * m + (1.0f - A.b1) * g;
  v = A.b2 * v + (1.0f - A.b2) * (g * g);
  const float mh = m / A.bc1, vh = v / A.bc2;
  return th - lr * mh / (sqrtf(vh) + A.eps);
}

// element-wise groups with identity or exp activation
template <bool EXP, typename I>
__device__ __forceinline__ void step_elem(float* raw, float* m, float* v, const float* g, float* act,
                                          I i, float lr, const AdamArgs& A) {
  const float r = raw[i];
  float gi = g[i];
  if (EXP) gi *= expf(r);                      // d exp(r)/dr = exp(r)
  float mi = m[i], vi = v[i];
  const float r2 = adam1(r, mi, vi, gi, lr, A);
  raw[i] = r2; m[i] = mi; v[i] = vi;
  act[i] = EXP ? expf(r2) : r2;
}

template <int D, typename I>
__device__ __forceinline__ void step_unit(float* raw, float* m, float* v, const float* g, float* act,
                                          I i, float lr, bool live, const AdamArgs& A) {
  float r[D], gr[D];
  float nn = 0.f, ug = 0.f;
#pragma unroll
  for (int k = 0; k < D; ++k) { r[k] = raw[D * i + k]; nn += r[k] * r[k]; }
  const float nr = sqrtf(nn);
#pragma unroll
  for (int k = 0; k < D; ++k) { gr[k] = g[D * i + k]; ug += (r[k] / nr) * gr[k]; }
  float r2[D], n2 = 0.f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    if (live) {
      const float gk = (gr[k] - (r[k] / nr) * ug) / nr;   // (I - u u^T) g / |r|
      float mk = m[D * i + k], vk = v[D * i + k];
      r2[k] = adam1(r[k], mk, vk, gk, lr, A);
      m[D * i + k] = mk; v[D * i + k] = vk;
      raw[D * i + k] = r2[k];
    } else {
      r2[k] = r[k];
    }
    n2 += r2[k] * r2[k];
  }
  const float inv = sqrtf(n2);
#pragma unroll
  for (int k = 0; k < D; ++k) act[D * i + k] = r2[k] / inv;
}

// 32-bit item indices (the launcher falls back to the 64-bit instantiation
// above 2^31 items): the segment decode is then a few compares and 32-bit
// divisions by small constants
template <typename I>
__global__ void __launch_bounds__(256, 8) k_adam(const AdamArgs A) {
  const I total = (I)A.seg[8];
  const I s1 = (I)A.seg[1], s2 = (I)A.seg[2], s3 = (I)A.seg[3], s4 = (I)A.seg[4], s5 = (I)A.seg[5],
          s6 = (I)A.seg[6], s7 = (I)A.seg[7];
  const I nc = (I)A.nc, G = (I)(A.G > 0 ? A.G : 1);
  for (I t = blockIdx.x * (I)blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
    if (t < s1) {                                         // mean [n,3]
      step_elem<false>(A.raw.mean, A.m.mean, A.v.mean, A.g.mean, A.act.mean, t, A.lr[0], A);
    } else if (t < s2) {                                  // quat [n,4] as units
      step_unit<4>(A.raw.quat, A.m.quat, A.v.quat, A.g.quat, A.act.quat, t - s1, A.lr[1], true, A);
    } else if (t < s3) {                                  // scale [n,3]
      step_elem<true>(A.raw.scale, A.m.scale, A.v.scale, A.g.scale, A.act.scale, t - s2, A.lr[2], A);
    } else if (t < s4) {                                  // density [n]
      step_elem<true>(A.raw.density, A.m.density, A.v.density, A.g.density, A.act.density, t - s3,
                      A.lr[3], A);
    } else if (t < s5) {                                  // sh [n,nc,3]
      const I i = t - s4;
      const I c = (i / 3) % nc;
      if (c < (I)A.sh_active)
        step_elem<false>(A.raw.sh, A.m.sh, A.v.sh, A.g.sh, A.act.sh, i, c == 0 ? A.lr[4] : A.lr[5], A);
      else
        A.act.sh[i] = A.raw.sh[i];
    } else if (t < s6) {                                  // sg_amp [n,G,3]
      const I i = t - s5;
      if ((i / 3) % G < (I)A.sg_active)
        step_elem<false>(A.raw.sg_amp, A.m.sg_amp, A.v.sg_amp, A.g.sg_amp, A.act.sg_amp, i, A.lr[6], A);
      else
        A.act.sg_amp[i] = A.raw.sg_amp[i];
    } else if (t < s7) {                                  // sg_sharp [n,G]
      const I i = t - s6;
      if (i % G < (I)A.sg_active)
        step_elem<false>(A.raw.sg_sharp, A.m.sg_sharp, A.v.sg_sharp, A.g.sg_sharp, A.act.sg_sharp, i,
                         A.lr[7], A);
      else
        A.act.sg_sharp[i] = A.raw.sg_sharp[i];
    } else {                                              // sg_axis [n,G,3] as units
      const I i = t - s7;
      step_unit<3>(A.raw.sg_axis, A.m.sg_axis, A.v.sg_axis, A.g.sg_axis, A.act.sg_axis, i, A.lr[8],
                   i % G < (I)A.sg_active, A);
    }
  }
}

}  // namespace

cudaError_t launch_adam(const rg_adam_config& c, const rg_gaussian_grads& g,
                        const rg_gaussian_grads& raw, const rg_gaussian_grads& m,
                        const rg_gaussian_grads& v, const rg_gaussian_grads& act, cudaStream_t st) {
  AdamArgs A{};
  A.n = c.n;
  A.nc = (c.sh_degree + 1) * (c.sh_degree + 1);
  A.G = c.sg_count;
  A.sh_active = c.sh_active;
  A.sg_active = c.sg_active;
  for (int k = 0; k < 9; ++k) A.lr[k] = c.lr[k];
  A.b1 = c.beta1; A.b2 = c.beta2; A.eps = c.eps;
  A.bc1 = (float)(1.0 - pow((double)c.beta1, (double)c.step));
  A.bc2 = (float)(1.0 - pow((double)c.beta2, (double)c.step));
  A.g = g; A.raw = raw; A.m = m; A.v = v; A.act = act;
  const int64_t n = c.n;
  const int64_t cnt[8] = {3 * n, n, 3 * n, n, 3 * A.nc * n, 3 * A.G * n, A.G * n, A.G * n};
  A.seg[0] = 0;
  for (int k = 0; k < 8; ++k) A.seg[k + 1] = A.seg[k] + cnt[k];
  if (A.seg[8] == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (A.seg[8] + 255) / 256;
  const int blocks = (int)(want < (int64_t)sms * 16 ? want : (int64_t)sms * 16);
  if (A.seg[8] < ((int64_t)1 << 31)) k_adam<uint32_t><<<blocks, 256, 0, st>>>(A);
  else k_adam<int64_t><<<blocks, 256, 0, st>>>(A);
  count_launches(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Fused L1 + D-SSIM loss gradient (3DGS practice; L26-L27):
//   L = (1 - lam) mean|x - y| + lam (1 - mean SSIM(x, y)),
// SSIM per pixel and channel from 11x11 Gaussian-window moments (sigma 1.5,
// zero padding).  Two tiled passes over 16x16 pixel tiles:
//   k_dssim_moments: separable filter of (x, y, x^2, y^2, xy) -> S and the
//     partials G1 = dS/dmu_x, G2 = dS/dE[x^2], G3 = dS/dE[xy] per pixel
//     (workspace, 9 planes), block sums of S and |x - y| -> loss;
//   k_dssim_grad: adjoint filter of (G1, G2, G3) and
//     dL/dx = (1-lam) sign(x-y)/N - lam/N (wG1 + 2 x wG2 + y wG3),  N = 3 H W.
// ---------------------------------------------------------------------------
namespace {

constexpr int kT = 16, kHalo = 5, kE = kT + 2 * kHalo;   // tile, halo, extended tile
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

struct SsimArgs {
  const float* x;
  const float* y;
  float* d;
  float* loss;
  float* gmap;     // [9][H*W]: (channel, G1..G3) planes
  int H, W;
  float lam, invN;
  float w[11];
};

__global__ void __launch_bounds__(256) k_dssim_moments(const SsimArgs A) {
  __shared__ float sx[kE][kE], sy[kE][kE];
  __shared__ float hs[5][kE][kT];
  __shared__ float red[2][8];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int X0 = blockIdx.x * kT, Y0 = blockIdx.y * kT;
  const int px = X0 + tx, py = Y0 + ty;
  const bool in = px < A.W && py < A.H;
  float s_sum = 0.f, l1_sum = 0.f;
  for (int c = 0; c < 3; ++c) {
    __syncthreads();
    for (int k = threadIdx.x; k < kE * kE; k += 256) {
      const int ex = k % kE, ey = k / kE;
      const int gx = X0 - kHalo + ex, gy = Y0 - kHalo + ey;
      const bool ok = gx >= 0 && gx < A.W && gy >= 0 && gy < A.H;
      const size_t gi = 3 * ((size_t)gy * A.W + gx) + c;
      sx[ey][ex] = ok ? A.x[gi] : 0.f;
      sy[ey][ex] = ok ? A.y[gi] : 0.f;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kE * kT; k += 256) {      // horizontal pass
      const int ox = k % kT, ey = k / kT;
      float a = 0.f, b = 0.f, aa = 0.f, bb = 0.f, ab = 0.f;
#pragma unroll
      for (int t = 0; t < 11; ++t) {
        const float u = sx[ey][ox + t], v = sy[ey][ox + t], w = A.w[t];
        a = fmaf(w, u, a); b = fmaf(w, v, b);
        aa = fmaf(w, u * u, aa); bb = fmaf(w, v * v, bb); ab = fmaf(w, u * v, ab);
      }
      hs[0][ey][ox] = a; hs[1][ey][ox] = b; hs[2][ey][ox] = aa; hs[3][ey][ox] = bb; hs[4][ey][ox] = ab;
    }
    __syncthreads();
    float mx = 0.f, my = 0.f, exx = 0.f, eyy = 0.f, exy = 0.f;   // vertical pass
#pragma unroll
    for (int t = 0; t < 11; ++t) {
      const float w = A.w[t];
      mx = fmaf(w, hs[0][ty + t][tx], mx); my = fmaf(w, hs[1][ty + t][tx], my);
      exx = fmaf(w, hs[2][ty + t][tx], exx); eyy = fmaf(w, hs[3][ty + t][tx], eyy);
      exy = fmaf(w, hs[4][ty + t][tx], exy);
    }
    if (in) {
      const float sxx = exx - mx * mx, syy = eyy - my * my, sxy = exy - mx * my;
      const float N1 = 2.f * mx * my + kC1, N2 = 2.f * sxy + kC2;
      const float D1 = mx * mx + my * my + kC1, D2 = sxx + syy + kC2;
      const float D = D1 * D2;
      const float S = N1 * N2 / D;
      const size_t p = (size_t)py * A.W + px, HW = (size_t)A.H * A.W;
      A.gmap[(3 * c + 0) * HW + p] = (2.f * my * (N2 - N1) - 2.f * mx * S * (D2 - D1)) / D;
      A.gmap[(3 * c + 1) * HW + p] = -S / D2;
      A.gmap[(3 * c + 2) * HW + p] = 2.f * N1 / D;
      s_sum += S;
      l1_sum += fabsf(sx[ty + kHalo][tx + kHalo] - sy[ty + kHalo][tx + kHalo]);
    }
  }
  // block sums -> loss += (1-lam) L1/N - lam S/N  (+ lam once)
  for (int o = 16; o > 0; o >>= 1) {
    s_sum += __shfl_xor_sync(0xffffffffu, s_sum, o);
    l1_sum += __shfl_xor_sync(0xffffffffu, l1_sum, o);
  }
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = s_sum; red[1][threadIdx.x >> 5] = l1_sum; }
  __syncthreads();
  if (threadIdx.x == 0 && A.loss) {
    float s = 0.f, l = 0.f;
    for (int k = 0; k < 8; ++k) { s += red[0][k]; l += red[1][k]; }
    float v = ((1.f - A.lam) * l - A.lam * s) * A.invN;
    if (blockIdx.x == 0 && blockIdx.y == 0) v += A.lam;
    atomicAdd(A.loss, v);
  }
}

__global__ void __launch_bounds__(256) k_dssim_grad(const SsimArgs A) {
  __shared__ float sg[3][kE][kE];
  __shared__ float hs[3][kE][kT];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int X0 = blockIdx.x * kT, Y0 = blockIdx.y * kT;
  const int px = X0 + tx, py = Y0 + ty;
  const bool in = px < A.W && py < A.H;
  const size_t HW = (size_t)A.H * A.W;
  for (int c = 0; c < 3; ++c) {
    __syncthreads();
    for (int k = threadIdx.x; k < kE * kE; k += 256) {
      const int ex = k % kE, ey = k / kE;
      const int gx = X0 - kHalo + ex, gy = Y0 - kHalo + ey;
      const bool ok = gx >= 0 && gx < A.W && gy >= 0 && gy < A.H;
      const size_t p = (size_t)gy * A.W + gx;
#pragma unroll
      for (int j = 0; j < 3; ++j) sg[j][ey][ex] = ok ? A.gmap[(3 * c + j) * HW + p] : 0.f;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kE * kT; k += 256) {
      const int ox = k % kT, ey = k / kT;
      float a = 0.f, b = 0.f, e = 0.f;
#pragma unroll
      for (int t = 0; t < 11; ++t) {
        const float w = A.w[t];
        a = fmaf(w, sg[0][ey][ox + t], a); b = fmaf(w, sg[1][ey][ox + t], b);
        e = fmaf(w, sg[2][ey][ox + t], e);
      }
      hs[0][ey][ox] = a; hs[1][ey][ox] = b; hs[2][ey][ox] = e;
    }
    __syncthreads();
    float a = 0.f, b = 0.f, e = 0.f;
#pragma unroll
    for (int t = 0; t < 11; ++t) {
      const float w = A.w[t];
      a = fmaf(w, hs[0][ty + t][tx], a); b = fmaf(w, hs[1][ty + t][tx], b);
      e = fmaf(w, hs[2][ty + t][tx], e);
    }
    if (in) {
      const size_t gi = 3 * ((size_t)py * A.W + px) + c;
      const float x = A.x[gi], y = A.y[gi];
      const float sgn = x > y ? 1.f : (x < y ? -1.f : 0.f);
      A.d[gi] = ((1.f - A.lam) * sgn - A.lam * (a + 2.f * x * b + y * e)) * A.invN;
    }
  }
}

}  // namespace

size_t dssim_workspace_bytes(int H, int W) { return sizeof(float) * 9 * (size_t)H * (size_t)W; }

cudaError_t launch_l1_dssim(const float* x, const float* y, int H, int W, float lam, float* d,
                            float* loss, float* ws, cudaStream_t st) {
  if ((size_t)H * W == 0) return cudaSuccess;
  SsimArgs A{};
  A.x = x; A.y = y; A.d = d; A.loss = loss; A.gmap = ws;
  A.H = H; A.W = W; A.lam = lam;
  A.invN = (float)(1.0 / (3.0 * (double)H * (double)W));
  double g[11], s = 0.0;
  for (int k = 0; k < 11; ++k) { g[k] = exp(-((k - 5) * (k - 5)) / (2.0 * 1.5 * 1.5)); s += g[k]; }
  for (int k = 0; k < 11; ++k) A.w[k] = (float)(g[k] / s);
  const dim3 grid((W + kT - 1) / kT, (H + kT - 1) / kT);
  k_dssim_moments<<<grid, 256, 0, st>>>(A);
  k_dssim_grad<<<grid, 256, 0, st>>>(A);
  count_launches(2);
  return cudaGetLastError();
}

// RayGauss4x pixel <-> ray maps: resolve = box-filter mean of a pixel's spp
// rays, spread = its adjoint (d_ray = d_px / spp)
namespace {
__global__ void k_ss_resolve(const float* r, int64_t n, int spp, float* px) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // (pixel, channel)
  if (i >= 3 * n) return;
  const int64_t p = i / 3, c = i - 3 * p;
  float s = 0.f;
  for (int k = 0; k < spp; ++k) s += r[3 * (p * spp + k) + c];
  px[i] = s / (float)spp;
}
__global__ void k_ss_spread(const float* dpx, int64_t n, int spp, float* dr) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // (ray, channel)
  if (i >= 3 * n * spp) return;
  const int64_t ray = i / 3, c = i - 3 * ray;
  dr[i] = dpx[3 * (ray / spp) + c] / (float)spp;
}
}  // namespace

cudaError_t launch_ss_resolve(const float* r, int64_t n, int spp, float* px, cudaStream_t st) {
  if (n > 0) {
    k_ss_resolve<<<(unsigned)((3 * n + 255) / 256), 256, 0, st>>>(r, n, spp, px);
    count_launches(1);
  }
  return cudaGetLastError();
}
cudaError_t launch_ss_spread(const float* dpx, int64_t n, int spp, float* dr, cudaStream_t st) {
  if (n > 0) {
    k_ss_spread<<<(unsigned)((3 * n * spp + 255) / 256), 256, 0, st>>>(dpx, n, spp, dr);
    count_launches(1);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Adaptive density control (Alg. 3; readings L30-L32):
//   k_dens_acc:   acc += ||dL/dmu||, cnt += (||dL/dmu|| > 0) per Gaussian (fp32);
//   k_dens_plan:  action 0 keep / 1 clone / 2 split / 3 prune (fp32 decisions) and the
//                 three output-order flags, block-scanned;  k_dens_scan: block totals;
//   k_dens_apply: per input Gaussian, write its output rows (survivors in index
//                 order, then clones, then 2 split children per split parent).
// ---------------------------------------------------------------------------
namespace {

constexpr int kDensT = 256;

__global__ void k_dens_acc(const float* g, int n, float* acc, int* cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float x = g[3 * i], y = g[3 * i + 1], z = g[3 * i + 2];
  const float nrm = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y)), __fmul_rn(z, z)));
  acc[i] = __fadd_rn(acc[i], nrm);
  cnt[i] += nrm > 0.f ? 1 : 0;
}

// action + inclusive block scans of (survivor, clone, split) flags; block totals
__global__ void __launch_bounds__(kDensT) k_dens_plan(rg_gaussians g, const float* acc, const int* cnt,
                                                      float grad_eps, float small_lim, float sigma_eps,
                                                      int* action, int4* scan, int4* block_tot) {
  __shared__ int3 sh[kDensT];
  const int i = blockIdx.x * kDensT + threadIdx.x;
  int3 f = make_int3(0, 0, 0);
  if (i < g.n) {
    const float avg = cnt[i] > 0 ? __fdiv_rn(acc[i], (float)cnt[i]) : 0.f;
    const bool dens = avg >= grad_eps;
    const float* sc = g.scale + 3 * (size_t)i;
    const bool small = fmaxf(fmaxf(sc[0], sc[1]), sc[2]) <= small_lim;
    const bool prune = g.density[i] < sigma_eps;
    const int a = prune ? 3 : (dens ? (small ? 1 : 2) : 0);
    action[i] = a;
    f = make_int3(a <= 1 ? 1 : 0, a == 1 ? 1 : 0, a == 2 ? 1 : 0);
  }
  sh[threadIdx.x] = f;
  __syncthreads();
  for (int off = 1; off < kDensT; off <<= 1) {        // Hillis-Steele inclusive scan
    int3 v = make_int3(0, 0, 0);
    if ((int)threadIdx.x >= off) v = sh[threadIdx.x - off];
    __syncthreads();
    sh[threadIdx.x].x += v.x; sh[threadIdx.x].y += v.y; sh[threadIdx.x].z += v.z;
    __syncthreads();
  }
  if (i < g.n) {
    const int3 v = sh[threadIdx.x];
    scan[i] = make_int4(v.x - f.x, v.y - f.y, v.z - f.z, 0);   // exclusive within the block
  }
  if (threadIdx.x == kDensT - 1) {
    const int3 v = sh[kDensT - 1];
    block_tot[blockIdx.x] = make_int4(v.x, v.y, v.z, 0);
  }
}

// exclusive scan of the block totals (one block, looping) and the grand totals
__global__ void k_dens_scan(int4* block_tot, int nb, int* counts) {
  __shared__ int3 carry;
  if (threadIdx.x == 0) carry = make_int3(0, 0, 0);
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int k = base + threadIdx.x;
    int4 v = k < nb ? block_tot[k] : make_int4(0, 0, 0, 0);
    // warp-level inclusive scans then across warps via shared memory
    __shared__ int3 wsum[32];
    int3 x = make_int3(v.x, v.y, v.z);
    for (int o = 1; o < 32; o <<= 1) {
      const int ax = __shfl_up_sync(0xffffffffu, x.x, o), ay = __shfl_up_sync(0xffffffffu, x.y, o),
                az = __shfl_up_sync(0xffffffffu, x.z, o);
      if ((threadIdx.x & 31) >= o) { x.x += ax; x.y += ay; x.z += az; }
    }
    if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      int3 w = wsum[threadIdx.x];
      for (int o = 1; o < 32; o <<= 1) {
        const int ax = __shfl_up_sync(0xffffffffu, w.x, o), ay = __shfl_up_sync(0xffffffffu, w.y, o),
                  az = __shfl_up_sync(0xffffffffu, w.z, o);
        if (threadIdx.x >= (unsigned)o) { w.x += ax; w.y += ay; w.z += az; }
      }
      wsum[threadIdx.x] = w;
    }
    __syncthreads();
    const int3 wp = (threadIdx.x >> 5) ? wsum[(threadIdx.x >> 5) - 1] : make_int3(0, 0, 0);
    const int3 c = carry;
    if (k < nb)
      block_tot[k] = make_int4(c.x + wp.x + x.x - v.x, c.y + wp.y + x.y - v.y, c.z + wp.z + x.z - v.z, 0);
    __syncthreads();
    if (threadIdx.x == 0) {
      const int3 t = wsum[31];
      carry = make_int3(c.x + t.x, c.y + t.y, c.z + t.z);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    counts[0] = carry.x; counts[1] = carry.y; counts[2] = carry.z;
    counts[3] = carry.x + carry.y + 2 * carry.z;      // output Gaussians
  }
}

struct DensArgs {
  rg_gaussians g;          // activated input (geometry of the split)
  rg_gaussian_grads in;    // rows to move (mode 0: the activated arrays themselves)
  rg_gaussian_grads out;
  const int* action;
  const int4* scan;
  const int4* block_tot;
  const int* counts;
  const float* z;          // [n, 2, 3] standard normal draws
  int nc, G, mode;         // 0 activated, 1 raw optimiser parameters, 2 moments (new rows zero)
};

__device__ __forceinline__ void copy_row(const float* a, float* b, int64_t src, int64_t dst, int w,
                                         bool zero) {
  for (int k = 0; k < w; ++k) b[dst * w + k] = zero ? 0.f : a[src * w + k];
}

__global__ void __launch_bounds__(kDensT) k_dens_apply(const DensArgs A) {
  const int i = blockIdx.x * kDensT + threadIdx.x;
  if (i >= A.g.n) return;
  const int a = A.action[i];
  if (a == 3) return;
  const int4 sc = A.scan[i], bt = A.block_tot[blockIdx.x];
  const int nkeep = A.counts[0], nclone = A.counts[1];
  const int w[8] = {3, 4, 3, 1, 3 * A.nc, 3 * A.G, A.G, 3 * A.G};
  const float* src[8] = {A.in.mean, A.in.quat, A.in.scale, A.in.density, A.in.sh, A.in.sg_amp,
                         A.in.sg_sharp, A.in.sg_axis};
  float* dst[8] = {A.out.mean, A.out.quat, A.out.scale, A.out.density, A.out.sh, A.out.sg_amp,
                   A.out.sg_sharp, A.out.sg_axis};
  if (a <= 1) {                                       // survivor (original row)
    const int64_t o = sc.x + bt.x;
    for (int k = 0; k < 8; ++k)
      if (w[k]) copy_row(src[k], dst[k], i, o, w[k], false);
  }
  if (a == 1) {                                       // clone: a copy after the survivors
    const int64_t o = nkeep + sc.y + bt.y;
    for (int k = 0; k < 8; ++k)
      if (w[k]) copy_row(src[k], dst[k], i, o, w[k], A.mode == 2);
  }
  if (a == 2) {                                       // split: two children
    const float* q = A.g.quat + 4 * (size_t)i;
    const float* s = A.g.scale + 3 * (size_t)i;
    const float* mu = A.g.mean + 3 * (size_t)i;
    const float nq = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    const float qw = q[0] / nq, qx = q[1] / nq, qy = q[2] / nq, qz = q[3] / nq;
    const float R[9] = {1.f - 2.f * (qy * qy + qz * qz), 2.f * (qx * qy - qw * qz), 2.f * (qx * qz + qw * qy),
                        2.f * (qx * qy + qw * qz), 1.f - 2.f * (qx * qx + qz * qz), 2.f * (qy * qz - qw * qx),
                        2.f * (qx * qz - qw * qy), 2.f * (qy * qz + qw * qx), 1.f - 2.f * (qx * qx + qy * qy)};
    for (int c = 0; c < 2; ++c) {
      const int64_t o = nkeep + nclone + 2 * (int64_t)(sc.z + bt.z) + c;
      for (int k = 0; k < 8; ++k)
        if (w[k]) copy_row(src[k], dst[k], i, o, w[k], A.mode == 2);
      if (A.mode == 2) continue;
      const float* zz = A.z + 6 * (size_t)i + 3 * c;
      const float l0 = s[0] * zz[0], l1 = s[1] * zz[1], l2 = s[2] * zz[2];
      for (int r = 0; r < 3; ++r)                      // identity activation: raw mean = mean
        dst[0][3 * o + r] = mu[r] + (R[3 * r] * l0 + R[3 * r + 1] * l1 + R[3 * r + 2] * l2);
      for (int r = 0; r < 3; ++r)
        dst[2][3 * o + r] = A.mode == 0 ? s[r] / 1.6f : src[2][3 * (size_t)i + r] - 0.47000362924573558f;
    }
  }
}

}  // namespace

size_t densify_workspace_bytes(int n) {
  const size_t nb = (size_t)(n + kDensT - 1) / kDensT;
  return 16 * (size_t)(n > 0 ? n : 1) + 16 * (nb > 0 ? nb : 1) + 16;
}

cudaError_t launch_dens_acc(const float* g, int n, float* acc, int* cnt, cudaStream_t st) {
  if (n > 0) { k_dens_acc<<<(n + 255) / 256, 256, 0, st>>>(g, n, acc, cnt); count_launches(1); }
  return cudaGetLastError();
}

cudaError_t launch_dens_plan(const rg_gaussians& g, const float* acc, const int* cnt, float grad_eps,
                             float extent, float sigma_eps, float percent_dense, int* action,
                             char* ws, int* counts, cudaStream_t st) {
  const int n = g.n;
  const int nb = (n + kDensT - 1) / kDensT;
  int4* scan = reinterpret_cast<int4*>(ws);
  int4* bt = reinterpret_cast<int4*>(ws + 16 * (size_t)(n > 0 ? n : 1));
  if (n == 0) {
    cudaMemsetAsync(counts, 0, 16, st);
    return cudaGetLastError();
  }
  const float small_lim = percent_dense * extent;     // fp32 product (as the oracle)
  k_dens_plan<<<nb, kDensT, 0, st>>>(g, acc, cnt, grad_eps, small_lim, sigma_eps, action, scan, bt);
  k_dens_scan<<<1, 1024, 0, st>>>(bt, nb, counts);
  count_launches(2);
  return cudaGetLastError();
}

cudaError_t launch_dens_apply(const rg_gaussians& g, const rg_gaussian_grads& in,
                              const rg_gaussian_grads& out, const int* action, const char* ws,
                              const int* counts, const float* z, int mode, cudaStream_t st) {
  const int n = g.n;
  if (n == 0) return cudaSuccess;
  DensArgs A{};
  A.g = g; A.in = in; A.out = out; A.action = action;
  A.scan = reinterpret_cast<const int4*>(ws);
  A.block_tot = reinterpret_cast<const int4*>(ws + 16 * (size_t)n);
  A.counts = counts; A.z = z;
  A.nc = (g.sh_degree + 1) * (g.sh_degree + 1); A.G = g.sg_count; A.mode = mode;
  k_dens_apply<<<(n + kDensT - 1) / kDensT, kDensT, 0, st>>>(A);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace rg
