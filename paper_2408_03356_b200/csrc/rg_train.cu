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
template <bool EXP>
__device__ __forceinline__ void step_elem(float* raw, float* m, float* v, const float* g, float* act,
                                          int64_t i, float lr, const AdamArgs& A) {
  const float r = raw[i];
  float gi = g[i];
  if (EXP) gi *= expf(r);                      // d exp(r)/dr = exp(r)
  float mi = m[i], vi = v[i];
  const float r2 = adam1(r, mi, vi, gi, lr, A);
  raw[i] = r2; m[i] = mi; v[i] = vi;
  act[i] = EXP ? expf(r2) : r2;
}

template <int D>
__device__ __forceinline__ void step_unit(float* raw, float* m, float* v, const float* g, float* act,
                                          int64_t i, float lr, bool live, const AdamArgs& A) {
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

__global__ void __launch_bounds__(256) k_adam(const AdamArgs A) {
  const int64_t total = A.seg[8];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t < A.seg[1]) {                                   // mean [n,3]
      step_elem<false>(A.raw.mean, A.m.mean, A.v.mean, A.g.mean, A.act.mean, t, A.lr[0], A);
    } else if (t < A.seg[2]) {                            // quat [n,4] as units
      step_unit<4>(A.raw.quat, A.m.quat, A.v.quat, A.g.quat, A.act.quat, t - A.seg[1], A.lr[1],
                   true, A);
    } else if (t < A.seg[3]) {                            // scale [n,3]
      step_elem<true>(A.raw.scale, A.m.scale, A.v.scale, A.g.scale, A.act.scale, t - A.seg[2],
                      A.lr[2], A);
    } else if (t < A.seg[4]) {                            // density [n]
      step_elem<true>(A.raw.density, A.m.density, A.v.density, A.g.density, A.act.density,
                      t - A.seg[3], A.lr[3], A);
    } else if (t < A.seg[5]) {                            // sh [n,nc,3]
      const int64_t i = t - A.seg[4];
      const int c = (int)((i / 3) % A.nc);
      if (c < A.sh_active)
        step_elem<false>(A.raw.sh, A.m.sh, A.v.sh, A.g.sh, A.act.sh, i, c == 0 ? A.lr[4] : A.lr[5], A);
      else
        A.act.sh[i] = A.raw.sh[i];
    } else if (t < A.seg[6]) {                            // sg_amp [n,G,3]
      const int64_t i = t - A.seg[5];
      if ((int)((i / 3) % A.G) < A.sg_active)
        step_elem<false>(A.raw.sg_amp, A.m.sg_amp, A.v.sg_amp, A.g.sg_amp, A.act.sg_amp, i, A.lr[6], A);
      else
        A.act.sg_amp[i] = A.raw.sg_amp[i];
    } else if (t < A.seg[7]) {                            // sg_sharp [n,G]
      const int64_t i = t - A.seg[6];
      if ((int)(i % A.G) < A.sg_active)
        step_elem<false>(A.raw.sg_sharp, A.m.sg_sharp, A.v.sg_sharp, A.g.sg_sharp, A.act.sg_sharp, i,
                         A.lr[7], A);
      else
        A.act.sg_sharp[i] = A.raw.sg_sharp[i];
    } else {                                              // sg_axis [n,G,3] as units
      const int64_t i = t - A.seg[7];
      step_unit<3>(A.raw.sg_axis, A.m.sg_axis, A.v.sg_axis, A.g.sg_axis, A.act.sg_axis, i, A.lr[8],
                   (int)(i % A.G) < A.sg_active, A);
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
  k_adam<<<blocks, 256, 0, st>>>(A);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace rg
