// rg_build.cu -- LBVH build over the padded support AABBs of the Gaussians
// (PAPER.md P:239):
//   k_preprocess : validity, support radius, padded tight AABB (ARITH-1..4),
//                  block-reduced bbox of valid means (ordered-int atomics)
//   k_morton     : 30-bit Morton codes of the means (ARITH-6)
//   k_digit_hist + k_radix_scatter<true> : stable LSD radix sort, 3 + 4 x 8-bit
//                  passes, CUB-free, Onesweep (all digit counts of a key set in
//                  one read; one launch per pass with decoupled look-back over the
//                  tiles; stable tile scatter ranked with __match_any_sync);
//                  RG_ONESWEEP=0: tile histogram -> single-block scan -> scatter
//   k_collapse_* : 32-wide collapse (leaf children as ranges, rg_internal.cuh)
//   k_pack       : Morton-ordered 64-B geometry records + appearance records
//   k_karras     : Karras 2012 hierarchy (one thread per internal node)
//   k_refit      : bottom-up AABB union with per-node arrival counters
#include <climits>

#include "rg_internal.cuh"

namespace rg {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;   // keys per radix tile

__device__ __forceinline__ int ord_enc(float f) {
  int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float ord_dec(int i) {
  return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF);
}

__global__ void k_init(int* bounds, float* root_box) {
  if (threadIdx.x < 3) {
    bounds[threadIdx.x] = ord_enc(INFINITY);
    bounds[3 + threadIdx.x] = ord_enc(-INFINITY);
    root_box[threadIdx.x] = INFINITY;
    root_box[3 + threadIdx.x] = -INFINITY;
  }
}

__device__ __forceinline__ bool finite_(float x) { return isfinite(x); }

// validity of every parameter of Gaussian i (non-finite -> inactive)
__device__ bool gaussian_valid(const rg_gaussians& g, int i) {
  bool ok = true;
  for (int k = 0; k < 3; ++k) {
    const float m = g.mean[3 * (size_t)i + k], s = g.scale[3 * (size_t)i + k];
    ok &= finite_(m) && finite_(s) && s > 0.0f;
  }
  for (int k = 0; k < 4; ++k) ok &= finite_(g.quat[4 * (size_t)i + k]);
  ok &= finite_(g.density[i]);
  const int nc = (g.sh_degree + 1) * (g.sh_degree + 1);
  for (int k = 0; k < 3 * nc; ++k) ok &= finite_(g.sh[(size_t)i * 3 * nc + k]);
  const int G = g.sg_count;
  for (int k = 0; k < 3 * G; ++k) ok &= finite_(g.sg_amp[(size_t)i * 3 * G + k]);
  for (int k = 0; k < G; ++k) ok &= finite_(g.sg_sharp[(size_t)i * G + k]);
  for (int k = 0; k < 3 * G; ++k) ok &= finite_(g.sg_axis[(size_t)i * 3 * G + k]);
  return ok;
}

// ARITH-2/3: M and r^2 (r2 < 0 marks inactive)
__device__ void support_exact(const rg_gaussians& g, const rg_config& c, int i, bool active,
                              float R[9], float M[9], float& r2) {
  const float* q = g.quat + 4 * (size_t)i;
  const float* s = g.scale + 3 * (size_t)i;
  rot_exact(q[0], q[1], q[2], q[3], R);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) M[3 * a + b] = div_(R[3 * b + a], s[a]);
  if (!active) { r2 = -1.0f; return; }
  if (c.radius_mode == 0) {
    // r = phi^-1(sigma_eps / sigma~) in fp64, rounded once; compact bases:
    // the unit ball
    const double k = (double)g.density[i] / (double)c.sigma_eps;
    switch (c.basis) {
      case 1: case 2: r2 = 1.0f; break;
      case 3: r2 = (float)(k * k - 1.0); break;
      case 4: r2 = (float)(k - 1.0); break;
      case 5: {
        const double l = log((double)g.density[i]) - log((double)c.sigma_eps);
        r2 = (float)(l * l);
        break;
      }
      default: r2 = (float)(2.0 * (log((double)g.density[i]) - log((double)c.sigma_eps)));
    }
  } else {
    r2 = mul_(c.k_sigma, c.k_sigma);
  }
}

__global__ void __launch_bounds__(kThreads) k_preprocess(rg_gaussians g, rg_config c,
                                                         float* box_orig, int* flags,
                                                         int* bounds) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  if (i < g.n) {
    const bool valid = gaussian_valid(g, i);
    const bool active = valid && (g.density[i] > c.sigma_eps);
    flags[i] = (valid ? 1 : 0) | (active ? 2 : 0);
    float bx[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    if (active) {
      float R[9], M[9], r2;
      support_exact(g, c, i, true, R, M, r2);
      const float* s = g.scale + 3 * (size_t)i;
      for (int a = 0; a < 3; ++a) {                             // ARITH-4
        const float a0 = mul_(s[0], R[3 * a + 0]);
        const float a1 = mul_(s[1], R[3 * a + 1]);
        const float a2 = mul_(s[2], R[3 * a + 2]);
        const float ss = dot3_(a0, a1, a2, a0, a1, a2);
        const float e = sqrt_(mul_(r2, ss));
        const float mu = g.mean[3 * (size_t)i + a];
        const float e1 = mul_(e, 0x1p-8f);
        const float m1 = mul_(add_(fabsf(mu), e), 0x1p-18f);
        const float ep = add_(add_(e, e1), m1);
        bx[a] = sub_(mu, ep);
        bx[3 + a] = add_(mu, ep);
      }
    }
    for (int k = 0; k < 6; ++k) box_orig[6 * (size_t)i + k] = bx[k];
    if (valid)
      for (int a = 0; a < 3; ++a) lo[a] = hi[a] = g.mean[3 * (size_t)i + a];
  }
  // block reduction of the bbox of valid means (exact min/max)
  for (int a = 0; a < 3; ++a) {
    for (int off = 16; off > 0; off >>= 1) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], off));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], off));
    }
  }
  if ((threadIdx.x & 31) == 0 && lo[0] <= hi[0]) {
    for (int a = 0; a < 3; ++a) {
      atomicMin(bounds + a, ord_enc(lo[a]));
      atomicMax(bounds + 3 + a, ord_enc(hi[a]));
    }
  }
}

__device__ __forceinline__ uint32_t spread10(uint32_t x) {
  x = (x * 0x00010001u) & 0xFF0000FFu;
  x = (x * 0x00000101u) & 0x0F00F00Fu;
  x = (x * 0x00000011u) & 0xC30C30C3u;
  x = (x * 0x00000005u) & 0x49249249u;
  return x;
}

__global__ void __launch_bounds__(kThreads) k_morton(rg_gaussians g, const int* flags,
                                                     const int* bounds, uint32_t* codes,
                                                     uint32_t* keys, uint32_t* vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  uint32_t code = 0xFFFFFFFFu, fine = 0u;
  if (flags[i] & 1) {
    uint32_t q[3], f[3];
    for (int a = 0; a < 3; ++a) {                               // ARITH-6
      const float lo = ord_dec(bounds[a]), hi = ord_dec(bounds[3 + a]);
      const float ext = sub_(hi, lo);
      float u = 0.0f;
      if (ext > 0.0f) u = div_(sub_(g.mean[3 * (size_t)i + a], lo), ext);
      const float v = mul_(u, 1024.0f);
      int qi = (int)floorf(v);
      qi = qi < 0 ? 0 : (qi > 1023 ? 1023 : qi);
      q[a] = (uint32_t)qi;
      int fi = (int)floorf(mul_(u, 131072.0f));                 // L34: 7 more bits per axis
      fi = fi < 0 ? 0 : (fi > 131071 ? 131071 : fi);
      f[a] = (uint32_t)fi & 127u;
    }
    code = (spread10(q[0]) << 2) | (spread10(q[1]) << 1) | spread10(q[2]);
    fine = (spread10(f[0]) << 2) | (spread10(f[1]) << 1) | spread10(f[2]);
  }
  codes[i] = code;
  keys[i] = fine;            // the first (tie-break) sort runs on the fine code
  vals[i] = (uint32_t)i;
}

// keys of the second (primary) sort: the 30-bit codes in the fine-sorted order
__global__ void __launch_bounds__(kThreads) k_gather_codes(const uint32_t* codes, const uint32_t* vin,
                                                           uint32_t* kout, uint32_t* vout, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint32_t v = vin[j];
  kout[j] = codes[v];
  vout[j] = v;
}

// --- radix sort -----------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_radix_hist(const uint32_t* keys, int n, int shift,
                                                         uint32_t* hist, int tiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int base = blockIdx.x * kTile;
  for (int r = 0; r < kItems; ++r) {
    const int i = base + r * kThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xFF], 1u);
  }
  __syncthreads();
  hist[threadIdx.x * tiles + blockIdx.x] = h[threadIdx.x];   // digit-major
}

// exclusive scan of hist[256*tiles] in place, one block of 1024 threads; the
// counts are first staged in shared memory by coalesced loads (all in flight at
// once: the per-thread serial loads of a contiguous run were latency-bound)
constexpr int kScanStage = 49152;        // staged counts (192 KB, n <= 786k); larger totals read global
__global__ void __launch_bounds__(1024) k_radix_scan(uint32_t* hist, int total) {
  extern __shared__ uint32_t stage[];
  __shared__ uint32_t part[1024];
  const int t = threadIdx.x;
  const bool staged = total <= kScanStage;
  if (staged)
    for (int i = t; i < total; i += 1024) stage[i] = hist[i];
  __syncthreads();
  const uint32_t* src = staged ? stage : hist;
  const int per = (total + 1023) / 1024;
  const int b = t * per, e = min(total, b + per);
  uint32_t s = 0;
  for (int i = b; i < e; ++i) s += src[i];
  part[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const uint32_t v = t >= off ? part[t - off] : 0u;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  uint32_t run = part[t] - s;
  for (int i = b; i < e; ++i) {
    const uint32_t v = src[i];
    if (staged) stage[i] = run; else hist[i] = run;
    run += v;
  }
  if (staged) {
    __syncthreads();
    for (int i = t; i < total; i += 1024) hist[i] = stage[i];
  }
}

// Onesweep (Adinets & Merrill 2022) building blocks: the digit counts of every
// pass from ONE read of the keys (LSD passes permute the keys, never change them)
constexpr int kOsPasses = 7;              // 3 fine-code + 4 code passes
#ifndef RG_ONESWEEP
#define RG_ONESWEEP 1
#endif
constexpr bool kOnesweep = RG_ONESWEEP != 0;
__global__ void __launch_bounds__(kThreads) k_digit_hist(const uint32_t* keys, int n, int npass,
                                                         uint32_t* gcount) {
  __shared__ uint32_t h[4][256];
  for (int p = 0; p < 4; ++p) h[p][threadIdx.x] = 0;
  __syncthreads();
  for (int i = blockIdx.x * kThreads + threadIdx.x; i < n; i += gridDim.x * kThreads) {
    const uint32_t k = keys[i];
    for (int p = 0; p < npass; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xFF], 1u);
  }
  __syncthreads();
  for (int p = 0; p < npass; ++p)
    if (h[p][threadIdx.x]) atomicAdd(&gcount[p * 256 + threadIdx.x], h[p][threadIdx.x]);
}

// Stable scatter of one LSD pass.  OS = false: the tile's digit offsets come from
// k_radix_hist + k_radix_scan (hist, digit-major).  OS = true (Onesweep): one launch
// per pass; tiles are taken in launch order from a counter, each publishes its digit
// counts (flag | count in one word: 1 = aggregate, 2 = inclusive prefix) and looks
// back over its predecessors' words (decoupled look-back) for its exclusive prefix;
// the digit bases are the exclusive scan of the pass's global counts.
constexpr uint32_t kOsAgg = 1u << 30, kOsInc = 2u << 30, kOsVal = (1u << 30) - 1u;
template <bool OS>
__global__ void __launch_bounds__(kThreads) k_radix_scatter(const uint32_t* kin, const uint32_t* vin,
                                                            uint32_t* kout, uint32_t* vout, int n,
                                                            int shift, const uint32_t* hist,
                                                            int tiles, const uint32_t* gcount,
                                                            uint32_t* status, int* tile_ctr) {
  constexpr int kWarps = kThreads / 32;
  __shared__ uint32_t base_off[256];
  __shared__ uint32_t run[256];
  __shared__ uint32_t wcnt[kWarps][256];   // (round << 16) | count
  __shared__ int tile_s;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int tile = blockIdx.x;
  if (!OS) {
    base_off[t] = hist[t * tiles + blockIdx.x];
  } else {
    if (t == 0) tile_s = atomicAdd(tile_ctr, 1);
    run[t] = 0;
    base_off[t] = gcount[t];
    __syncthreads();
    tile = tile_s;
    for (int r = 0; r < kItems; ++r) {                // this tile's digit counts
      const int i = tile * kTile + r * kThreads + t;
      if (i < n) atomicAdd(&run[(kin[i] >> shift) & 0xFF], 1u);
    }
    for (int off = 1; off < 256; off <<= 1) {         // inclusive scan of the digit bases
      const uint32_t v = t >= off ? base_off[t - off] : 0u;
      __syncthreads();
      base_off[t] += v;
      __syncthreads();
    }
    const uint32_t c = run[t];
    volatile uint32_t* vs = status;
    vs[(size_t)tile * 256 + t] = (tile == 0 ? kOsInc : kOsAgg) | c;
    uint32_t excl = 0;
    for (int p = tile - 1; p >= 0;) {                 // look-back (predecessors are resident:
      const uint32_t v = vs[(size_t)p * 256 + t];     // they took smaller tickets)
      if (!(v & (kOsAgg | kOsInc))) continue;
      excl += v & kOsVal;
      if (v & kOsInc) break;
      --p;
    }
    if (tile > 0) vs[(size_t)tile * 256 + t] = kOsInc | (excl + c);
    base_off[t] = base_off[t] - gcount[t] + excl;     // exclusive digit base + tile prefix
  }
  run[t] = 0;
  for (int w = 0; w < kWarps; ++w) wcnt[w][t] = 0xFFFF0000u;
  __syncthreads();
  const int tbase = tile * kTile;
  const uint32_t lt = (1u << lane) - 1u;
  for (int r = 0; r < kItems; ++r) {
    const int i = tbase + r * kThreads + t;
    const bool valid = i < n;
    const uint32_t key = valid ? kin[i] : 0u;
    const uint32_t val = valid ? vin[i] : 0u;
    const uint32_t dig = valid ? ((key >> shift) & 0xFF) : 256u;   // 256: invalid
    const uint32_t peers = __match_any_sync(0xffffffffu, dig);
    const uint32_t rank = __popc(peers & lt);
    if (valid && rank == 0) wcnt[warp][dig] = ((uint32_t)r << 16) | (uint32_t)__popc(peers);
    __syncthreads();
    if (valid) {
      uint32_t pre = 0;
      for (int w = 0; w < warp; ++w) {
        const uint32_t e = wcnt[w][dig];
        if ((e >> 16) == (uint32_t)r) pre += e & 0xFFFFu;
      }
      const uint32_t pos = base_off[dig] + run[dig] + pre + rank;
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncthreads();
    {
      uint32_t add = 0;
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t e = wcnt[w][t];
        if ((e >> 16) == (uint32_t)r) add += e & 0xFFFFu;
      }
      run[t] += add;
    }
    __syncthreads();
  }
}

// --- pack records in Morton order -------------------------------------------
__global__ void __launch_bounds__(kThreads) k_pack(rg_gaussians g, rg_config c,
                                                   const uint32_t* order, const float* box_orig,
                                                   const int* flags, float4* geom, float* app,
                                                   int stride, float* leaf_box) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.n) return;
  const int i = (int)order[p];
  const bool active = (flags[i] & 2) != 0;
  float R[9], M[9], r2;
  support_exact(g, c, i, active, R, M, r2);
  const float* mu = g.mean + 3 * (size_t)i;
  float4* gp = geom + 4 * (size_t)p;
  gp[0] = make_float4(mu[0], mu[1], mu[2], g.density[i]);
  gp[1] = make_float4(M[0], M[1], M[2], M[3]);
  gp[2] = make_float4(M[4], M[5], M[6], M[7]);
  gp[3] = make_float4(M[8], r2, __int_as_float(i), 0.0f);
  for (int k = 0; k < 6; ++k) leaf_box[6 * (size_t)p + k] = box_orig[6 * (size_t)i + k];
  (void)app;
  (void)stride;
}

// appearance record in Morton order, one warp per Gaussian row (coalesced):
// SH [(deg+1)^2 x 3] zero-padded to 48 floats, then per lobe
// (k0,k1,k2, lambda, p0,p1,p2), zero pad.
__global__ void __launch_bounds__(kThreads) k_pack_app(rg_gaussians g, const uint32_t* order,
                                                       float* app, int stride) {
  const int lane = threadIdx.x & 31;
  const int nc3 = 3 * (g.sh_degree + 1) * (g.sh_degree + 1);
  const int G = g.sg_count;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < g.n;
       p += (gridDim.x * blockDim.x) >> 5) {
    const size_t i = order[p];
    float* ap = app + (size_t)p * stride;
    // <= 100 floats per row: up to 4 per lane, all loads issued before the stores
    constexpr int kPer = (kShFloats + 7 * kMaxLobes + 3 + 31) / 32;
    float v[kPer];
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int f = lane + 32 * t;
      v[t] = 0.0f;
      if (f < nc3) {
        v[t] = g.sh[i * nc3 + f];
      } else if (f >= kShFloats && f < kShFloats + 7 * G) {
        const int j = (f - kShFloats) / 7, r = (f - kShFloats) - 7 * j;
        const size_t ij = i * G + j;
        v[t] = r < 3 ? g.sg_amp[3 * ij + r] : (r == 3 ? g.sg_sharp[ij] : g.sg_axis[3 * ij + r - 4]);
      }
    }
#pragma unroll
    for (int t = 0; t < kPer; ++t) {
      const int f = lane + 32 * t;
      if (f < stride) ap[f] = v[t];
    }
  }
}

// --- Karras 2012 ---------------------------------------------------------------
__device__ __forceinline__ int delta(const uint32_t* k, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  const uint32_t a = k[i], b = k[j];
  return a == b ? 32 + __clz(i ^ j) : __clz(a ^ b);
}

__global__ void __launch_bounds__(kThreads) k_karras(const uint32_t* k, int n, float4* nodes,
                                                     int* parent_int, int* parent_leaf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  const int d = (delta(k, n, i, i + 1) - delta(k, n, i, i - 1)) > 0 ? 1 : -1;
  const int dmin = delta(k, n, i, i - d);
  int lmax = 2;
  while (delta(k, n, i, i + lmax * d) > dmin) lmax <<= 1;
  int l = 0;
  for (int t = lmax >> 1; t >= 1; t >>= 1)
    if (delta(k, n, i, i + (l + t) * d) > dmin) l += t;
  const int j = i + l * d;
  const int dnode = delta(k, n, i, j);
  int s = 0;
  for (int div = 2;; div <<= 1) {
    const int t = (l + div - 1) / div;
    if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
    if (t <= 1) break;
  }
  const int gamma = i + s * d + min(d, 0);
  const int left = (min(i, j) == gamma) ? ~gamma : gamma;
  const int right = (max(i, j) == gamma + 1) ? ~(gamma + 1) : gamma + 1;
  nodes[4 * (size_t)i + 3] = make_float4(__int_as_float(left), __int_as_float(right),
                                         __int_as_float(min(i, j)), __int_as_float(max(i, j)));
  if (left < 0) parent_leaf[~left] = i; else parent_int[left] = i;
  if (right < 0) parent_leaf[~right] = i; else parent_int[right] = i;
  if (i == 0) parent_int[0] = -1;
}

// --- refit ------------------------------------------------------------------------
__device__ __forceinline__ void store_child_box(float4* nodes, int parent, bool is_left,
                                                const float b[6]) {
  float* w = reinterpret_cast<float*>(nodes + 4 * (size_t)parent);
  const int o = is_left ? 0 : 6;
  for (int k = 0; k < 6; ++k) __stcg(w + o + k, b[k]);
}

__global__ void __launch_bounds__(kThreads) k_refit(const float* leaf_box, float4* nodes,
                                                    const int* parent_int, const int* parent_leaf,
                                                    int* cnt, float* root_box, int n) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  float b[6];
  for (int k = 0; k < 6; ++k) b[k] = leaf_box[6 * (size_t)p + k];
  if (n == 1) {
    for (int k = 0; k < 6; ++k) root_box[k] = b[k];
    return;
  }
  int child = ~p;
  int node = parent_leaf[p];
  while (true) {
    const int4 ids = __ldcg(reinterpret_cast<const int4*>(nodes + 4 * (size_t)node + 3));
    store_child_box(nodes, node, ids.x == child, b);
    __threadfence();
    if (atomicAdd(cnt + node, 1) == 0) return;     // first arrival: sibling finishes
    __threadfence();
    const float* w = reinterpret_cast<const float*>(nodes + 4 * (size_t)node);
    float l[6], r[6];
    for (int k = 0; k < 6; ++k) { l[k] = __ldcg(w + k); r[k] = __ldcg(w + 6 + k); }
    for (int k = 0; k < 3; ++k) {
      b[k] = fminf(l[k], r[k]);
      b[3 + k] = fmaxf(l[3 + k], r[3 + k]);
    }
    if (node == 0) {
      for (int k = 0; k < 6; ++k) root_box[k] = b[k];
      return;
    }
    child = node;
    node = parent_int[node];
  }
}

// --- collapse of the binary tree into 32-wide nodes (traversal structure) --------
// Greedy top-down: a wide node's children are a cut of the binary subtree,
// grown by repeatedly opening the internal entry with the largest box surface
// area until 32 entries (or only leaves) remain.  One persistent launch over a
// device work queue of (binary id, wide id) items (k_collapse_warp).
__device__ __forceinline__ float box_area(const float* b) {
  const float dx = b[3] - b[0], dy = b[4] - b[1], dz = b[5] - b[2];
  return (dx < 0.f || dy < 0.f || dz < 0.f) ? -1.f : dx * dy + dy * dz + dz * dx;
}

__global__ void k_collapse_init(int n, const float* leaf_box, WideNode* wide, int2* wq,
                                int* wide_src, int* counts) {
  const int l = threadIdx.x;
  if (l == 0) {
    // [0] wide nodes allocated, [1] head, [2] done, [3] error, [4] reserved
    for (int k = 0; k < 8; ++k) counts[k] = 0;
    counts[0] = 1;
    wide_src[0] = 0;
    if (n > 1) {
      wq[0] = make_int2(0, 0);   // binary root -> wide node 0
      counts[4] = 1;
    }
  }
  if (n == 1) {
    wide[0].lox[l] = l == 0 ? leaf_box[0] : INFINITY;
    wide[0].loy[l] = l == 0 ? leaf_box[1] : INFINITY;
    wide[0].loz[l] = l == 0 ? leaf_box[2] : INFINITY;
    wide[0].hix[l] = l == 0 ? leaf_box[3] : -INFINITY;
    wide[0].hiy[l] = l == 0 ? leaf_box[4] : -INFINITY;
    wide[0].hiz[l] = l == 0 ? leaf_box[5] : -INFINITY;
    wide[0].child[l] = l == 0 ? ~0 : kWideEmpty;
  }
}

// refit of the wide nodes after k_refit (rg_refit_bvh): one warp per wide
// node, lane = child slot; an internal child's box is the union of its binary
// node's two child boxes, a leaf's its padded AABB; the topology is kept.
__global__ void __launch_bounds__(128) k_wide_refit(const float4* nodes, const float* leaf_box,
                                                    const int* wide_src, const int* counts,
                                                    WideNode* wide, int capacity) {
  const int lane = threadIdx.x & 31;
  const int nw = min(counts[0], capacity);
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw;
       w += (gridDim.x * blockDim.x) >> 5) {
    WideNode& W = wide[w];
    const int child = W.child[lane];
    if (child == kWideEmpty) continue;
    float b[6];
    if (child < 0) {                                  // union of the range's leaf boxes
      const int f = leaf_range_first(child), c = leaf_range_count(child);
      for (int k = 0; k < 6; ++k) b[k] = leaf_box[6 * (size_t)f + k];
      for (int r = 1; r < c; ++r)
        for (int k = 0; k < 3; ++k) {
          b[k] = fminf(b[k], leaf_box[6 * (size_t)(f + r) + k]);
          b[3 + k] = fmaxf(b[3 + k], leaf_box[6 * (size_t)(f + r) + 3 + k]);
        }
    } else {
      const float* x = reinterpret_cast<const float*>(nodes + 4 * (size_t)wide_src[child]);
      for (int k = 0; k < 3; ++k) {
        b[k] = fminf(x[k], x[6 + k]);
        b[3 + k] = fmaxf(x[3 + k], x[9 + k]);
      }
    }
    W.lox[lane] = b[0]; W.loy[lane] = b[1]; W.loz[lane] = b[2];
    W.hix[lane] = b[3]; W.hiy[lane] = b[4]; W.hiz[lane] = b[5];
  }
}

// entries opened per round of the 32-wide collapse and resident blocks per SM of the
// persistent collapse kernel: medians of 9 (tools/ab.py, C1; profiles/r2/ab_build.log):
// open 1 / 16 blocks 0.911 ms, open 1 / 4 blocks 0.838 ms (more spinning warps contend
// on the queue counters), open 2 / 16 blocks 0.797 ms with the forward +0.014 ms (the
// two-per-round cut is a slightly worse tree, far less than the build time it saves)
// Re-measured on the final round-2 code (profiles/r2/ab_knobs_final.log): open 1 builds
// in 0.695 ms against 0.779 ms for open 2, forward 6.223 vs 6.237 ms -> 1 again
#ifndef RG_COLLAPSE_OPEN
#define RG_COLLAPSE_OPEN 1
#endif
#ifndef RG_COLLAPSE_BLOCKS
#define RG_COLLAPSE_BLOCKS 4
#endif
#ifndef RG_COLLAPSE_PREFETCH
#define RG_COLLAPSE_PREFETCH 0   // prefetch entries when placed (medians of 9: 0.783 vs 0.787 ms, no gain)
#endif
// Collapse of the binary tree into 32-wide nodes, one persistent launch over a
// device work queue of (binary id, wide id) items.  The queue is pre-filled with
// -1; an item is written with one 8-byte store after its slot is reserved.  A
// warp whose claimed slot is not reserved exits once done == reserved is observed
// (done read before reserved): every reserved item is then finished, so no
// further item can appear.  counts: [0] wide nodes allocated, [1] head (claims),
// [2] items done, [3] error flag, [4] items reserved.
// Per item (one warp): lane k holds candidate entry k (id, box,
// area) in registers; each round opens, in parallel, the largest-area internal
// entries (RG_COLLAPSE_OPEN per round; 1 = the greedy cut of the thread variant),
// left child in place, right child appended; no local-memory candidate arrays.
// Bulk reservations of wide ids and queue slots per item.
__global__ void __launch_bounds__(128) k_collapse_warp(const float4* nodes, WideNode* wide, int2* q,
                                                       int* wide_src, int* counts, int capacity) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  volatile int* vc = counts;
  volatile long long* vq = reinterpret_cast<volatile long long*>(q);
  while (true) {
    long long raw = -1;
    int have = 0;
    if (lane == 0) {
      const int it = atomicAdd(counts + 1, 1);
      while (true) {
        const int done = vc[2];
        __threadfence();
        const int res = vc[4];
        if (it < res) {
          raw = vq[it];
          if ((int)(raw & 0xFFFFFFFF) != -1) { have = 1; break; }
        } else if (done == res) {
          break;
        }
        __nanosleep(64);
      }
    }
    have = __shfl_sync(full, have, 0);
    if (!have) return;
    raw = __shfl_sync(full, raw, 0);
    const int jb = (int)(raw & 0xFFFFFFFF), jw = (int)(raw >> 32);
    if (jw < 0) {                                     // no-op item (capacity guard)
      if (lane == 0) atomicAdd(counts + 2, 1);
      continue;
    }
    // entries 0, 1: the binary node's children
    // each entry also carries its leaf range [f, f + cnt) (Morton order)
    int id = -1, f = 0, cnt = 0;
    float b[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    if (lane < 2) {
      const float* w = reinterpret_cast<const float*>(nodes + 4 * (size_t)jb);
      const int4 c = *reinterpret_cast<const int4*>(nodes + 4 * (size_t)jb + 3);
      id = lane == 0 ? c.x : c.y;
      const int gamma = c.x >= 0 ? c.x : ~c.x;        // left child's last leaf
      f = lane == 0 ? c.z : gamma + 1;
      cnt = lane == 0 ? gamma - c.z + 1 : c.w - gamma;
      for (int k = 0; k < 6; ++k) b[k] = w[6 * lane + k];
    }
#if RG_COLLAPSE_PREFETCH
    // each lane prefetches the binary record (child ids and boxes) of its entry as
    // soon as it holds it, so opening an entry no longer waits on a dependent load
    int2 pc = make_int2(-1, -1);
    float pw[12];
    auto prefetch = [&]() {
      if (id >= 0) {
        const float4* nd = nodes + 4 * (size_t)id;
        const float4 n0 = nd[0], n1 = nd[1], n2 = nd[2], n3 = nd[3];
        pw[0] = n0.x; pw[1] = n0.y; pw[2] = n0.z; pw[3] = n0.w;
        pw[4] = n1.x; pw[5] = n1.y; pw[6] = n1.z; pw[7] = n1.w;
        pw[8] = n2.x; pw[9] = n2.y; pw[10] = n2.z; pw[11] = n2.w;
        pc = make_int2(__float_as_int(n3.x), __float_as_int(n3.y));
      }
    };
    prefetch();
#endif
    int m = 2;
    while (m < kWide) {
      const bool internal = lane < m && id >= 0;
      if (!__ballot_sync(full, internal)) break;
      // subtrees of more than kLeafRange leaves open first (largest area); the
      // small ones (future leaf ranges) only open while slots remain
      const bool big = internal && (kLeafRange == 1 || cnt > kLeafRange);
      const unsigned bm = __ballot_sync(full, big);
      const bool cand = bm ? big : internal;
      const unsigned cm = __ballot_sync(full, cand);
      const float area = cand ? box_area(b) : -2.f;
      int rank = 0;                                   // by area, descending (ties: lane)
      if (RG_COLLAPSE_OPEN <= 2) {
        // only ranks < 2 open: the largest areas, lowest lane on ties (reductions
        // instead of a 32-step rank loop; the same entries as the rank order)
        const int key = ord_enc(area);
        const int kmax = __reduce_max_sync(full, key);
        const int first = __ffs(__ballot_sync(full, key == kmax)) - 1;
        rank = lane == first ? 0 : 2;
        if (RG_COLLAPSE_OPEN == 2) {
          const int key2 = lane == first ? INT_MIN : key;
          const int kmax2 = __reduce_max_sync(full, key2);
          const int second = __ffs(__ballot_sync(full, key2 == kmax2)) - 1;
          if (lane == second && lane != first) rank = 1;
        }
      } else {
        for (unsigned mm = cm; mm; mm &= mm - 1) {
          const int o = __ffs(mm) - 1;
          const float ao = __shfl_sync(full, area, o);
          rank += (ao > area) || (ao == area && o < lane);
        }
      }
      const int r = min(min(__popc(cm), kWide - m), RG_COLLAPSE_OPEN);
      const bool open = cand && rank < r;
      int rid = -1, rf = 0, rcnt = 0;
      float rb[6];
      if (open) {                                     // left child in place, right one out
#if RG_COLLAPSE_PREFETCH
        id = pc.x;
        rid = pc.y;
        for (int k = 0; k < 6; ++k) { b[k] = pw[k]; rb[k] = pw[6 + k]; }
#else
        const float* w = reinterpret_cast<const float*>(nodes + 4 * (size_t)id);
        const int4 c = *reinterpret_cast<const int4*>(nodes + 4 * (size_t)id + 3);
        id = c.x;
        rid = c.y;
        for (int k = 0; k < 6; ++k) { b[k] = w[k]; rb[k] = w[6 + k]; }
#endif
        if (kLeafRange > 1) {                         // ranges tracked only when used
          const int gamma = id >= 0 ? id : ~id;
          rf = gamma + 1;
          rcnt = f + cnt - 1 - gamma;
          cnt = gamma - f + 1;
        }
      }
      bool fresh = open;
      for (int j = 0; j < r; ++j) {                   // right child of rank j -> lane m + j
        const int src = __ffs(__ballot_sync(full, open && rank == j)) - 1;
        const int vid = __shfl_sync(full, rid, src);
        const int vf = kLeafRange > 1 ? __shfl_sync(full, rf, src) : 0;
        const int vc = kLeafRange > 1 ? __shfl_sync(full, rcnt, src) : 0;
        float vb[6];
        for (int k = 0; k < 6; ++k) vb[k] = __shfl_sync(full, open ? rb[k] : 0.f, src);
        if (lane == m + j) {
          id = vid;
          f = vf;
          cnt = vc;
          for (int k = 0; k < 6; ++k) b[k] = vb[k];
          fresh = true;
        }
      }
#if RG_COLLAPSE_PREFETCH
      if (fresh) prefetch();
#else
      (void)fresh;
#endif
      m += r;
    }
    // write the wide node; internal children of more than kLeafRange leaves become
    // queue items, the others leaf ranges (single leaves: ranges of one)
    const bool live = lane < m;
    const bool internal = live && id >= 0 && (kLeafRange == 1 || cnt > kLeafRange);
    const unsigned im = __ballot_sync(full, internal);
    const int nint = __popc(im);
    int wid0 = 0, qs0 = 0;
    if (lane == 0 && nint) {
      wid0 = atomicAdd(counts + 0, nint);
      qs0 = atomicAdd(counts + 4, nint);              // reserve the queue slots
    }
    wid0 = __shfl_sync(full, wid0, 0);
    qs0 = __shfl_sync(full, qs0, 0);
    int child = !live ? kWideEmpty : id < 0 ? leaf_range_enc(~id, 1) : leaf_range_enc(f, cnt);
    if (internal) {
      const int rk = __popc(im & ((1u << lane) - 1u));
      const int wid = wid0 + rk;
      if (wid < capacity) {
        wide_src[wid] = id;
        vq[qs0 + rk] = ((long long)wid << 32) | (unsigned)id;   // publish with one store
        child = wid;
      } else {
        // beyond the proven wide_capacity bound (cannot happen): flag, drop the subtree
        // and publish a no-op item (wide id -1) so that the queue still drains
        counts[3] = 1;
        vq[qs0 + rk] = (long long)(~0ull << 32) | (unsigned)id;
        child = kWideEmpty;
      }
    }
    WideNode& W = wide[jw];
    W.lox[lane] = b[0]; W.loy[lane] = b[1]; W.loz[lane] = b[2];
    W.hix[lane] = b[3]; W.hiy[lane] = b[4]; W.hiz[lane] = b[5];
    W.child[lane] = child;
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicAdd(counts + 2, 1);          // this item is done
  }
}

// error flag: unfinished items or wide-node capacity exceeded (the guard in
// k_collapse_warp may already have set it)
__global__ void k_collapse_check(int* counts, int capacity) {
  counts[3] = (counts[3] != 0 || counts[2] != counts[4] || counts[0] > capacity) ? 1 : 0;
}

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

BvhLayout bvh_layout(int n, int deg, int lobes) {
  BvhLayout L{};
  const size_t nn = n > 0 ? (size_t)n : 1;
  const size_t ni = n > 1 ? (size_t)(n - 1) : 1;
  L.tiles = (int)((nn + kTile - 1) / kTile);
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += al(bytes); return r; };
  L.geom = take(64 * nn);
  L.app = take(sizeof(float) * (size_t)app_stride(deg, lobes) * nn);
  L.nodes = take(64 * ni);
  L.leaf_box = take(24 * nn);
  L.root_box = take(32);
  L.codes = take(4 * nn);
  L.keys_a = take(4 * nn);
  L.keys_b = take(4 * nn);
  L.vals_a = take(4 * nn);
  L.vals_b = take(4 * nn);
  L.box_orig = take(24 * nn);
  L.flags = take(4 * nn);
  L.parent_int = take(4 * ni);
  L.parent_leaf = take(4 * nn);
  L.refit_cnt = take(4 * ni);
  L.bounds = take(32);
  // hist: [256 * tiles] of the per-pass hist/scan sort, or the Onesweep words:
  // [kOsPasses][tiles][256] status, [kOsPasses][256] digit counts, [8] tile counters
  L.hist = take(4 * ((size_t)kOsPasses * 256 * (L.tiles + 1) + 8));
  L.wide = take(sizeof(WideNode) * wide_capacity(n));
  L.wq_a = take(8 * nn);
  L.wide_src = take(8 * nn);
  L.wcounts = take(32);
  L.total = o;
  return L;
}

cudaError_t launch_build(const rg_gaussians& g, const rg_config& c, char* ws, const BvhLayout& L,
                         cudaStream_t st) {
  const int n = g.n;
  float* root_box = reinterpret_cast<float*>(ws + L.root_box);
  int* bounds = reinterpret_cast<int*>(ws + L.bounds);
  k_init<<<1, 32, 0, st>>>(bounds, root_box);
  count_launches(1);
  if (n == 0) return cudaGetLastError();
  // preprocess, morton, gather, pack, pack_app (+ karras, refit) and the sort: 7 x 3
  // launches, or 7 Onesweep passes + 2 digit histograms
  count_launches((n > 1 ? 28 : 27) - (kOnesweep ? 12 : 0));
  const int blocks = (n + kThreads - 1) / kThreads;
  float* box_orig = reinterpret_cast<float*>(ws + L.box_orig);
  int* flags = reinterpret_cast<int*>(ws + L.flags);
  k_preprocess<<<blocks, kThreads, 0, st>>>(g, c, box_orig, flags, bounds);
  uint32_t* ka = reinterpret_cast<uint32_t*>(ws + L.keys_a);
  uint32_t* kb = reinterpret_cast<uint32_t*>(ws + L.keys_b);
  uint32_t* va = reinterpret_cast<uint32_t*>(ws + L.vals_a);
  uint32_t* vb = reinterpret_cast<uint32_t*>(ws + L.vals_b);
  k_morton<<<blocks, kThreads, 0, st>>>(g, flags, bounds,
                                        reinterpret_cast<uint32_t*>(ws + L.codes), ka, va);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist);
  const size_t scan_smem = 256 * (size_t)L.tiles <= (size_t)kScanStage ? 4 * 256 * (size_t)L.tiles : 0;
  {
    static bool opted = false;          // > 48 KB of dynamic shared memory needs an opt-in
    if (!opted) {
      cudaFuncSetAttribute(k_radix_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           4 * kScanStage);
      opted = true;
    }
  }
  uint32_t* os_status = hist;
  uint32_t* os_count = hist + (size_t)kOsPasses * 256 * L.tiles;
  int* os_ctr = reinterpret_cast<int*>(os_count + kOsPasses * 256);
  const int hblocks = min(L.tiles, 148 * 2);
  if (kOnesweep)
    cudaMemsetAsync(hist, 0, 4 * ((size_t)kOsPasses * 256 * (L.tiles + 1) + 8), st);
  int os_pass = 0;
  auto radix_pass = [&](const uint32_t* ki, const uint32_t* vi, uint32_t* ko, uint32_t* vo,
                        int shift) {
    if (kOnesweep) {
      k_radix_scatter<true><<<L.tiles, kThreads, 0, st>>>(
          ki, vi, ko, vo, n, shift, nullptr, L.tiles, os_count + 256 * os_pass,
          os_status + (size_t)256 * L.tiles * os_pass, os_ctr + os_pass);
      ++os_pass;
      return;
    }
    k_radix_hist<<<L.tiles, kThreads, 0, st>>>(ki, n, shift, hist, L.tiles);
    k_radix_scan<<<1, 1024, scan_smem, st>>>(hist, 256 * L.tiles);
    k_radix_scatter<false><<<L.tiles, kThreads, 0, st>>>(ki, vi, ko, vo, n, shift, hist, L.tiles,
                                                         nullptr, nullptr, nullptr);
  };
  // stable LSD sort by (code, fine code, index) (L34): first the 21-bit fine code
  // (3 passes, ending in kb/vb), then the 30-bit code (4 passes, ending in ka/va)
  if (kOnesweep) k_digit_hist<<<hblocks, kThreads, 0, st>>>(ka, n, 3, os_count);
  radix_pass(ka, va, kb, vb, 0);
  radix_pass(kb, vb, ka, va, 8);
  radix_pass(ka, va, kb, vb, 16);
  k_gather_codes<<<blocks, kThreads, 0, st>>>(reinterpret_cast<const uint32_t*>(ws + L.codes), vb,
                                              ka, va, n);
  if (kOnesweep) k_digit_hist<<<hblocks, kThreads, 0, st>>>(ka, n, 4, os_count + 3 * 256);
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 8 * pass;
    if (pass & 1) radix_pass(kb, vb, ka, va, shift);
    else radix_pass(ka, va, kb, vb, shift);
  }
  float4* geom = reinterpret_cast<float4*>(ws + L.geom);
  float* app = reinterpret_cast<float*>(ws + L.app);
  float* leaf_box = reinterpret_cast<float*>(ws + L.leaf_box);
  k_pack<<<blocks, kThreads, 0, st>>>(g, c, va, box_orig, flags, geom, app,
                                      app_stride(g.sh_degree, g.sg_count), leaf_box);
  {
    const int warps_needed = n, per_block = kThreads / 32;
    const int ablocks = min((warps_needed + per_block - 1) / per_block, 148 * 16);
    k_pack_app<<<ablocks, kThreads, 0, st>>>(g, va, app, app_stride(g.sh_degree, g.sg_count));
  }
  float4* nodes = reinterpret_cast<float4*>(ws + L.nodes);
  int* parent_int = reinterpret_cast<int*>(ws + L.parent_int);
  int* parent_leaf = reinterpret_cast<int*>(ws + L.parent_leaf);
  int* cnt = reinterpret_cast<int*>(ws + L.refit_cnt);
  if (n > 1) {
    const int bi = (n - 1 + kThreads - 1) / kThreads;
    k_karras<<<bi, kThreads, 0, st>>>(ka, n, nodes, parent_int, parent_leaf);
    cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)(n - 1), st);
  }
  k_refit<<<blocks, kThreads, 0, st>>>(leaf_box, nodes, parent_int, parent_leaf, cnt, root_box, n);
  // 32-wide collapse: one persistent launch over the device work queue
  WideNode* wide = reinterpret_cast<WideNode*>(ws + L.wide);
  int2* qa = reinterpret_cast<int2*>(ws + L.wq_a);
  int* wc = reinterpret_cast<int*>(ws + L.wcounts);
  int* wsrc = reinterpret_cast<int*>(ws + L.wide_src);
  if (n > 1) cudaMemsetAsync(qa, 0xFF, 8 * (size_t)n, st);
  k_collapse_init<<<1, 32, 0, st>>>(n, leaf_box, wide, qa, wsrc, wc);
  count_launches(1);
  if (n > 1) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // persistent warps over the work queue (a warp claims a slot, then waits for its
    // item; unclaimed blocks hold nothing, so co-residency is not needed).  Each item
    // is ~31 dependent rounds (one L2 load each): latency-bound, so the whole SM is
    // filled -- RG_COLLAPSE_BLOCKS blocks of 128 per SM (28 registers: 16 fit)
    k_collapse_warp<<<RG_COLLAPSE_BLOCKS * sms, 128, 0, st>>>(nodes, wide, qa, wsrc, wc,
                                                             (int)wide_capacity(n));
    k_collapse_check<<<1, 1, 0, st>>>(wc, (int)wide_capacity(n));
    count_launches(2);
  }
  return cudaGetLastError();
}

// UpdateBVH by refit: new parameters, same n and the
// topology of the last launch_build on this workspace (Morton order, Karras
// tree, 32-wide collapse).  Records, AABBs and every box are recomputed; a
// stale order only costs traversal efficiency, never correctness (boxes stay
// conservative unions).
cudaError_t launch_refit(const rg_gaussians& g, const rg_config& c, char* ws, const BvhLayout& L,
                         cudaStream_t st) {
  const int n = g.n;
  float* root_box = reinterpret_cast<float*>(ws + L.root_box);
  int* bounds = reinterpret_cast<int*>(ws + L.bounds);
  k_init<<<1, 32, 0, st>>>(bounds, root_box);
  count_launches(1);
  if (n == 0) return cudaGetLastError();
  const int blocks = (n + kThreads - 1) / kThreads;
  float* box_orig = reinterpret_cast<float*>(ws + L.box_orig);
  int* flags = reinterpret_cast<int*>(ws + L.flags);
  k_preprocess<<<blocks, kThreads, 0, st>>>(g, c, box_orig, flags, bounds);
  const uint32_t* va = reinterpret_cast<const uint32_t*>(ws + L.vals_a);
  float4* geom = reinterpret_cast<float4*>(ws + L.geom);
  float* app = reinterpret_cast<float*>(ws + L.app);
  float* leaf_box = reinterpret_cast<float*>(ws + L.leaf_box);
  const int stride = app_stride(g.sh_degree, g.sg_count);
  k_pack<<<blocks, kThreads, 0, st>>>(g, c, va, box_orig, flags, geom, app, stride, leaf_box);
  k_pack_app<<<min((n + kThreads / 32 - 1) / (kThreads / 32), 148 * 16), kThreads, 0, st>>>(
      g, va, app, stride);
  float4* nodes = reinterpret_cast<float4*>(ws + L.nodes);
  int* cnt = reinterpret_cast<int*>(ws + L.refit_cnt);
  if (n > 1) cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)(n - 1), st);
  k_refit<<<blocks, kThreads, 0, st>>>(leaf_box, nodes, reinterpret_cast<const int*>(ws + L.parent_int),
                                       reinterpret_cast<const int*>(ws + L.parent_leaf), cnt,
                                       root_box, n);
  WideNode* wide = reinterpret_cast<WideNode*>(ws + L.wide);
  int* wsrc = reinterpret_cast<int*>(ws + L.wide_src);
  int* wc = reinterpret_cast<int*>(ws + L.wcounts);
  count_launches(5);
  if (n == 1) {
    k_collapse_init<<<1, 32, 0, st>>>(n, leaf_box, wide, reinterpret_cast<int2*>(ws + L.wq_a), wsrc,
                                      wc);
  } else {
    const int wblocks = min((int)((wide_capacity(n) + 3) / 4), 148 * 8);
    k_wide_refit<<<wblocks, 128, 0, st>>>(nodes, leaf_box, wsrc, wc, wide, (int)wide_capacity(n));
  }
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace rg
