// rg_render.cu -- slab-by-slab volume ray casting of the Gaussians through the
// BVH, forward and backward:
//
//   PAPER.md Alg. 2: per ray, bbox clip, then slabs of B samples
//   of length dt*B; per slab the set of Gaussians whose support overlaps the
//   slab (Alg. 1 any-hit collection, capped at K = n_max with the
//   K smallest (t_entry, index) kept -- DESIGN.md L7), sorted by entry depth;
//   UpdateRay = evaluate sigma and the density-weighted colour at the B
//   samples (Eq. 10-16) and composite front to back (Eq. 4); early
//   termination at slab granularity when T <= T_eps.
//
// B200 design: ONE WARP PER RAY.  The ray keeps a sorted
// ACTIVE LIST (shared memory, capacity kA) of its upcoming/overlapping
// Gaussians with their per-pair data (exact interval, weight-exponent
// polynomial, colour), refilled by a warp-cooperative k-nearest-by-t_entry
// traversal of the 32-wide BVH ("next k keys after a cursor"): one node visit
// = 32 lanes testing the node's 32 child boxes, leaf children tested exactly
// by their lane, the k-buffer held one key per lane (rank/ballot merge),
// internal children pushed nearest-last on a shared stack.  Empty slabs are
// skipped exactly (jump to the slab holding the next t_entry).  Integration
// maps lanes to (entry-subset x sample) and reduces with shuffles;
// compositing is a segmented scan over the slab's samples with the optical
// depth accumulated (Kahan) so T does not drift over thousands of samples.
// Backward replays the same march, walks each sample group front to back with
// suffix = P - prefix (L16), accumulates per-pair moments in shared memory
// and scatters each pair's 16 + app_stride gradient floats as one coalesced
// burst of float4 atomics (one per lane) into a Morton-ordered buffer;
// k_finalize converts (mu, M) -> (mu, q, s) and un-permutes.
#include "rg_internal.cuh"

namespace rg {

namespace {

constexpr int kWarps = 4;              // rays (warps) per block
constexpr int kBlock = 32 * kWarps;
constexpr int kA = 64;                 // persistent active-list capacity
constexpr int kSlots = kA + 32;        // + one transient chunk (slab sets > kA)
constexpr int kStk = 256;              // traversal stack (wide nodes)
constexpr unsigned kFull = 0xffffffffu;

struct Counters {
  uint32_t slabs, pairs, evals, samples, overflows, fetches, nodes, stackov;
};

struct RenderArgs {
  SceneView S;
  rg_config c;
  int cam_mode;
  rg_camera cam;
  int rw, rh, tiles_x;
  const float* ro;
  const float* rd;
  int n_rays;
  float* rgb;
  float* T;
  int32_t* replay;
  rg_stats* stats;
  int dbg_rays, dbg_cap;
  int32_t* dbg_counts;
  int32_t* dbg_rec;
  // backward
  const float* rgb_in;
  const int32_t* replay_in;
  const float* d_rgb;
  float* gbuf;
  int gstride;
};

struct WarpMem {
  float te[kSlots], tx[kSlots], tm[kSlots], c0[kSlots], c1[kSlots], c2[kSlots];
  float cr[kSlots], cg[kSlots], cb[kSlots];
  int pos[kSlots];
  uint32_t idx[kSlots];
  int stk[kStk];
  unsigned long long kscr[32];
  uint32_t pscr[32];
  float Y[16];
};
struct WarpAcc {
  float a[6][kSlots];   // Sw, Sw1, Sw2, dc_r, dc_g, dc_b per slot
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned long long shfl64(unsigned long long v, int src) {
  const unsigned lo = __shfl_sync(kFull, (unsigned)v, src);
  const unsigned hi = __shfl_sync(kFull, (unsigned)(v >> 32), src);
  return ((unsigned long long)hi << 32) | lo;
}

// conservative ray/AABB overlap (sign-selected slabs: empty boxes never hit)
__device__ __forceinline__ void box_t(float lx, float ly, float lz, float hx, float hy, float hz,
                                      const float3& inv, const float3& oinv, float& tn, float& tf) {
  const float ax = fmaf(lx, inv.x, -oinv.x), bx = fmaf(hx, inv.x, -oinv.x);
  const float ay = fmaf(ly, inv.y, -oinv.y), by = fmaf(hy, inv.y, -oinv.y);
  const float az = fmaf(lz, inv.z, -oinv.z), bz = fmaf(hz, inv.z, -oinv.z);
  const float nx = inv.x >= 0.f ? ax : bx, fx = inv.x >= 0.f ? bx : ax;
  const float ny = inv.y >= 0.f ? ay : by, fy = inv.y >= 0.f ? by : ay;
  const float nz = inv.z >= 0.f ? az : bz, fz = inv.z >= 0.f ? bz : az;
  tn = fmaxf(fmaxf(nx, ny), nz);
  tf = fminf(fminf(fx, fy), fz);
}

struct Ray {
  float3 o, d, inv, oinv;
};

// Warp-cooperative k-nearest query on the 32-wide BVH: the kmax (<= 32)
// smallest keys (t_entry bits, index) > cursor among Gaussians whose exact
// support interval satisfies t_exit >= seg_lo and t_entry <= seg_hi.
// Result: lane l < return value holds the l-th smallest key and its position.
__device__ int fetch(const SceneView& S, WarpMem& M, const Ray& R, float seg_lo, float seg_hi,
                     unsigned long long cursor, int kmax, unsigned long long& key, uint32_t& pos,
                     Counters& cnt) {
  const unsigned lane = lane_id();
  const unsigned lt_mask = (1u << lane) - 1u;
  if (lane == 0) cnt.fetches++;
  key = ~0ull;
  pos = 0;
  int nk = 0;
  float te_lim = INFINITY;
  unsigned long long kth = ~0ull;
  const float slack = 1e-5f * (fabsf(seg_lo) + fabsf(seg_hi)) + 1e-6f;
  const float lo_s = seg_lo - slack, hi_s = seg_hi + slack;
  int sp = 1;
  if (lane == 0) M.stk[0] = 0;
  __syncwarp();
  while (sp > 0) {
    const int node = M.stk[sp - 1];
    --sp;
    if (lane == 0) cnt.nodes++;
    const WideNode& W = S.wide[node];
    const int child = __ldg(&W.child[lane]);
    float tn, tf;
    box_t(__ldg(&W.lox[lane]), __ldg(&W.loy[lane]), __ldg(&W.loz[lane]), __ldg(&W.hix[lane]),
          __ldg(&W.hiy[lane]), __ldg(&W.hiz[lane]), R.inv, R.oinv, tn, tf);
    const bool hit = child != kWideEmpty && tn <= tf && tf >= lo_s && tn <= hi_s &&
                     tn <= te_lim + slack;
    bool cand = false;
    unsigned long long ck = ~0ull;
    uint32_t cp = 0;
    if (hit && child < 0) {
      cp = (uint32_t)(~child);
      const float4* gp = S.geom + 4 * (size_t)cp;
      const float4 g0 = __ldg(gp), g1 = __ldg(gp + 1), g2 = __ldg(gp + 2), g3 = __ldg(gp + 3);
      PairGeom pg;
      if (isect_exact(g0, g1, g2, g3, R.o, R.d, pg) && pg.tx >= seg_lo && pg.te <= seg_hi) {
        ck = ((unsigned long long)fkey(pg.te) << 32) | (uint32_t)__float_as_int(g3.z);
        cand = ck > cursor && ck < kth;
      }
    }
    // internal children: push sorted so that the nearest is on top
    const unsigned im = __ballot_sync(kFull, hit && child >= 0);
    if (im) {
      int rank = 0;
      unsigned mm = im;
      while (mm) {
        const int b = __ffs(mm) - 1;
        mm &= mm - 1;
        const float tb = __shfl_sync(kFull, tn, b);
        rank += (tb > tn) || (tb == tn && b < (int)lane);
      }
      const int np = __popc(im);
      __syncwarp();
      if (sp + np <= kStk) {
        if (hit && child >= 0) M.stk[sp + rank] = child;
        sp += np;
      } else if (lane == 0) {
        cnt.stackov++;
      }
      __syncwarp();
    }
    // leaf candidates: rank-merge into the per-lane sorted k-buffer
    const unsigned cm = __ballot_sync(kFull, cand);
    if (cm) {
      int crank = 0, shift = 0, krank = 0;
      unsigned mm = cm;
      while (mm) {
        const int b = __ffs(mm) - 1;
        mm &= mm - 1;
        const unsigned long long kb = shfl64(ck, b);
        crank += (cand && kb < ck) ? 1 : 0;
        shift += (kb < key) ? 1 : 0;
        const unsigned ltm = __ballot_sync(kFull, key < kb);
        if ((int)lane == b) krank = __popc(ltm);
      }
      const int newk = (int)lane + shift, newc = krank + crank;
      if ((int)lane < nk && newk < kmax) { M.kscr[newk] = key; M.pscr[newk] = pos; }
      if (cand && newc < kmax) { M.kscr[newc] = ck; M.pscr[newc] = cp; }
      __syncwarp();
      nk = min(kmax, nk + __popc(cm));
      key = ((int)lane < nk) ? M.kscr[lane] : ~0ull;
      pos = ((int)lane < nk) ? M.pscr[lane] : 0u;
      __syncwarp();
      if (nk == kmax) {
        kth = shfl64(key, kmax - 1);
        te_lim = fkey_inv((uint32_t)(kth >> 32));
      }
    }
    (void)lt_mask;
  }
  return nk;
}

__device__ __forceinline__ float3 pair_color(const SceneView& S, int pos, const float3& d) {
  float Y[16];
  sh_basis(S.deg, d.x, d.y, d.z, Y);
  const float* ap = S.app + (size_t)pos * S.app_stride;
  const int nc = (S.deg + 1) * (S.deg + 1);
  float r = 0.f, g = 0.f, b = 0.f;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    if (m < nc) {
      r = fmaf(Y[m], __ldg(ap + 3 * m), r);
      g = fmaf(Y[m], __ldg(ap + 3 * m + 1), g);
      b = fmaf(Y[m], __ldg(ap + 3 * m + 2), b);
    }
  }
  const float* lp = ap + 3 * nc;
#pragma unroll
  for (int j = 0; j < kMaxLobes; ++j) {
    if (j < S.lobes) {
      const float* q = lp + 7 * j;
      const float dp = d.x * __ldg(q + 4) + d.y * __ldg(q + 5) + d.z * __ldg(q + 6);
      const float e = ex2_approx(__ldg(q + 3) * (dp - 1.0f) * kLog2e);
      r = fmaf(__ldg(q), e, r);
      g = fmaf(__ldg(q + 1), e, g);
      b = fmaf(__ldg(q + 2), e, b);
    }
  }
  return make_float3(r, g, b);
}

// Per-(ray, Gaussian) set-up into slot `sl`: exact interval and the exponent
// polynomial of w(tau) = sigma~ exp(-|u + tau d_l|^2 / 2) = 2^(c0 + tau (c1 + c2 tau)),
// tau = t - t_mid, u = M x' from the compensated offset x' (value path).
__device__ void setup_pair(const SceneView& S, WarpMem& M, int sl, const Ray& R,
                           unsigned long long key, uint32_t pos) {
  const float4* gp = S.geom + 4 * (size_t)pos;
  const float4 g0 = __ldg(gp), g1 = __ldg(gp + 1), g2 = __ldg(gp + 2), g3 = __ldg(gp + 3);
  PairGeom pg;
  isect_exact(g0, g1, g2, g3, R.o, R.d, pg);
  const float x0 = offset_at(R.o.x, g0.x, pg.tm, R.d.x);
  const float x1 = offset_at(R.o.y, g0.y, pg.tm, R.d.y);
  const float x2 = offset_at(R.o.z, g0.z, pg.tm, R.d.z);
  const float u0 = g1.x * x0 + g1.y * x1 + g1.z * x2;
  const float u1 = g1.w * x0 + g2.x * x1 + g2.y * x2;
  const float u2 = g2.z * x0 + g2.w * x1 + g3.x * x2;
  const float qm = u0 * u0 + u1 * u1 + u2 * u2;
  const float b1 = u0 * pg.dl0 + u1 * pg.dl1 + u2 * pg.dl2;
  const float3 col = pair_color(S, (int)pos, R.d);
  M.te[sl] = pg.te;
  M.tx[sl] = pg.tx;
  M.tm[sl] = pg.tm;
  M.c0[sl] = lg2_approx(g0.w) - 0.5f * kLog2e * qm;
  M.c1[sl] = -kLog2e * b1;
  M.c2[sl] = -0.5f * kLog2e * pg.A;
  M.cr[sl] = col.x;
  M.cg[sl] = col.y;
  M.cb[sl] = col.z;
  M.pos[sl] = (int)pos;
  M.idx[sl] = (uint32_t)(key & 0xFFFFFFFFu);
}

// 1 - exp(-x) without cancellation for small x
__device__ __forceinline__ float alpha_of(float x, float e) {
  if (x < 0.0625f) return x * (1.f - 0.5f * x * (1.f - (1.f / 3.f) * x * (1.f - 0.25f * x)));
  return 1.0f - e;
}

struct Lanes {   // lane -> (entry subset, sample) mapping for one sample group
  int GW, ER, j, esub;
};

// sigma and sigma*c at this lane's sample from slots [e0, e1)
__device__ __forceinline__ void eval_range(const WarpMem& M, int e0, int e1, const Lanes& L, float tk,
                                           bool val, float& s, float& r, float& g, float& b,
                                           uint32_t& evals) {
  for (int e = e0 + L.esub; e < e1; e += L.ER) {
    const float te = M.te[e], tx = M.tx[e];
    if (val && te <= tk && tk <= tx) {
      const float tau = tk - M.tm[e];
      const float w = ex2_approx(fmaf(tau, fmaf(M.c2[e], tau, M.c1[e]), M.c0[e]));
      s += w;
      r = fmaf(w, M.cr[e], r);
      g = fmaf(w, M.cg[e], g);
      b = fmaf(w, M.cb[e], b);
      ++evals;
    }
  }
}

struct SampleGrad {   // per-sample backward quantities (lane j of the group)
  float dls, dc0, dc1, dc2, gc, inv;
};

// accumulate the per-pair moments of slots [e0, e1) for this group's samples
__device__ __forceinline__ void grad_range(const WarpMem& M, WarpAcc& A, int e0, int e1,
                                           const Lanes& L, float tk, bool live,
                                           const SampleGrad& H) {
  const int rounds = (e1 - e0 + L.ER - 1) / L.ER;
  for (int r = 0; r < rounds; ++r) {
    const int e = e0 + L.esub + r * L.ER;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f, a5 = 0.f;
    if (e < e1 && live && M.te[e] <= tk && tk <= M.tx[e]) {
      const float tau = tk - M.tm[e];
      const float w = ex2_approx(fmaf(tau, fmaf(M.c2[e], tau, M.c1[e]), M.c0[e]));
      const float dldw = H.dls + (H.dc0 * M.cr[e] + H.dc1 * M.cg[e] + H.dc2 * M.cb[e] - H.gc) * H.inv;
      const float wd = w * dldw, wi = w * H.inv;
      a0 = wd;
      a1 = wd * tau;
      a2 = wd * tau * tau;
      a3 = wi * H.dc0;
      a4 = wi * H.dc1;
      a5 = wi * H.dc2;
    }
    for (int off = 1; off < L.GW; off <<= 1) {
      a0 += __shfl_xor_sync(kFull, a0, off);
      a1 += __shfl_xor_sync(kFull, a1, off);
      a2 += __shfl_xor_sync(kFull, a2, off);
      a3 += __shfl_xor_sync(kFull, a3, off);
      a4 += __shfl_xor_sync(kFull, a4, off);
      a5 += __shfl_xor_sync(kFull, a5, off);
    }
    if (L.j == 0 && e < e1) {
      A.a[0][e] += a0; A.a[1][e] += a1; A.a[2][e] += a2;
      A.a[3][e] += a3; A.a[4][e] += a4; A.a[5][e] += a5;
    }
  }
  __syncwarp();
}

// Warp-cooperative gradient scatter of slot `e` (lane c writes float4 chunk c):
//  chunk 0 = (dL/dmu, dL/dsigma~), chunks 1-3 = dL/dM (9 + pad), chunks 4.. = appearance.
//  With x = x' + tau d, u = M x', d_l = M d and Sw = sum w dL/dw, Sw1 = sum w dL/dw tau,
//  Sw2 = sum w dL/dw tau^2:  dL/dmu = M^T (Sw u + Sw1 d_l),
//  dL/dM = -(Sw u x'^T + Sw1 (u d^T + d_l x'^T) + Sw2 d_l d^T),  dL/dsigma~ = Sw / sigma~.
__device__ void scatter_slot(const SceneView& S, const WarpMem& M, const WarpAcc& A, int e,
                             const Ray& R, float* gbuf, int gstride) {
  const float Sw = A.a[0][e], Sw1 = A.a[1][e], Sw2 = A.a[2][e];
  const float d0 = A.a[3][e], d1 = A.a[4][e], d2 = A.a[5][e];
  if (Sw == 0.f && Sw1 == 0.f && Sw2 == 0.f && d0 == 0.f && d1 == 0.f && d2 == 0.f) return;
  const int c = (int)lane_id();
  const int pos = M.pos[e];
  const int nchunks = 4 + S.app_stride / 4;
  float v[4] = {0.f, 0.f, 0.f, 0.f};
  if (c < 4) {
    const float4* gp = S.geom + 4 * (size_t)pos;
    const float4 g0 = __ldg(gp), g1 = __ldg(gp + 1), g2 = __ldg(gp + 2), g3 = __ldg(gp + 3);
    const float Mm[9] = {g1.x, g1.y, g1.z, g1.w, g2.x, g2.y, g2.z, g2.w, g3.x};
    const float tm = M.tm[e];
    const float xp[3] = {offset_at(R.o.x, g0.x, tm, R.d.x), offset_at(R.o.y, g0.y, tm, R.d.y),
                         offset_at(R.o.z, g0.z, tm, R.d.z)};
    const float dv[3] = {R.d.x, R.d.y, R.d.z};
    float u[3], dl[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      u[r] = Mm[3 * r] * xp[0] + Mm[3 * r + 1] * xp[1] + Mm[3 * r + 2] * xp[2];
      dl[r] = Mm[3 * r] * dv[0] + Mm[3 * r + 1] * dv[1] + Mm[3 * r + 2] * dv[2];
    }
    float out[16];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      float acc = 0.f;
#pragma unroll
      for (int r = 0; r < 3; ++r) acc += Mm[3 * r + b] * (Sw * u[r] + Sw1 * dl[r]);
      out[b] = acc;
    }
    out[3] = Sw / g0.w;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int b = 0; b < 3; ++b)
        out[4 + 3 * r + b] = -(Sw * u[r] * xp[b] + Sw1 * (u[r] * dv[b] + dl[r] * xp[b]) +
                               Sw2 * dl[r] * dv[b]);
    out[13] = out[14] = out[15] = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = out[4 * c + k];
  } else if (c < nchunks) {
    const int nc = (S.deg + 1) * (S.deg + 1);
    const float dc[3] = {d0, d1, d2};
    const float* ap = S.app + (size_t)pos * S.app_stride + 3 * nc;
    int lobe_cached = -1;
    float e_j = 0.f, kd = 0.f, dp = 0.f, lam = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int f = 4 * (c - 4) + k;
      if (f < 3 * nc) {
        v[k] = dc[f % 3] * M.Y[f / 3];
      } else if (f < 3 * nc + 7 * S.lobes) {
        const int j = (f - 3 * nc) / 7, rr = (f - 3 * nc) % 7;
        if (j != lobe_cached) {
          const float* q = ap + 7 * j;
          lam = __ldg(q + 3);
          dp = R.d.x * __ldg(q + 4) + R.d.y * __ldg(q + 5) + R.d.z * __ldg(q + 6);
          e_j = ex2_approx(lam * (dp - 1.0f) * kLog2e);
          kd = (d0 * __ldg(q) + d1 * __ldg(q + 1) + d2 * __ldg(q + 2)) * e_j;
          lobe_cached = j;
        }
        if (rr < 3) v[k] = dc[rr] * e_j;
        else if (rr == 3) v[k] = kd * (dp - 1.0f);
        else v[k] = kd * lam * (rr == 4 ? R.d.x : (rr == 5 ? R.d.y : R.d.z));
      }
    }
  }
  if (c < nchunks)
    atomicAdd(reinterpret_cast<float4*>(gbuf + (size_t)pos * gstride) + c,
              make_float4(v[0], v[1], v[2], v[3]));
}

__device__ __forceinline__ int skip_to(float te, int s, int B, float dt, float t0, float t1) {
  int est = (int)((te - t0) / ((float)B * dt));
  if (est < s + 1) est = s + 1;
  while (fminf(t1, fma_((float)((est + 1) * B), dt, t0)) < te) ++est;
  while (est > s + 1 && fminf(t1, fma_((float)(est * B), dt, t0)) >= te) --est;
  return est;
}

__device__ __forceinline__ void flush_stats(rg_stats* st, const Counters& c, bool hit) {
  const unsigned lane = lane_id();
  const uint32_t v[10] = {lane == 0 ? 1u : 0u, (lane == 0 && hit) ? 1u : 0u, c.slabs, c.pairs,
                          c.evals, c.samples, c.overflows, c.fetches, c.nodes, c.stackov};
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(st);
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    const uint32_t s = __reduce_add_sync(kFull, v[k]);
    if (lane == 0 && s) atomicAdd(dst + k, (unsigned long long)s);
  }
}

// Kahan accumulation
__device__ __forceinline__ void kadd(float& s, float& comp, float x) {
  const float y = x - comp;
  const float t = s + y;
  comp = (t - s) - y;
  s = t;
}

template <bool BWD>
__global__ void __launch_bounds__(kBlock, 4) k_render(const RenderArgs P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const unsigned lane = lane_id();
  const int wid = threadIdx.x >> 5;
  WarpMem& M = reinterpret_cast<WarpMem*>(smem_raw)[wid];
  WarpAcc& A = reinterpret_cast<WarpAcc*>(smem_raw + sizeof(WarpMem) * kWarps)[BWD ? wid : 0];
  int ray;
  Ray R;
  if (P.cam_mode) {
    const int tile = blockIdx.x;
    const int px = 2 * (tile % P.tiles_x) + (wid & 1);
    const int py = 2 * (tile / P.tiles_x) + (wid >> 1);
    if (px >= P.rw || py >= P.rh) return;
    ray = py * P.rw + px;
    camera_ray(P.cam, P.cam.x0 + px, P.cam.y0 + py, R.o, R.d);
  } else {
    ray = blockIdx.x * kWarps + wid;
    if (ray >= P.n_rays) return;
    R.o = make_float3(P.ro[3 * ray], P.ro[3 * ray + 1], P.ro[3 * ray + 2]);
    R.d = make_float3(P.rd[3 * ray], P.rd[3 * ray + 1], P.rd[3 * ray + 2]);
  }
  const rg_config& c = P.c;
  const int B = c.slab_samples;
  const int K = c.hit_capacity;
  float C0 = 0.f, C1 = 0.f, C2 = 0.f, k0c = 0.f, k1c = 0.f, k2c = 0.f;
  float tau = 0.f, tauc = 0.f, T = 1.f;
  int replay = -1;
  Counters cnt = {};
  const bool dbg = (!BWD) && P.dbg_rec != nullptr && ray < P.dbg_rays;
  int dbg_n = 0;
  float gr0 = 0.f, gr1 = 0.f, gr2 = 0.f, Pp0 = 0.f, Pp1 = 0.f, Pp2 = 0.f;
  int replay_in = -1;
  if (BWD) {
    gr0 = P.d_rgb[3 * ray]; gr1 = P.d_rgb[3 * ray + 1]; gr2 = P.d_rgb[3 * ray + 2];
    Pp0 = P.rgb_in[3 * ray]; Pp1 = P.rgb_in[3 * ray + 1]; Pp2 = P.rgb_in[3 * ray + 2];
    replay_in = P.replay_in[ray];
  }
  float t0 = 0.f, t1 = 0.f;
  const bool hit = P.S.n > 0 && clip_exact(P.S.root_box, R.o, R.d, c.t_near, t0, t1);
  if (hit && !(BWD && gr0 == 0.f && gr1 == 0.f && gr2 == 0.f)) {
    R.inv = make_float3(1.0f / R.d.x, 1.0f / R.d.y, 1.0f / R.d.z);
    R.oinv = make_float3(R.o.x * R.inv.x, R.o.y * R.inv.y, R.o.z * R.inv.z);
    if (BWD) {
      float Y[16];
      sh_basis(P.S.deg, R.d.x, R.d.y, R.d.z, Y);
      if (lane < 16) {
#pragma unroll
        for (int m = 0; m < 16; ++m)
          if ((int)lane == m) M.Y[m] = Y[m];
      }
      __syncwarp();
    }
    // lane mapping for sample groups
    Lanes L;
    L.GW = B >= 8 ? 8 : (B >= 4 ? 4 : (B >= 2 ? 2 : 1));
    if (B == 3) L.GW = 4;
    if (B > 4 && B < 8) L.GW = 8;
    L.ER = 32 / L.GW;
    L.j = (int)lane % L.GW;
    L.esub = (int)lane / L.GW;
    int count = 0;
    unsigned long long cursor = 0;
    bool exhausted = false;
    int s = 0;
    while (true) {
      const int k0 = s * B;
      if (!(sample_t(k0, c.dt, t0) < t1)) break;
      const float tlo = fma_((float)k0, c.dt, t0);
      const float thi = fminf(t1, fma_((float)(k0 + B), c.dt, t0));
      // ---- expire Gaussians whose support ended before this slab
      {
        int nc = 0;
        for (int base = 0; base < count; base += 32) {
          const int e = base + (int)lane;
          const bool valid = e < count;
          const bool keep = valid && M.tx[e] >= tlo;
          if (BWD) {
            unsigned xm = __ballot_sync(kFull, valid && !keep);
            while (xm) {
              const int b = __ffs(xm) - 1;
              xm &= xm - 1;
              scatter_slot(P.S, M, A, base + b, R, P.gbuf, P.gstride);
            }
          }
          float f[9];
          int ps = 0;
          uint32_t ix = 0;
          float ac[6];
          if (keep) {
            f[0] = M.te[e]; f[1] = M.tx[e]; f[2] = M.tm[e]; f[3] = M.c0[e]; f[4] = M.c1[e];
            f[5] = M.c2[e]; f[6] = M.cr[e]; f[7] = M.cg[e]; f[8] = M.cb[e];
            ps = M.pos[e]; ix = M.idx[e];
            if (BWD)
              for (int k = 0; k < 6; ++k) ac[k] = A.a[k][e];
          }
          const unsigned km = __ballot_sync(kFull, keep);
          const int dst = nc + __popc(km & ((1u << lane) - 1u));
          __syncwarp();
          if (keep) {
            M.te[dst] = f[0]; M.tx[dst] = f[1]; M.tm[dst] = f[2]; M.c0[dst] = f[3];
            M.c1[dst] = f[4]; M.c2[dst] = f[5]; M.cr[dst] = f[6]; M.cg[dst] = f[7];
            M.cb[dst] = f[8]; M.pos[dst] = ps; M.idx[dst] = ix;
            if (BWD)
              for (int k = 0; k < 6; ++k) A.a[k][dst] = ac[k];
          }
          nc += __popc(km);
          __syncwarp();
        }
        count = nc;
      }
      // ---- refill in key order until every Gaussian entering by t_hi is held
      while (!exhausted && count < kA && (count == 0 || M.te[count - 1] <= thi)) {
        const int want = min(32, kA - count);
        unsigned long long key;
        uint32_t pos;
        const int got = fetch(P.S, M, R, tlo, t1, cursor, want, key, pos, cnt);
        if ((int)lane < got) {
          setup_pair(P.S, M, count + (int)lane, R, key, pos);
          if (BWD)
            for (int k = 0; k < 6; ++k) A.a[k][count + lane] = 0.f;
        }
        if (lane == 0) cnt.pairs += got;
        if (got > 0) cursor = shfl64(key, got - 1);
        count += got;
        if (got < want) exhausted = true;
        __syncwarp();
      }
      if (count == 0) break;
      if (M.te[0] > thi) {   // empty slab(s): jump to the slab holding the next entry
        s = skip_to(M.te[0], s, B, c.dt, t0, t1);
        continue;
      }
      int n_in = 0;
      for (int base = 0; base < count; base += 32) {
        const int e = base + (int)lane;
        const unsigned m = __ballot_sync(kFull, e < count && M.te[e] <= thi);
        n_in += __popc(m);
        if (m != kFull) break;
      }
      const int n_use = min(n_in, K);
      const bool more = (n_in == kA) && !exhausted && (K > kA);
      if (n_in > K) {
        if (lane == 0) cnt.overflows++;
      } else if (!BWD && n_in == K && n_in == kA && !exhausted) {
        unsigned long long pk;
        uint32_t pp;
        if (fetch(P.S, M, R, tlo, thi, cursor, 1, pk, pp, cnt) > 0 && lane == 0) cnt.overflows++;
      }
      if (dbg) {
        for (int e = (int)lane; e < n_use; e += 32)
          if (dbg_n + e < P.dbg_cap) {
            int32_t* r = P.dbg_rec + 2 * ((size_t)ray * P.dbg_cap + dbg_n + e);
            r[0] = s;
            r[1] = (int32_t)M.idx[e];
          }
        dbg_n = min(P.dbg_cap, dbg_n + n_use);
      }
      for (int g0 = 0; g0 < B; g0 += L.GW) {
        const float tk = sample_t(k0 + g0 + L.j, c.dt, t0);
        const bool val = (g0 + L.j < B) && (tk < t1);
        float sg = 0.f, sr = 0.f, sgg = 0.f, sb = 0.f;
        uint32_t ev = 0;
        eval_range(M, 0, n_use, L, tk, val, sg, sr, sgg, sb, ev);
        if (more) {   // slab set larger than the active list: stream the rest
          unsigned long long cur2 = cursor;
          int remaining = K - n_use;
          bool full_last = true;
          while (remaining > 0) {
            const int want = min(32, remaining);
            unsigned long long key;
            uint32_t pos;
            const int got = fetch(P.S, M, R, tlo, thi, cur2, want, key, pos, cnt);
            if ((int)lane < got) setup_pair(P.S, M, kA + (int)lane, R, key, pos);
            __syncwarp();
            eval_range(M, kA, kA + got, L, tk, val, sg, sr, sgg, sb, ev);
            if (dbg && g0 == 0) {
              if ((int)lane < got && dbg_n + (int)lane < P.dbg_cap) {
                int32_t* r = P.dbg_rec + 2 * ((size_t)ray * P.dbg_cap + dbg_n + lane);
                r[0] = s;
                r[1] = (int32_t)M.idx[kA + lane];
              }
              dbg_n = min(P.dbg_cap, dbg_n + got);
            }
            if (g0 == 0 && lane == 0) cnt.pairs += got;
            remaining -= got;
            if (got > 0) cur2 = shfl64(key, got - 1);
            __syncwarp();
            if (got < want) { full_last = false; break; }
          }
          if (g0 == 0 && remaining == 0 && full_last) {
            unsigned long long pk;
            uint32_t pp;
            if (fetch(P.S, M, R, tlo, thi, cur2, 1, pk, pp, cnt) > 0 && lane == 0) cnt.overflows++;
          }
        }
        cnt.evals += ev;
        // reduce over the entry subsets: every lane of sample j holds the totals
        for (int off = L.GW; off < 32; off <<= 1) {
          sg += __shfl_xor_sync(kFull, sg, off);
          sr += __shfl_xor_sync(kFull, sr, off);
          sgg += __shfl_xor_sync(kFull, sgg, off);
          sb += __shfl_xor_sync(kFull, sb, off);
        }
        // ---- composite the group front to back (Eq. 4): segmented scans over GW lanes
        const bool live = val && sg > 0.f;
        const float x = live ? sg * c.dt : 0.f;
        float incl = x;
        for (int dd = 1; dd < L.GW; dd <<= 1) {
          const float v = __shfl_up_sync(kFull, incl, dd, L.GW);
          if (L.j >= dd) incl += v;
        }
        const float excl = incl - x;
        const float Tb = ex2_approx(-(tau + excl) * kLog2e);   // T before this sample
        const float e_s = ex2_approx(-x * kLog2e);
        const float al = alpha_of(x, e_s);
        const float inv_s = live ? 1.0f / sg : 0.f;
        const float cr = sr * inv_s, cg = sgg * inv_s, cb = sb * inv_s;
        const float wgt = live ? Tb * al : 0.f;
        float q0 = wgt * cr, q1 = wgt * cg, q2 = wgt * cb;
        // inclusive prefix of the contributions (backward needs C after each sample)
        float p0 = q0, p1 = q1, p2 = q2;
        for (int dd = 1; dd < L.GW; dd <<= 1) {
          const float v0 = __shfl_up_sync(kFull, p0, dd, L.GW);
          const float v1 = __shfl_up_sync(kFull, p1, dd, L.GW);
          const float v2 = __shfl_up_sync(kFull, p2, dd, L.GW);
          if (L.j >= dd) { p0 += v0; p1 += v1; p2 += v2; }
        }
        SampleGrad H = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (BWD && live) {
          const float Ta = Tb * e_s;
          H.dc0 = gr0 * wgt; H.dc1 = gr1 * wgt; H.dc2 = gr2 * wgt;
          const float gcj = gr0 * cr + gr1 * cg + gr2 * cb;
          const float gS = gr0 * (Pp0 - (C0 + p0)) + gr1 * (Pp1 - (C1 + p1)) + gr2 * (Pp2 - (C2 + p2));
          H.dls = c.dt * (Ta * gcj - gS);
          H.gc = H.dc0 * cr + H.dc1 * cg + H.dc2 * cb;
          H.inv = inv_s;
        }
        const int last = L.GW - 1;
        const float tot_x = __shfl_sync(kFull, incl, last, L.GW);
        const float t0c = __shfl_sync(kFull, p0, last, L.GW);
        const float t1c = __shfl_sync(kFull, p1, last, L.GW);
        const float t2c = __shfl_sync(kFull, p2, last, L.GW);
        kadd(tau, tauc, tot_x);
        kadd(C0, k0c, t0c);
        kadd(C1, k1c, t1c);
        kadd(C2, k2c, t2c);
        T = ex2_approx(-tau * kLog2e);
        const unsigned smask = __ballot_sync(kFull, live && L.esub == 0);
        if (lane == 0) cnt.samples += __popc(smask);
        if (BWD) {
          grad_range(M, A, 0, n_use, L, tk, live, H);
          if (more) {
            unsigned long long cur2 = cursor;
            int remaining = K - n_use;
            while (remaining > 0) {
              const int want = min(32, remaining);
              unsigned long long key;
              uint32_t pos;
              const int got = fetch(P.S, M, R, tlo, thi, cur2, want, key, pos, cnt);
              if ((int)lane < got) {
                setup_pair(P.S, M, kA + (int)lane, R, key, pos);
                for (int k = 0; k < 6; ++k) A.a[k][kA + lane] = 0.f;
              }
              __syncwarp();
              grad_range(M, A, kA, kA + got, L, tk, live, H);
              for (int e = kA; e < kA + got; ++e) scatter_slot(P.S, M, A, e, R, P.gbuf, P.gstride);
              remaining -= got;
              if (got > 0) cur2 = shfl64(key, got - 1);
              __syncwarp();
              if (got < want) break;
            }
          }
        }
      }
      if (lane == 0) cnt.slabs++;
      if (BWD) {
        if (s == replay_in) break;
      } else if (T <= c.t_eps) {
        replay = s;
        break;
      }
      ++s;
    }
    if (BWD)
      for (int e = 0; e < count; ++e) scatter_slot(P.S, M, A, e, R, P.gbuf, P.gstride);
  }
  if (!BWD && lane == 0) {
    P.rgb[3 * ray] = C0 + T * c.background[0];
    P.rgb[3 * ray + 1] = C1 + T * c.background[1];
    P.rgb[3 * ray + 2] = C2 + T * c.background[2];
    P.T[ray] = T;
    P.replay[ray] = replay;
    if (P.dbg_counts && ray < P.dbg_rays) P.dbg_counts[ray] = dbg_n;
  }
  if (P.stats) flush_stats(P.stats, cnt, hit);
}

// (mu, M) -> (mu, q, s) and Morton -> caller order
__global__ void __launch_bounds__(256) k_finalize(const float* gbuf, int gstride,
                                                  const uint32_t* order, rg_gaussians g,
                                                  rg_gaussian_grads out, rg_stats* stats) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= g.n) return;
  const int i = (int)order[p];
  const float* row = gbuf + (size_t)p * gstride;
  const float* q = g.quat + 4 * (size_t)i;
  const float* s = g.scale + 3 * (size_t)i;
  const float w = q[0], x = q[1], y = q[2], z = q[3];
  const float R[9] = {1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y),
                      2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x),
                      2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)};
  float dR[9];
  float ds[3];
  for (int a = 0; a < 3; ++a) {
    ds[a] = 0.f;
    for (int b = 0; b < 3; ++b) {
      const float dM = row[4 + 3 * a + b];   // M_ab = R_ba / s_a
      ds[a] -= dM * R[3 * b + a] / (s[a] * s[a]);
      dR[3 * b + a] = dM / s[a];
    }
  }
  // d R / d q (polynomial ARITH-1 differentiated)
  float dq[4];
  dq[0] = dR[1] * (-2 * z) + dR[2] * (2 * y) + dR[3] * (2 * z) + dR[5] * (-2 * x) +
          dR[6] * (-2 * y) + dR[7] * (2 * x);
  dq[1] = dR[1] * (2 * y) + dR[2] * (2 * z) + dR[3] * (2 * y) + dR[4] * (-4 * x) +
          dR[5] * (-2 * w) + dR[6] * (2 * z) + dR[7] * (2 * w) + dR[8] * (-4 * x);
  dq[2] = dR[0] * (-4 * y) + dR[1] * (2 * x) + dR[2] * (2 * w) + dR[3] * (2 * x) +
          dR[5] * (2 * z) + dR[6] * (-2 * w) + dR[7] * (2 * z) + dR[8] * (-4 * y);
  dq[3] = dR[0] * (-4 * z) + dR[1] * (-2 * w) + dR[2] * (2 * x) + dR[3] * (2 * w) +
          dR[4] * (-4 * z) + dR[5] * (2 * y) + dR[6] * (2 * x) + dR[7] * (2 * y);
  uint32_t bad = 0;
  auto put = [&](float* base, size_t k, float v) {
    if (!isfinite(v)) ++bad;
    if (base) base[k] += v;
  };
  for (int a = 0; a < 3; ++a) put(out.mean, 3 * (size_t)i + a, row[a]);
  put(out.density, i, row[3]);
  for (int a = 0; a < 3; ++a) put(out.scale, 3 * (size_t)i + a, ds[a]);
  for (int a = 0; a < 4; ++a) put(out.quat, 4 * (size_t)i + a, dq[a]);
  const int nc = (g.sh_degree + 1) * (g.sh_degree + 1);
  const float* ap = row + 16;
  for (int k = 0; k < 3 * nc; ++k) put(out.sh, (size_t)i * 3 * nc + k, ap[k]);
  for (int j = 0; j < g.sg_count; ++j) {
    const float* v = ap + 3 * nc + 7 * j;
    const size_t ij = (size_t)i * g.sg_count + j;
    for (int a = 0; a < 3; ++a) put(out.sg_amp, 3 * ij + a, v[a]);
    put(out.sg_sharp, ij, v[3]);
    for (int a = 0; a < 3; ++a) put(out.sg_axis, 3 * ij + a, v[4 + a]);
  }
  if (bad && stats) atomicAdd(&stats->nonfinite_grads, (unsigned long long)bad);
}

__global__ void k_camera_rays(const rg_camera cam, float* o, float* d) {
  const int rw = cam.x1 - cam.x0, rh = cam.y1 - cam.y0;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rw * rh) return;
  float3 oo, dd;
  camera_ray(cam, cam.x0 + r % rw, cam.y0 + r / rw, oo, dd);
  o[3 * r] = oo.x; o[3 * r + 1] = oo.y; o[3 * r + 2] = oo.z;
  d[3 * r] = dd.x; d[3 * r + 1] = dd.y; d[3 * r + 2] = dd.z;
}

__global__ void k_l1(const float* a, const float* b, int64_t n, float scale, float* g,
                     float* loss) {
  float acc = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float diff = a[i] - b[i];
    g[i] = diff > 0.f ? scale : (diff < 0.f ? -scale : 0.f);
    acc += fabsf(diff);
  }
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) atomicAdd(loss, acc * scale);
}

SceneView view_of(const rg_bvh& b) {
  SceneView S;
  S.geom = reinterpret_cast<const float4*>(b.geom);
  S.app = b.app;
  S.nodes = reinterpret_cast<const float4*>(b.nodes);
  S.wide = reinterpret_cast<const WideNode*>(b.wide);
  S.root_box = b.root_box;
  S.n = b.n;
  S.deg = b.sh_degree;
  S.lobes = b.sg_count;
  S.app_stride = b.app_stride;
  return S;
}

void ray_grid(RenderArgs& A, const rg_rays* rays, const rg_camera* cam, dim3& grid) {
  if (cam) {
    A.cam_mode = 1;
    A.cam = *cam;
    A.rw = cam->x1 - cam->x0;
    A.rh = cam->y1 - cam->y0;
    A.n_rays = A.rw * A.rh;
    A.tiles_x = (A.rw + 1) / 2;
    grid = dim3((unsigned)(A.tiles_x * ((A.rh + 1) / 2)));
  } else {
    A.cam_mode = 0;
    A.ro = rays->origin;
    A.rd = rays->dir;
    A.n_rays = rays->n;
    grid = dim3((unsigned)((rays->n + kWarps - 1) / kWarps));
  }
}

constexpr size_t kSmemFwd = sizeof(WarpMem) * kWarps;
constexpr size_t kSmemBwd = (sizeof(WarpMem) + sizeof(WarpAcc)) * kWarps;

}  // namespace

cudaError_t launch_camera_rays(const rg_camera& cam, float* o, float* d, cudaStream_t st) {
  const int n = (cam.x1 - cam.x0) * (cam.y1 - cam.y0);
  if (n > 0) { k_camera_rays<<<(n + 255) / 256, 256, 0, st>>>(cam, o, d); count_launches(1); }
  return cudaGetLastError();
}

cudaError_t launch_forward(const rg_gaussians& g, const rg_bvh& b, const rg_config& c,
                           const rg_rays* rays, const rg_camera* cam, float* rgb, float* T,
                           int32_t* replay, rg_stats* stats, int dbg_rays, int dbg_cap,
                           int32_t* dbg_counts, int32_t* dbg_rec, cudaStream_t st) {
  (void)g;
  RenderArgs A = {};
  A.S = view_of(b);
  A.c = c;
  dim3 grid;
  ray_grid(A, rays, cam, grid);
  if (A.n_rays == 0) return cudaSuccess;
  A.rgb = rgb; A.T = T; A.replay = replay; A.stats = stats;
  A.dbg_rays = dbg_rec ? dbg_rays : 0;
  A.dbg_cap = dbg_cap; A.dbg_counts = dbg_counts; A.dbg_rec = dbg_rec;
  k_render<false><<<grid, kBlock, kSmemFwd, st>>>(A);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_backward(const rg_gaussians& g, const rg_bvh& b, const rg_config& c,
                            const rg_rays* rays, const rg_camera* cam, const float* rgb,
                            const float* T, const int32_t* replay, const float* d_rgb,
                            const rg_gaussian_grads& grads, rg_stats* stats, float* gbuf,
                            cudaStream_t st) {
  (void)T;
  RenderArgs A = {};
  A.S = view_of(b);
  A.c = c;
  dim3 grid;
  ray_grid(A, rays, cam, grid);
  const int gs = grad_stride(b.sh_degree, b.sg_count);
  if (b.n > 0) cudaMemsetAsync(gbuf, 0, sizeof(float) * (size_t)gs * b.n, st);
  A.stats = stats;
  A.rgb_in = rgb; A.replay_in = replay; A.d_rgb = d_rgb; A.gbuf = gbuf; A.gstride = gs;
  if (A.n_rays > 0) { k_render<true><<<grid, kBlock, kSmemBwd, st>>>(A); count_launches(1); }
  if (b.n > 0) {
    k_finalize<<<(b.n + 255) / 256, 256, 0, st>>>(gbuf, gs, b.order, g, grads, stats);
    count_launches(1);
  }
  return cudaGetLastError();
}

cudaError_t launch_l1(const float* rgb, const float* target, int64_t n, float scale, float* d_rgb,
                      float* loss, cudaStream_t st) {
  if (n > 0) {
    const int64_t nb = (n + 255) / 256; const int blocks = (int)(nb < 148 * 8 ? nb : 148 * 8);
    k_l1<<<blocks, 256, 0, st>>>(rgb, target, n, scale, d_rgb, loss);
    count_launches(1);
  }
  return cudaGetLastError();
}

}  // namespace rg
