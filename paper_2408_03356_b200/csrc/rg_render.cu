// rg_render.cu -- slab-by-slab volume ray casting of the Gaussians through the
// LBVH, forward and backward:
//
//   PAPER.md Alg. 2: per ray, bbox clip, then slabs of B samples
//   of length dt*B; per slab the set of Gaussians whose support overlaps the
//   slab (Alg. 1 any-hit collection, capped at K = n_max with the
//   K smallest (t_entry, index) kept -- DESIGN.md L7), sorted by entry depth;
//   UpdateRay = evaluate sigma and the density-weighted colour at the B
//   samples (Eq. 10-16) and composite front to back (Eq. 4); early
//   termination at slab granularity when T <= T_eps.
//
// B200 design: one thread per ray, 8x4-pixel warps; instead of
// a BVH traversal per slab, each ray keeps a sorted ACTIVE LIST (local memory,
// capacity kACap) of its upcoming/overlapping Gaussians, refilled by a
// k-nearest-by-t_entry traversal ("fetch the next k after a cursor") with a
// short stack; empty slabs are skipped exactly (jump to the slab holding the
// next t_entry).  Per-slab hit sets are reproduced bit for bit from the exact
// fp32 intervals.  Per-pair work (interval, colour, exponent coefficients) is
// done once per (ray, Gaussian) and reused across the slabs it spans.
// Backward replays the same march, recomputes each slab's samples, walks them
// front to back with suffix = P - prefix (L16), accumulates four per-pair
// moments and scatters 16 + app_stride floats per pair with float4 atomics
// into a Morton-ordered buffer; k_finalize converts (mu, M) -> (mu, q, s) and
// un-permutes to caller order.
#include "rg_internal.cuh"

namespace rg {

namespace {

constexpr int kBlock = 128;

struct Counters {
  uint32_t slabs, pairs, evals, samples, overflows, fetches, nodes, stackov;
};

struct RenderArgs {
  SceneView S;
  rg_config c;
  int cam_mode;
  rg_camera cam;
  int rw, rh;              // camera rect size
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

struct Entry {
  float te, tx, tm, c0, c1, c2, cr, cg, cb;
  int pos;
  uint32_t idx;
};

__device__ __forceinline__ float4 ldg4(const float4* p) { return __ldg(p); }

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

// Collect, in ascending (t_entry, index) key order, the `kmax` smallest keys
// > cursor among Gaussians whose exact support interval satisfies
// t_exit >= seg_lo and t_entry <= seg_hi.  Node pruning: segment overlap and,
// once kmax keys are held, box entry > current kmax-th t_entry.
__device__ int fetch(const SceneView& S, const float3& o, const float3& d, const float3& inv,
                     const float3& oinv, float seg_lo, float seg_hi, uint64_t cursor, int kmax,
                     uint64_t* hk, uint32_t* hp, Counters& cnt) {
  cnt.fetches++;
  int nb = 0;
  float te_lim = INFINITY;
  const float slack = 1e-5f * (fabsf(seg_lo) + fabsf(seg_hi)) + 1e-6f;
  const float lo_s = seg_lo - slack, hi_s = seg_hi + slack;
  int stk[kStack];
  int sp = 0;
  stk[sp++] = (S.n == 1) ? ~0 : 0;
  while (sp > 0) {
    const int id = stk[--sp];
    if (id >= 0) {
      cnt.nodes++;
      const float4* np = S.nodes + 4 * (size_t)id;
      const float4 a = ldg4(np), b = ldg4(np + 1), c = ldg4(np + 2), e = ldg4(np + 3);
      float ln, lf, rn, rf;
      box_t(a.x, a.y, a.z, a.w, b.x, b.y, inv, oinv, ln, lf);
      box_t(b.z, b.w, c.x, c.y, c.z, c.w, inv, oinv, rn, rf);
      const float lim = te_lim + slack;
      const bool hl = ln <= lf && lf >= lo_s && ln <= hi_s && ln <= lim;
      const bool hr = rn <= rf && rf >= lo_s && rn <= hi_s && rn <= lim;
      const int cl = __float_as_int(e.x), cr = __float_as_int(e.y);
      if (hl && hr) {
        if (sp + 2 > kStack) { cnt.stackov++; continue; }
        const bool lfirst = ln <= rn;
        stk[sp++] = lfirst ? cr : cl;
        stk[sp++] = lfirst ? cl : cr;
      } else if (hl || hr) {
        if (sp + 1 > kStack) { cnt.stackov++; continue; }
        stk[sp++] = hl ? cl : cr;
      }
    } else {
      const int p = ~id;
      const float4* gp = S.geom + 4 * (size_t)p;
      const float4 g0 = ldg4(gp), g1 = ldg4(gp + 1), g2 = ldg4(gp + 2), g3 = ldg4(gp + 3);
      PairGeom pg;
      if (!isect_exact(g0, g1, g2, g3, o, d, pg)) continue;
      if (!(pg.tx >= seg_lo && pg.te <= seg_hi)) continue;
      const uint64_t key = ((uint64_t)fkey(pg.te) << 32) | (uint32_t)__float_as_int(g3.z);
      if (key <= cursor) continue;
      if (nb == kmax && key >= hk[kmax - 1]) continue;
      int i = nb < kmax ? nb++ : kmax - 1;
      while (i > 0 && hk[i - 1] > key) {
        hk[i] = hk[i - 1];
        hp[i] = hp[i - 1];
        --i;
      }
      hk[i] = key;
      hp[i] = (uint32_t)p;
      if (nb == kmax) te_lim = fkey_inv((uint32_t)(hk[kmax - 1] >> 32));
    }
  }
  return nb;
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

// Per-(ray, Gaussian) set-up: exact interval, exponent polynomial of the
// weight w(tau) = sigma~ exp(-|u + tau d_l|^2 / 2) = 2^(c0 + tau (c1 + c2 tau)),
// tau = t - t_mid, with u = M x' from the compensated offset x' (value path).
__device__ void setup_pair(const SceneView& S, const float3& o, const float3& d, uint64_t key,
                           uint32_t pos, Entry& E) {
  const float4* gp = S.geom + 4 * (size_t)pos;
  const float4 g0 = ldg4(gp), g1 = ldg4(gp + 1), g2 = ldg4(gp + 2), g3 = ldg4(gp + 3);
  PairGeom pg;
  isect_exact(g0, g1, g2, g3, o, d, pg);
  const float x0 = offset_at(o.x, g0.x, pg.tm, d.x);
  const float x1 = offset_at(o.y, g0.y, pg.tm, d.y);
  const float x2 = offset_at(o.z, g0.z, pg.tm, d.z);
  const float u0 = g1.x * x0 + g1.y * x1 + g1.z * x2;
  const float u1 = g1.w * x0 + g2.x * x1 + g2.y * x2;
  const float u2 = g2.z * x0 + g2.w * x1 + g3.x * x2;
  const float qm = u0 * u0 + u1 * u1 + u2 * u2;
  const float b1 = u0 * pg.dl0 + u1 * pg.dl1 + u2 * pg.dl2;
  E.te = pg.te;
  E.tx = pg.tx;
  E.tm = pg.tm;
  E.c0 = lg2_approx(g0.w) - 0.5f * kLog2e * qm;
  E.c1 = -kLog2e * b1;
  E.c2 = -0.5f * kLog2e * pg.A;
  const float3 col = pair_color(S, (int)pos, d);
  E.cr = col.x; E.cg = col.y; E.cb = col.z;
  E.pos = (int)pos;
  E.idx = (uint32_t)(key & 0xFFFFFFFFu);
}

// 1 - exp(-x) without cancellation for small x
__device__ __forceinline__ float alpha_of(float x, float e) {
  if (x < 0.0625f) return x * (1.f - 0.5f * x * (1.f - (1.f / 3.f) * x * (1.f - 0.25f * x)));
  return 1.0f - e;
}

struct Group {
  float tk[kGroup];
  bool val[kGroup];
  float sg[kGroup], sr[kGroup], sgg[kGroup], sb[kGroup];
};

__device__ __forceinline__ void accum_entry(const Entry& E, Group& G, Counters& cnt) {
#pragma unroll
  for (int j = 0; j < kGroup; ++j) {
    if (G.val[j] && E.te <= G.tk[j] && G.tk[j] <= E.tx) {
      const float tau = G.tk[j] - E.tm;
      const float w = ex2_approx(fmaf(tau, fmaf(E.c2, tau, E.c1), E.c0));
      G.sg[j] += w;
      G.sr[j] = fmaf(w, E.cr, G.sr[j]);
      G.sgg[j] = fmaf(w, E.cg, G.sgg[j]);
      G.sb[j] = fmaf(w, E.cb, G.sb[j]);
      cnt.evals++;
    }
  }
}

struct BwdGroup {
  float dls[kGroup], dc0[kGroup], dc1[kGroup], dc2[kGroup], gc[kGroup], inv[kGroup];
};

__device__ __forceinline__ void grad_entry(const Entry& E, const Group& G, const BwdGroup& H,
                                           float* a) {
#pragma unroll
  for (int j = 0; j < kGroup; ++j) {
    if (G.val[j] && G.sg[j] > 0.f && E.te <= G.tk[j] && G.tk[j] <= E.tx) {
      const float tau = G.tk[j] - E.tm;
      const float w = ex2_approx(fmaf(tau, fmaf(E.c2, tau, E.c1), E.c0));
      const float dldw =
          H.dls[j] + (H.dc0[j] * E.cr + H.dc1[j] * E.cg + H.dc2[j] * E.cb - H.gc[j]) * H.inv[j];
      const float wd = w * dldw;
      const float wi = w * H.inv[j];
      a[0] += wd;
      a[1] = fmaf(wd, tau, a[1]);
      a[2] = fmaf(wd * tau, tau, a[2]);
      a[3] = fmaf(wi, H.dc0[j], a[3]);
      a[4] = fmaf(wi, H.dc1[j], a[4]);
      a[5] = fmaf(wi, H.dc2[j], a[5]);
    }
  }
}

// Per-pair gradient scatter into the Morton-ordered buffer:
//  [0..2] dL/dmu, [3] dL/dsigma~, [4..12] dL/dM, [16..] appearance grads.
//  With w = sigma~ exp(-|M x|^2/2), x = x' + tau d, u = M x', d_l = M d and
//  moments Sw = sum w dL/dw, Sw1 = sum w dL/dw tau, Sw2 = sum w dL/dw tau^2:
//    dL/dmu = M^T (Sw u + Sw1 d_l)
//    dL/dM  = -(Sw u x'^T + Sw1 (u d^T + d_l x'^T) + Sw2 d_l d^T)
//    dL/dsigma~ = Sw / sigma~
__device__ void scatter_pair(const SceneView& S, const Entry& E, const float* a, const float3& o,
                             const float3& d, float* gbuf, int gstride) {
  if (a[0] == 0.f && a[1] == 0.f && a[2] == 0.f && a[3] == 0.f && a[4] == 0.f && a[5] == 0.f)
    return;
  const float4* gp = S.geom + 4 * (size_t)E.pos;
  const float4 g0 = ldg4(gp), g1 = ldg4(gp + 1), g2 = ldg4(gp + 2), g3 = ldg4(gp + 3);
  const float M[9] = {g1.x, g1.y, g1.z, g1.w, g2.x, g2.y, g2.z, g2.w, g3.x};
  const float xp[3] = {offset_at(o.x, g0.x, E.tm, d.x), offset_at(o.y, g0.y, E.tm, d.y),
                       offset_at(o.z, g0.z, E.tm, d.z)};
  const float dv[3] = {d.x, d.y, d.z};
  float u[3], dl[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    u[r] = M[3 * r] * xp[0] + M[3 * r + 1] * xp[1] + M[3 * r + 2] * xp[2];
    dl[r] = M[3 * r] * dv[0] + M[3 * r + 1] * dv[1] + M[3 * r + 2] * dv[2];
  }
  const float Sw = a[0], Sw1 = a[1], Sw2 = a[2];
  float* row = gbuf + (size_t)E.pos * gstride;
  float gm[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    gm[b] = 0.f;
#pragma unroll
    for (int r = 0; r < 3; ++r) gm[b] += M[3 * r + b] * (Sw * u[r] + Sw1 * dl[r]);
  }
  float dM[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int b = 0; b < 3; ++b)
      dM[3 * r + b] = -(Sw * u[r] * xp[b] + Sw1 * (u[r] * dv[b] + dl[r] * xp[b]) +
                        Sw2 * dl[r] * dv[b]);
  float4* r4 = reinterpret_cast<float4*>(row);
  atomicAdd(r4 + 0, make_float4(gm[0], gm[1], gm[2], Sw / g0.w));
  atomicAdd(r4 + 1, make_float4(dM[0], dM[1], dM[2], dM[3]));
  atomicAdd(r4 + 2, make_float4(dM[4], dM[5], dM[6], dM[7]));
  atomicAdd(r4 + 3, make_float4(dM[8], 0.f, 0.f, 0.f));
  // appearance
  float Y[16];
  sh_basis(S.deg, d.x, d.y, d.z, Y);
  const int nc = (S.deg + 1) * (S.deg + 1);
  float v[kMaxApp + 3];
#pragma unroll
  for (int m = 0; m < 16; ++m)
    if (m < nc) {
      v[3 * m] = a[3] * Y[m];
      v[3 * m + 1] = a[4] * Y[m];
      v[3 * m + 2] = a[5] * Y[m];
    }
  const float* ap = S.app + (size_t)E.pos * S.app_stride + 3 * nc;
  for (int j = 0; j < S.lobes; ++j) {
    const float* q = ap + 7 * j;
    const float k0 = __ldg(q), k1 = __ldg(q + 1), k2 = __ldg(q + 2), lam = __ldg(q + 3);
    const float dp = d.x * __ldg(q + 4) + d.y * __ldg(q + 5) + d.z * __ldg(q + 6);
    const float e = ex2_approx(lam * (dp - 1.0f) * kLog2e);
    const float kd = (a[3] * k0 + a[4] * k1 + a[5] * k2) * e;
    float* dst = v + 3 * nc + 7 * j;
    dst[0] = a[3] * e; dst[1] = a[4] * e; dst[2] = a[5] * e;
    dst[3] = kd * (dp - 1.0f);
    dst[4] = kd * lam * d.x; dst[5] = kd * lam * d.y; dst[6] = kd * lam * d.z;
  }
  const int nv = 3 * nc + 7 * S.lobes;
  for (int k = nv; k < S.app_stride; ++k) v[k] = 0.f;
  float4* a4 = r4 + 4;
  for (int k = 0; k < S.app_stride / 4; ++k)
    atomicAdd(a4 + k, make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
}

__device__ __forceinline__ int skip_to(float te, int s, int B, float dt, float t0, float t1) {
  int est = (int)((te - t0) / ((float)B * dt));
  if (est < s + 1) est = s + 1;
  while (fminf(t1, fma_((float)((est + 1) * B), dt, t0)) < te) ++est;
  while (est > s + 1 && fminf(t1, fma_((float)(est * B), dt, t0)) >= te) --est;
  return est;
}

__device__ __forceinline__ void flush_stats(rg_stats* st, const Counters& c, bool hit) {
  const unsigned m = __activemask();
  const unsigned lane = threadIdx.x & 31;
  const unsigned leader = __ffs(m) - 1;
  const uint32_t v[10] = {1u, hit ? 1u : 0u, c.slabs, c.pairs, c.evals, c.samples, c.overflows,
                          c.fetches, c.nodes, c.stackov};
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(st);
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    const uint32_t s = __reduce_add_sync(m, v[k]);
    if (lane == leader && s) atomicAdd(dst + k, (unsigned long long)s);
  }
}

template <bool BWD>
__global__ void __launch_bounds__(kBlock) k_render(const RenderArgs P) {
  int ray;
  float3 o, d;
  if (P.cam_mode) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int px = blockIdx.x * 16 + (w & 1) * 8 + (lane & 7);
    const int py = blockIdx.y * 8 + (w >> 1) * 4 + (lane >> 3);
    if (px >= P.rw || py >= P.rh) return;
    ray = py * P.rw + px;
    camera_ray(P.cam, P.cam.x0 + px, P.cam.y0 + py, o, d);
  } else {
    ray = blockIdx.x * kBlock + threadIdx.x;
    if (ray >= P.n_rays) return;
    o = make_float3(P.ro[3 * ray], P.ro[3 * ray + 1], P.ro[3 * ray + 2]);
    d = make_float3(P.rd[3 * ray], P.rd[3 * ray + 1], P.rd[3 * ray + 2]);
  }
  const rg_config& c = P.c;
  const int B = c.slab_samples;
  const int K = c.hit_capacity;
  float C0 = 0.f, C1 = 0.f, C2 = 0.f, T = 1.f;
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
  float t0, t1;
  const bool hit = P.S.n > 0 && clip_exact(P.S.root_box, o, d, c.t_near, t0, t1);
  if (hit && !(BWD && gr0 == 0.f && gr1 == 0.f && gr2 == 0.f)) {
    const float3 inv = make_float3(1.0f / d.x, 1.0f / d.y, 1.0f / d.z);
    const float3 oinv = make_float3(o.x * inv.x, o.y * inv.y, o.z * inv.z);
    Entry act[kACap];
    float acc[BWD ? kACap : 1][6];
    uint64_t hk[kACap];
    uint32_t hp[kACap];
    int count = 0;
    uint64_t cursor = 0;
    bool exhausted = false;
    int s = 0;
    while (true) {
      const int k0 = s * B;
      if (!(sample_t(k0, c.dt, t0) < t1)) break;
      const float tlo = fma_((float)k0, c.dt, t0);
      const float thi = fminf(t1, fma_((float)(k0 + B), c.dt, t0));
      // expire Gaussians whose support ended before this slab
      int wr = 0;
      for (int e = 0; e < count; ++e) {
        if (act[e].tx >= tlo) {
          if (wr != e) {
            act[wr] = act[e];
            if (BWD)
              for (int k = 0; k < 6; ++k) acc[wr][k] = acc[e][k];
          }
          ++wr;
        } else if (BWD) {
          scatter_pair(P.S, act[e], acc[e], o, d, P.gbuf, P.gstride);
        }
      }
      count = wr;
      // refill in key order until every Gaussian entering by t_hi is held
      while (!exhausted && count < kACap && (count == 0 || act[count - 1].te <= thi)) {
        const int want = kACap - count;
        const int got = fetch(P.S, o, d, inv, oinv, tlo, t1, cursor, want, hk, hp, cnt);
        for (int i = 0; i < got; ++i) {
          setup_pair(P.S, o, d, hk[i], hp[i], act[count]);
          if (BWD)
            for (int k = 0; k < 6; ++k) acc[count][k] = 0.f;
          ++count;
        }
        cnt.pairs += got;
        if (got > 0) cursor = hk[got - 1];
        if (got < want) exhausted = true;
      }
      if (count == 0) break;
      if (act[0].te > thi) {   // empty slab(s): jump to the slab holding the next entry
        s = skip_to(act[0].te, s, B, c.dt, t0, t1);
        continue;
      }
      int n_in = 0;
      while (n_in < count && act[n_in].te <= thi) ++n_in;
      const int n_use = min(n_in, K);
      const bool more = (n_in == kACap) && !exhausted && (K > kACap);
      if (n_in > K) {
        cnt.overflows++;
      } else if (!BWD && n_in == K && n_in == kACap && !exhausted &&
                 fetch(P.S, o, d, inv, oinv, tlo, thi, cursor, 1, hk, hp, cnt) > 0) {
        cnt.overflows++;   // exactly K held, at least one more member beyond the cursor
      }
      if (dbg)
        for (int e = 0; e < n_use; ++e)
          if (dbg_n < P.dbg_cap) {
            int32_t* r = P.dbg_rec + 2 * ((size_t)ray * P.dbg_cap + dbg_n++);
            r[0] = s;
            r[1] = (int32_t)act[e].idx;
          }
      for (int g0 = 0; g0 < B; g0 += kGroup) {
        Group G;
#pragma unroll
        for (int j = 0; j < kGroup; ++j) {
          G.tk[j] = sample_t(k0 + g0 + j, c.dt, t0);
          G.val[j] = (g0 + j < B) && (G.tk[j] < t1);
          G.sg[j] = G.sr[j] = G.sgg[j] = G.sb[j] = 0.f;
        }
        for (int e = 0; e < n_use; ++e) accum_entry(act[e], G, cnt);
        if (more) {   // slab set larger than the active list: stream the rest
          uint64_t cur2 = cursor;
          int remaining = K - n_use;
          bool full_last = true;
          while (remaining > 0) {
            const int want = min(kACap, remaining);
            const int got = fetch(P.S, o, d, inv, oinv, tlo, thi, cur2, want, hk, hp, cnt);
            for (int i = 0; i < got; ++i) {
              Entry E;
              setup_pair(P.S, o, d, hk[i], hp[i], E);
              accum_entry(E, G, cnt);
              if (dbg && g0 == 0 && dbg_n < P.dbg_cap) {
                int32_t* r = P.dbg_rec + 2 * ((size_t)ray * P.dbg_cap + dbg_n++);
                r[0] = s;
                r[1] = (int32_t)E.idx;
              }
            }
            if (g0 == 0) cnt.pairs += got;
            remaining -= got;
            if (got > 0) cur2 = hk[got - 1];
            if (got < want) { full_last = false; break; }
          }
          if (g0 == 0 && remaining == 0 && full_last &&
              fetch(P.S, o, d, inv, oinv, tlo, thi, cur2, 1, hk, hp, cnt) > 0)
            cnt.overflows++;
        }
        // composite front to back (Eq. 4)
        BwdGroup H;
#pragma unroll
        for (int j = 0; j < kGroup; ++j) {
          if (BWD) { H.dls[j] = H.dc0[j] = H.dc1[j] = H.dc2[j] = H.gc[j] = H.inv[j] = 0.f; }
          if (G.val[j] && G.sg[j] > 0.f) {
            const float inv_s = 1.0f / G.sg[j];
            const float cr = G.sr[j] * inv_s, cg = G.sgg[j] * inv_s, cb = G.sb[j] * inv_s;
            const float x = G.sg[j] * c.dt;
            const float e = ex2_approx(-x * kLog2e);
            const float al = alpha_of(x, e);
            const float ta = T * al;
            C0 = fmaf(ta, cr, C0);
            C1 = fmaf(ta, cg, C1);
            C2 = fmaf(ta, cb, C2);
            if (BWD) {
              const float Tn = T * e;
              H.dc0[j] = gr0 * ta; H.dc1[j] = gr1 * ta; H.dc2[j] = gr2 * ta;
              const float gcj = gr0 * cr + gr1 * cg + gr2 * cb;
              const float gS = gr0 * (Pp0 - C0) + gr1 * (Pp1 - C1) + gr2 * (Pp2 - C2);
              H.dls[j] = c.dt * (Tn * gcj - gS);
              H.gc[j] = H.dc0[j] * cr + H.dc1[j] * cg + H.dc2[j] * cb;
              H.inv[j] = inv_s;
            }
            T *= e;
            cnt.samples++;
          }
        }
        if (BWD) {
          for (int e = 0; e < n_use; ++e) grad_entry(act[e], G, H, acc[e]);
          if (more) {
            uint64_t cur2 = cursor;
            int remaining = K - n_use;
            while (remaining > 0) {
              const int want = min(kACap, remaining);
              const int got = fetch(P.S, o, d, inv, oinv, tlo, thi, cur2, want, hk, hp, cnt);
              for (int i = 0; i < got; ++i) {
                Entry E;
                setup_pair(P.S, o, d, hk[i], hp[i], E);
                float a[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                grad_entry(E, G, H, a);
                scatter_pair(P.S, E, a, o, d, P.gbuf, P.gstride);
              }
              remaining -= got;
              if (got > 0) cur2 = hk[got - 1];
              if (got < want) break;
            }
          }
        }
      }
      cnt.slabs++;
      if (BWD) {
        if (s == replay_in) break;
      } else if (T <= c.t_eps) {
        replay = s;
        break;
      }
      ++s;
    }
    if (BWD)
      for (int e = 0; e < count; ++e) scatter_pair(P.S, act[e], acc[e], o, d, P.gbuf, P.gstride);
  }
  if (!BWD) {
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
    grid = dim3((A.rw + 15) / 16, (A.rh + 7) / 8);
  } else {
    A.cam_mode = 0;
    A.ro = rays->origin;
    A.rd = rays->dir;
    A.n_rays = rays->n;
    grid = dim3((rays->n + kBlock - 1) / kBlock);
  }
}

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
  k_render<false><<<grid, kBlock, 0, st>>>(A);
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
  if (A.n_rays > 0) { k_render<true><<<grid, kBlock, 0, st>>>(A); count_launches(1); }
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
