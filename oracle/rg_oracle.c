/*
 * rg_oracle.c -- plain, slow, single-threaded CPU ORACLE of the RayGauss hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see rg_oracle.h).  Written from PAPER.md; every
 * function cites the passage it follows (P:<line>, SURVEY.md §8(c) step O<k>,
 * DESIGN.md ARITH-<k> for the fp32 decision sequences, DESIGN.md L<k> for the
 * readings where the paper is silent).  No blocking, fusion or reordering beyond
 * what the definitions state.  Build:
 *   gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared rg_oracle.c -lm
 *
 * Parity pins: tests/test_oracle_*.py.  Functions without an external pin would
 * say "parity unpinned" here; none currently does.
 */
#include "rg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#if defined(__FAST_MATH__)
#error "the oracle must not be built with -ffast-math"
#endif

/* ------------------------------------------------------------------------ */
/* small utilities                                                           */
/* ------------------------------------------------------------------------ */

/* order-preserving map float -> uint32 (ties broken later by index, L8) */
static uint32_t fkey(float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

static uint64_t key64(float te, uint32_t idx) { return ((uint64_t)fkey(te) << 32) | idx; }

static int isfin(float x) { return isfinite(x); }

/* ------------------------------------------------------------------------ */
/* ARITH-1  R(q), q = (w,x,y,z)   (reading L11 = 3DGS convention)  */
/* ------------------------------------------------------------------------ */
void og_rotation_f32(const float q[4], float R[9]) {
  const float w = q[0], x = q[1], y = q[2], z = q[3];
  const float xx = x * x, yy = y * y, zz = z * z;
  const float xy = x * y, xz = x * z, yz = y * z;
  const float wx = w * x, wy = w * y, wz = w * z;
  R[0] = 1.0f - 2.0f * (yy + zz);
  R[1] = 2.0f * (xy - wz);
  R[2] = 2.0f * (xz + wy);
  R[3] = 2.0f * (xy + wz);
  R[4] = 1.0f - 2.0f * (xx + zz);
  R[5] = 2.0f * (yz - wx);
  R[6] = 2.0f * (xz - wy);
  R[7] = 2.0f * (yz + wx);
  R[8] = 1.0f - 2.0f * (xx + yy);
}

static void rotation_f64(const double q[4], double R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1.0 - 2.0 * (y * y + z * z);
  R[1] = 2.0 * (x * y - w * z);
  R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);
  R[4] = 1.0 - 2.0 * (x * x + z * z);
  R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);
  R[7] = 2.0 * (y * z + w * x);
  R[8] = 1.0 - 2.0 * (x * x + y * y);
}

/* d R_ij / d q_c for the polynomial above: dR[c*9 + (3i+j)] */
static void rotation_jacobian_f64(const double q[4], double dR[36]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  memset(dR, 0, 36 * sizeof(double));
  double* Dw = dR; double* Dx = dR + 9; double* Dy = dR + 18; double* Dz = dR + 27;
  /* R00 = 1-2(y^2+z^2) */ Dy[0] = -4 * y; Dz[0] = -4 * z;
  /* R01 = 2(xy-wz) */ Dw[1] = -2 * z; Dx[1] = 2 * y; Dy[1] = 2 * x; Dz[1] = -2 * w;
  /* R02 = 2(xz+wy) */ Dw[2] = 2 * y; Dx[2] = 2 * z; Dy[2] = 2 * w; Dz[2] = 2 * x;
  /* R10 = 2(xy+wz) */ Dw[3] = 2 * z; Dx[3] = 2 * y; Dy[3] = 2 * x; Dz[3] = 2 * w;
  /* R11 = 1-2(x^2+z^2) */ Dx[4] = -4 * x; Dz[4] = -4 * z;
  /* R12 = 2(yz-wx) */ Dw[5] = -2 * x; Dx[5] = -2 * w; Dy[5] = 2 * z; Dz[5] = 2 * y;
  /* R20 = 2(xz-wy) */ Dw[6] = -2 * y; Dx[6] = 2 * z; Dy[6] = -2 * w; Dz[6] = 2 * x;
  /* R21 = 2(yz+wx) */ Dw[7] = 2 * x; Dx[7] = 2 * w; Dy[7] = 2 * z; Dz[7] = 2 * y;
  /* R22 = 1-2(x^2+y^2) */ Dx[8] = -4 * x; Dy[8] = -4 * y;
}

/* ------------------------------------------------------------------------ */
/* ARITH-2..4  per-Gaussian support ellipsoid and its tight AABB              */
/*   M = S^-1 R^T so that (x-mu)^T Sigma^-1 (x-mu) = |M (x-mu)|^2  */
/*   r = phi^-1(sigma_eps / sigma~) = sqrt(2 ln(sigma~/sigma_eps)) */
/*   half-extent_i = sqrt(sum_j (s~_j R_ij)^2), s~ = s r */
/*   padded so that traversal stays conservative (DESIGN.md ARITH-4)          */
/* ------------------------------------------------------------------------ */
void og_prim_setup(const og_gaussians* g, const og_config* c, int32_t i,
                   float M[9], float* r2, float box[6], int32_t* flags) {
  const float* mu = g->mean + 3 * (size_t)i;
  const float* q = g->quat + 4 * (size_t)i;
  const float* s = g->scale + 3 * (size_t)i;
  const float dens = g->density[i];
  const int nc = (g->sh_degree + 1) * (g->sh_degree + 1);
  const int G = g->sg_count;
  int valid = 1;
  for (int k = 0; k < 3; ++k) valid &= isfin(mu[k]) && isfin(s[k]) && s[k] > 0.0f;
  for (int k = 0; k < 4; ++k) valid &= isfin(q[k]);
  valid &= isfin(dens);
  for (int k = 0; k < nc * 3; ++k) valid &= isfin(g->sh[(size_t)i * nc * 3 + k]);
  for (int k = 0; k < G * 3; ++k) valid &= isfin(g->sg_amp[(size_t)i * G * 3 + k]);
  for (int k = 0; k < G; ++k) valid &= isfin(g->sg_sharp[(size_t)i * G + k]);
  for (int k = 0; k < G * 3; ++k) valid &= isfin(g->sg_axis[(size_t)i * G * 3 + k]);
  const int active = valid && (dens > c->sigma_eps);
  *flags = (valid ? 1 : 0) | (active ? 2 : 0);
  for (int k = 0; k < 9; ++k) M[k] = 0.0f;
  *r2 = 0.0f;
  box[0] = box[1] = box[2] = INFINITY;
  box[3] = box[4] = box[5] = -INFINITY;
  if (!active) return;
  float R[9];
  og_rotation_f32(q, R);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) M[3 * a + b] = R[3 * b + a] / s[a];   /* ARITH-2 */
  if (c->radius_mode == 0) {                                           /* ARITH-3 */
    /* r^2 = phi^-1(sigma_eps / sigma~)^2, fp64 then rounded once;
       compact supports are the unit ball (no truncation needed) */
    const double k = (double)dens / (double)c->sigma_eps;
    switch (c->basis) {
      case 1: case 2: *r2 = 1.0f; break;                                /* Bump, Wendland */
      case 3: *r2 = (float)(k * k - 1.0); break;                        /* (1+r^2)^-1/2 >= 1/k */
      case 4: *r2 = (float)(k - 1.0); break;                            /* 1/(1+r^2) >= 1/k */
      case 5: {                                                         /* e^-r >= 1/k */
        const double l = log((double)dens) - log((double)c->sigma_eps);
        *r2 = (float)(l * l);
        break;
      }
      default: *r2 = (float)(2.0 * (log((double)dens) - log((double)c->sigma_eps)));
    }
  } else {
    *r2 = c->k_sigma * c->k_sigma;
  }
  for (int a = 0; a < 3; ++a) {                                         /* ARITH-4 */
    const float a0 = s[0] * R[3 * a + 0];
    const float a1 = s[1] * R[3 * a + 1];
    const float a2 = s[2] * R[3 * a + 2];
    const float ss = (a0 * a0 + a1 * a1) + a2 * a2;
    const float e = sqrtf(*r2 * ss);
    const float e1 = e * 0x1p-8f;
    const float m1 = (fabsf(mu[a]) + e) * 0x1p-18f;
    const float ep = (e + e1) + m1;
    box[a] = mu[a] - ep;
    box[3 + a] = mu[a] + ep;
  }
}

/* ------------------------------------------------------------------------ */
/* ARITH-5  segment / ellipsoid support interval (Haines'19 form: */
/* discriminant as r^2 - |perpendicular|^2)                    */
/* ------------------------------------------------------------------------ */
int32_t og_isect(const float M[9], float r2, const float mu[3], const float o[3],
                 const float d[3], float* te, float* tx) {
  const float v0 = o[0] - mu[0], v1 = o[1] - mu[1], v2 = o[2] - mu[2];
  const float ol0 = (M[0] * v0 + M[1] * v1) + M[2] * v2;
  const float ol1 = (M[3] * v0 + M[4] * v1) + M[5] * v2;
  const float ol2 = (M[6] * v0 + M[7] * v1) + M[8] * v2;
  const float dl0 = (M[0] * d[0] + M[1] * d[1]) + M[2] * d[2];
  const float dl1 = (M[3] * d[0] + M[4] * d[1]) + M[5] * d[2];
  const float dl2 = (M[6] * d[0] + M[7] * d[1]) + M[8] * d[2];
  const float A = (dl0 * dl0 + dl1 * dl1) + dl2 * dl2;
  const float B = (ol0 * dl0 + ol1 * dl1) + ol2 * dl2;
  const float tm = -(B / A);
  const float u0 = ol0 + tm * dl0, u1 = ol1 + tm * dl1, u2 = ol2 + tm * dl2;
  const float qmin = (u0 * u0 + u1 * u1) + u2 * u2;
  if (!(qmin <= r2)) return 0;
  const float h = sqrtf((r2 - qmin) / A);
  *te = tm - h;
  *tx = tm + h;
  return 1;
}

/* ------------------------------------------------------------------------ */
/* ARITH-6  30-bit Morton codes of the means (north star; L18)               */
/* ------------------------------------------------------------------------ */
void og_morton(const og_gaussians* g, const og_config* c, uint32_t* codes, uint32_t* fine,
               float lo[3], float hi[3]) {
  const int n = g->n;
  int* valid = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int a = 0; a < 3; ++a) { lo[a] = INFINITY; hi[a] = -INFINITY; }
  for (int i = 0; i < n; ++i) {
    float M[9], r2, box[6];
    int32_t fl;
    og_prim_setup(g, c, i, M, &r2, box, &fl);
    valid[i] = fl & 1;
    if (!valid[i]) continue;
    for (int a = 0; a < 3; ++a) {
      const float m = g->mean[3 * (size_t)i + a];
      if (m < lo[a]) lo[a] = m;
      if (m > hi[a]) hi[a] = m;
    }
  }
  for (int i = 0; i < n; ++i) {
    if (!valid[i]) { codes[i] = 0xFFFFFFFFu; fine[i] = 0u; continue; }
    uint32_t qv[3], fv[3];
    for (int a = 0; a < 3; ++a) {
      const float ext = hi[a] - lo[a];
      float u = 0.0f;
      if (ext > 0.0f) u = (g->mean[3 * (size_t)i + a] - lo[a]) / ext;
      const float v = u * 1024.0f;
      int qi = (int)floorf(v);
      if (qi < 0) qi = 0;
      if (qi > 1023) qi = 1023;
      qv[a] = (uint32_t)qi;
      int fi = (int)floorf(u * 131072.0f);          /* 2^17: 7 more bits (exact scaling) */
      if (fi < 0) fi = 0;
      if (fi > 131071) fi = 131071;
      fv[a] = (uint32_t)fi & 127u;
    }
    uint32_t fc = 0;
    for (int b = 0; b < 7; ++b) {
      fc |= ((fv[0] >> b) & 1u) << (3 * b + 2);
      fc |= ((fv[1] >> b) & 1u) << (3 * b + 1);
      fc |= ((fv[2] >> b) & 1u) << (3 * b + 0);
    }
    fine[i] = fc;
    uint32_t code = 0;
    for (int b = 0; b < 10; ++b) {   /* x takes the top bit of each triplet */
      code |= ((qv[0] >> b) & 1u) << (3 * b + 2);
      code |= ((qv[1] >> b) & 1u) << (3 * b + 1);
      code |= ((qv[2] >> b) & 1u) << (3 * b + 0);
    }
    codes[i] = code;
  }
  free(valid);
}

/* stable merge sort of indices by (code, fine) (O3: "std::stable_sort on codes") */
static uint64_t sort_key(const uint32_t* codes, const uint32_t* fine, uint32_t i) {
  return ((uint64_t)codes[i] << 32) | fine[i];
}
static void msort(uint32_t* idx, uint32_t* tmp, const uint32_t* codes, const uint32_t* fine, int lo,
                  int hi) {
  if (hi - lo < 2) return;
  const int mid = lo + (hi - lo) / 2;
  msort(idx, tmp, codes, fine, lo, mid);
  msort(idx, tmp, codes, fine, mid, hi);
  int i = lo, j = mid, k = lo;
  while (i < mid && j < hi)
    tmp[k++] = (sort_key(codes, fine, idx[j]) < sort_key(codes, fine, idx[i])) ? idx[j++] : idx[i++];
  while (i < mid) tmp[k++] = idx[i++];
  while (j < hi) tmp[k++] = idx[j++];
  memcpy(idx + lo, tmp + lo, sizeof(uint32_t) * (hi - lo));
}

void og_sort(int32_t n, const uint32_t* codes, const uint32_t* fine, uint32_t* order,
             uint32_t* sorted) {
  uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) order[i] = (uint32_t)i;
  msort(order, tmp, codes, fine, 0, n);
  for (int i = 0; i < n; ++i) sorted[i] = codes[order[i]];
  free(tmp);
}

/* ------------------------------------------------------------------------ */
/* Karras 2012 hierarchy, top-down recursive definition with keys augmented  */
/* by the position (unique keys): node covering [first,last] splits at the  */
/* highest position gamma whose key shares a longer prefix with key[first]  */
/* than key[last] does; children gamma / gamma+1 (leaf if range is a point)  */
/* ------------------------------------------------------------------------ */
static uint64_t akey(const uint32_t* c, int i) { return ((uint64_t)c[i] << 32) | (uint32_t)i; }
static int clz64(uint64_t x) { return x ? __builtin_clzll(x) : 64; }

static int find_split(const uint32_t* c, int first, int last) {
  const uint64_t kf = akey(c, first);
  const int common = clz64(kf ^ akey(c, last));
  /* largest gamma in [first, last-1] with prefix(first, gamma) > common,
     found by plain bisection over the monotone predicate */
  int lo = first, hi = last - 1;   /* predicate true at lo (prefix(first,first)=64) */
  while (lo < hi) {
    const int mid = lo + (hi - lo + 1) / 2;
    if (clz64(kf ^ akey(c, mid)) > common) lo = mid; else hi = mid - 1;
  }
  return lo;
}

static void karras_rec(const uint32_t* c, int first, int last, int node, int32_t* left,
                       int32_t* right) {
  const int gamma = find_split(c, first, last);
  left[node] = (gamma == first) ? ~gamma : gamma;
  right[node] = (gamma + 1 == last) ? ~(gamma + 1) : (gamma + 1);
  if (gamma != first) karras_rec(c, first, gamma, gamma, left, right);
  if (gamma + 1 != last) karras_rec(c, gamma + 1, last, gamma + 1, left, right);
}

void og_karras(int32_t n, const uint32_t* sorted_codes, int32_t* left, int32_t* right) {
  if (n < 2) return;
  karras_rec(sorted_codes, 0, n - 1, 0, left, right);
}

static void box_union(const float* a, const float* b, float* o) {
  for (int k = 0; k < 3; ++k) {
    o[k] = fminf(a[k], b[k]);
    o[3 + k] = fmaxf(a[3 + k], b[3 + k]);
  }
}

static const float* refit_rec(int32_t id, const int32_t* left, const int32_t* right,
                              const float* leaf_boxes, float* node_boxes) {
  if (id < 0) return leaf_boxes + 6 * (size_t)(~id);
  const float* a = refit_rec(left[id], left, right, leaf_boxes, node_boxes);
  const float* b = refit_rec(right[id], left, right, leaf_boxes, node_boxes);
  box_union(a, b, node_boxes + 6 * (size_t)id);
  return node_boxes + 6 * (size_t)id;
}

void og_refit(int32_t n, const int32_t* left, const int32_t* right, const float* leaf_boxes,
              float* node_boxes, float root[6]) {
  if (n <= 0) {
    root[0] = root[1] = root[2] = INFINITY;
    root[3] = root[4] = root[5] = -INFINITY;
    return;
  }
  const float* r = (n == 1) ? leaf_boxes : refit_rec(0, left, right, leaf_boxes, node_boxes);
  memcpy(root, r, 6 * sizeof(float));
}

/* ------------------------------------------------------------------------ */
/* ARITH-7  pinhole ray through each pixel centre             */
/* ------------------------------------------------------------------------ */
void og_camera_rays(int32_t width, int32_t height, float fx, float fy, float cx, float cy,
                    const float* c2w, int32_t x0, int32_t y0, int32_t x1, int32_t y1,
                    float* o, float* d) {
  (void)width; (void)height;
  const int w = x1 - x0;
  for (int py = y0; py < y1; ++py)
    for (int px = x0; px < x1; ++px) {
      const size_t r = (size_t)(py - y0) * w + (px - x0);
      const float xc = (((float)px + 0.5f) - cx) / fx;
      const float yc = (((float)py + 0.5f) - cy) / fy;
      float dw[3];
      for (int a = 0; a < 3; ++a) dw[a] = (c2w[4 * a + 0] * xc + c2w[4 * a + 1] * yc) + c2w[4 * a + 2];
      const float nrm = sqrtf((dw[0] * dw[0] + dw[1] * dw[1]) + dw[2] * dw[2]);
      for (int a = 0; a < 3; ++a) {
        d[3 * r + a] = dw[a] / nrm;
        o[3 * r + a] = c2w[4 * a + 3];
      }
    }
}

void og_camera_rays_spp(int32_t width, int32_t height, float fx, float fy, float cx, float cy,
                        const float* c2w, int32_t x0, int32_t y0, int32_t x1, int32_t y1,
                        int32_t spp, float* o, float* d) {
  (void)width; (void)height;
  const int w = x1 - x0;
  for (int py = y0; py < y1; ++py)
    for (int px = x0; px < x1; ++px)
      for (int s = 0; s < spp; ++s) {
        const size_t r = ((size_t)(py - y0) * w + (px - x0)) * (size_t)spp + (size_t)s;
        const float ox = spp == 1 ? 0.5f : 0.25f + 0.5f * (float)(s & 1);
        const float oy = spp == 1 ? 0.5f : 0.25f + 0.5f * (float)(s >> 1);
        const float xc = (((float)px + ox) - cx) / fx;
        const float yc = (((float)py + oy) - cy) / fy;
        float dw[3];
        for (int a = 0; a < 3; ++a) dw[a] = (c2w[4 * a + 0] * xc + c2w[4 * a + 1] * yc) + c2w[4 * a + 2];
        const float nrm = sqrtf((dw[0] * dw[0] + dw[1] * dw[1]) + dw[2] * dw[2]);
        for (int a = 0; a < 3; ++a) {
          d[3 * r + a] = dw[a] / nrm;
          o[3 * r + a] = c2w[4 * a + 3];
        }
      }
}

/* ------------------------------------------------------------------------ */
/* ARITH-8  IntersectBBox (Alg. 2 line 2), t0 clipped at t_near (L13)  */
/* ------------------------------------------------------------------------ */
int32_t og_clip(const float box[6], const float o[3], const float d[3], float t_near, float* t0,
                float* t1) {
  if (!(box[0] <= box[3]) || !(box[1] <= box[4]) || !(box[2] <= box[5])) return 0;
  float tmin[3], tmax[3];
  for (int a = 0; a < 3; ++a) {
    const float inv = 1.0f / d[a];
    const float ta = (box[a] - o[a]) * inv;
    const float tb = (box[3 + a] - o[a]) * inv;
    tmin[a] = fminf(ta, tb);
    tmax[a] = fmaxf(ta, tb);
  }
  *t0 = fmaxf(fmaxf(fmaxf(tmin[0], tmin[1]), tmin[2]), t_near);
  *t1 = fminf(fminf(tmax[0], tmax[1]), tmax[2]);
  return *t0 < *t1;
}

/* ------------------------------------------------------------------------ */
/* BVH (O3)                                                                  */
/* ------------------------------------------------------------------------ */
struct og_bvh {
  int32_t n;
  uint32_t *codes, *sorted, *order, *fine;
  int32_t *left, *right;
  float *leaf_boxes, *node_boxes;
  float root[6], mean_lo[3], mean_hi[3];
};

og_bvh* og_build(const og_gaussians* g, const og_config* c) {
  og_bvh* b = (og_bvh*)calloc(1, sizeof(og_bvh));
  const int n = g->n;
  const size_t n1 = n > 0 ? (size_t)n : 1;
  b->n = n;
  b->codes = (uint32_t*)malloc(4 * n1);
  b->fine = (uint32_t*)malloc(4 * n1);
  b->sorted = (uint32_t*)malloc(4 * n1);
  b->order = (uint32_t*)malloc(4 * n1);
  b->left = (int32_t*)malloc(4 * n1);
  b->right = (int32_t*)malloc(4 * n1);
  b->leaf_boxes = (float*)malloc(24 * n1);
  b->node_boxes = (float*)malloc(24 * n1);
  og_morton(g, c, b->codes, b->fine, b->mean_lo, b->mean_hi);
  og_sort(n, b->codes, b->fine, b->order, b->sorted);
  og_karras(n, b->sorted, b->left, b->right);
  for (int p = 0; p < n; ++p) {
    float M[9], r2;
    int32_t fl;
    og_prim_setup(g, c, (int32_t)b->order[p], M, &r2, b->leaf_boxes + 6 * (size_t)p, &fl);
  }
  og_refit(n, b->left, b->right, b->leaf_boxes, b->node_boxes, b->root);
  return b;
}

void og_free(og_bvh* b) {
  if (!b) return;
  free(b->codes); free(b->fine); free(b->sorted); free(b->order); free(b->left); free(b->right);
  free(b->leaf_boxes); free(b->node_boxes); free(b);
}

void og_bvh_views(const og_bvh* b, const uint32_t** codes_unsorted, const uint32_t** sorted_codes,
                  const uint32_t** order, const int32_t** left, const int32_t** right,
                  const float** leaf_boxes_sorted, const float** node_boxes, const float** root,
                  const float** mean_lo, const float** mean_hi, const uint32_t** fine) {
  if (fine) *fine = b->fine;
  if (codes_unsorted) *codes_unsorted = b->codes;
  if (sorted_codes) *sorted_codes = b->sorted;
  if (order) *order = b->order;
  if (left) *left = b->left;
  if (right) *right = b->right;
  if (leaf_boxes_sorted) *leaf_boxes_sorted = b->leaf_boxes;
  if (node_boxes) *node_boxes = b->node_boxes;
  if (root) *root = b->root;
  if (mean_lo) *mean_lo = b->mean_lo;
  if (mean_hi) *mean_hi = b->mean_hi;
}

/* conservative segment/box test for traversal only (never decides a set) */
static int box_overlaps_segment(const float* bx, const float o[3], const float d[3], float tlo,
                                float thi) {
  if (!(bx[0] <= bx[3])) return 0;
  double a = (double)tlo, b = (double)thi;
  const double slack = 1e-6 * (fabs(a) + fabs(b) + 1.0);
  a -= slack; b += slack;
  for (int k = 0; k < 3; ++k) {
    const double dk = d[k], ok = o[k];
    if (dk == 0.0) {
      if (ok < bx[k] || ok > bx[3 + k]) return 0;
      continue;
    }
    double t0 = (bx[k] - ok) / dk, t1 = (bx[3 + k] - ok) / dk;
    if (t0 > t1) { const double t = t0; t0 = t1; t1 = t; }
    if (t0 > a) a = t0;
    if (t1 < b) b = t1;
    if (a > b) return 0;
  }
  return 1;
}

/* ------------------------------------------------------------------------ */
/* fp64 colour: Eq. 14-15; SH in the 3DGS real basis (L10)       */
/* constants from their closed forms                                         */
/* ------------------------------------------------------------------------ */
void og_sh_basis(int32_t degree, const double d[3], double* Y) {
  const double x = d[0], y = d[1], z = d[2];
  const double pi = 3.14159265358979323846;
  Y[0] = 0.5 / sqrt(pi);
  if (degree < 1) return;
  const double c1 = sqrt(3.0 / (4.0 * pi));
  Y[1] = -c1 * y; Y[2] = c1 * z; Y[3] = -c1 * x;
  if (degree < 2) return;
  const double c2a = 0.5 * sqrt(15.0 / pi), c2b = 0.25 * sqrt(5.0 / pi), c2c = 0.25 * sqrt(15.0 / pi);
  Y[4] = c2a * x * y;
  Y[5] = -c2a * y * z;
  Y[6] = c2b * (2.0 * z * z - x * x - y * y);
  Y[7] = -c2a * x * z;
  Y[8] = c2c * (x * x - y * y);
  if (degree < 3) return;
  const double c3a = 0.25 * sqrt(35.0 / (2.0 * pi)), c3b = 0.5 * sqrt(105.0 / pi);
  const double c3c = 0.25 * sqrt(21.0 / (2.0 * pi)), c3d = 0.25 * sqrt(7.0 / pi);
  const double c3e = 0.25 * sqrt(105.0 / pi);
  Y[9] = -c3a * y * (3.0 * x * x - y * y);
  Y[10] = c3b * x * y * z;
  Y[11] = -c3c * y * (4.0 * z * z - x * x - y * y);
  Y[12] = c3d * z * (2.0 * z * z - 3.0 * x * x - 3.0 * y * y);
  Y[13] = -c3c * x * (4.0 * z * z - x * x - y * y);
  Y[14] = c3e * z * (x * x - y * y);
  Y[15] = -c3a * x * (x * x - 3.0 * y * y);
}

void og_color(const og_gaussians* g, int32_t i, const double d[3], double rgb[3]) {
  const int nc = (g->sh_degree + 1) * (g->sh_degree + 1);
  double Y[16];
  og_sh_basis(g->sh_degree, d, Y);
  rgb[0] = rgb[1] = rgb[2] = 0.0;
  const float* sh = g->sh + (size_t)i * nc * 3;
  for (int m = 0; m < nc; ++m)
    for (int ch = 0; ch < 3; ++ch) rgb[ch] += (double)sh[3 * m + ch] * Y[m];
  for (int j = 0; j < g->sg_count; ++j) {
    const float* p = g->sg_axis + ((size_t)i * g->sg_count + j) * 3;
    const float* k = g->sg_amp + ((size_t)i * g->sg_count + j) * 3;
    const double lam = g->sg_sharp[(size_t)i * g->sg_count + j];
    const double dp = d[0] * p[0] + d[1] * p[1] + d[2] * p[2];
    const double e = exp(lam * (dp - 1.0));
    for (int ch = 0; ch < 3; ++ch) rgb[ch] += (double)k[ch] * e;
  }
}

/* ------------------------------------------------------------------------ */
/* render core                                                               */
/* ------------------------------------------------------------------------ */
typedef struct { uint64_t key; int32_t l; float te, tx; } member;
typedef struct { int32_t l; double w; } contrib;
typedef struct { double sigma, c[3], T, alpha; float tk; int32_t first, count; } srec;

typedef struct {
  srec* s; int ns, cs;
  contrib* c; int nc, cc;
} recorder;

typedef struct {
  const og_gaussians* g;     /* values */
  const og_config* cfg;
  int mode;
  const og_bvh* bvh;
  int n;
  /* decision data per original index (from dec or g) */
  float *M, *r2, *mu, *box;
  int32_t* flags;
  float root[6];
  /* fp64 value data */
  double *M64, *R64;
  double* col; int32_t* col_stamp; int32_t* pair_stamp;
  /* scratch */
  member* set; int cap_set;
  float *te_all, *tx_all; uint8_t* hit_all;
} ctx_t;

static int cmp_member(const void* a, const void* b) {
  const uint64_t ka = ((const member*)a)->key, kb = ((const member*)b)->key;
  return ka < kb ? -1 : (ka > kb ? 1 : 0);
}

static void set_push(ctx_t* cx, int* n, member m) {
  if (*n == cx->cap_set) {
    cx->cap_set = cx->cap_set ? 2 * cx->cap_set : 256;
    cx->set = (member*)realloc(cx->set, sizeof(member) * cx->cap_set);
  }
  cx->set[(*n)++] = m;
}

static const double* color_of(ctx_t* cx, int l, int ray, const double d[3]) {
  if (cx->col_stamp[l] != ray) {
    og_color(cx->g, l, d, cx->col + 3 * (size_t)l);
    cx->col_stamp[l] = ray;
  }
  return cx->col + 3 * (size_t)l;
}

/* basis functions of the supplementary as functions of q = r^2 */
double og_basis_phi(int32_t basis, double q) {
  const double r = sqrt(q);
  switch (basis) {
    case 1: return q < 1.0 ? exp(1.0 - 1.0 / (1.0 - q)) : 0.0;              /* Bump * e */
    case 2: return r <= 1.0 ? pow(1.0 - r, 4) * (4.0 * r + 1.0) : 0.0;        /* Wendland */
    case 3: return 1.0 / sqrt(1.0 + q);                                       /* inv. multiquadric */
    case 4: return 1.0 / (1.0 + q);                                           /* inv. quadratic */
    case 5: return exp(-r);                                                   /* C0-Matern */
    default: return exp(-0.5 * q);                                            /* Gaussian */
  }
}

/* psi = -2 sigma~ dphi/dq: dw/dy = -psi y for y = M(x - mu), |y|^2 = q */
double og_basis_psi(int32_t basis, double sigma, double q) {
  const double r = sqrt(q);
  switch (basis) {
    case 1: return q < 1.0 ? 2.0 * sigma * og_basis_phi(1, q) / ((1.0 - q) * (1.0 - q)) : 0.0;
    case 2: return r <= 1.0 ? 20.0 * sigma * pow(1.0 - r, 3) : 0.0;
    case 3: return sigma * pow(1.0 + q, -1.5);
    case 4: return 2.0 * sigma / ((1.0 + q) * (1.0 + q));
    case 5: return r > 0.0 ? sigma * exp(-r) / r : 0.0;    /* kink at r = 0: subgradient 0 */
    default: return sigma * exp(-0.5 * q);
  }
}

/* fp64 weight sigma~ * phi(|M(x-mu)|) at x (Eq. 12-13; other bases P:456-515) */
static double weight_at(const ctx_t* cx, int l, const double x[3], double y_out[3]) {
  const double* M = cx->M64 + 9 * (size_t)l;
  const float* mu = cx->g->mean + 3 * (size_t)l;
  const double v0 = x[0] - mu[0], v1 = x[1] - mu[1], v2 = x[2] - mu[2];
  double y[3];
  for (int a = 0; a < 3; ++a) y[a] = M[3 * a] * v0 + M[3 * a + 1] * v1 + M[3 * a + 2] * v2;
  if (y_out) { y_out[0] = y[0]; y_out[1] = y[1]; y_out[2] = y[2]; }
  return (double)cx->g->density[l] * og_basis_phi(cx->cfg->basis, y[0] * y[0] + y[1] * y[1] + y[2] * y[2]);
}

/* per-slab hit set: Gaussians whose support interval overlaps [tlo, thi] (L9) */
static int slab_set(ctx_t* cx, const float o[3], const float d[3], float tlo, float thi) {
  int n = 0;
  if (cx->mode == 1) {
    for (int l = 0; l < cx->n; ++l) {
      if (!cx->hit_all[l]) continue;
      if (cx->te_all[l] <= thi && cx->tx_all[l] >= tlo) {
        member m = {key64(cx->te_all[l], (uint32_t)l), l, cx->te_all[l], cx->tx_all[l]};
        set_push(cx, &n, m);
      }
    }
  } else {
    const og_bvh* b = cx->bvh;
    if (b->n == 0) return 0;
    int32_t stack[256];
    int sp = 0;
    stack[sp++] = (b->n == 1) ? ~0 : 0;
    while (sp) {
      const int32_t id = stack[--sp];
      if (id >= 0) {
        if (!box_overlaps_segment(b->node_boxes + 6 * (size_t)id, o, d, tlo, thi)) continue;
        stack[sp++] = b->left[id];
        stack[sp++] = b->right[id];
      } else {
        const int p = ~id;
        const int l = (int)b->order[p];
        if (!(cx->flags[l] & 2)) continue;
        float te, tx;
        if (!og_isect(cx->M + 9 * (size_t)l, cx->r2[l], cx->mu + 3 * (size_t)l, o, d, &te, &tx))
          continue;
        if (te <= thi && tx >= tlo) {
          member m = {key64(te, (uint32_t)l), l, te, tx};
          set_push(cx, &n, m);
        }
      }
    }
  }
  qsort(cx->set, n, sizeof(member), cmp_member);   /* L8: (t_entry, index) order */
  return n;
}

static void rec_sample(recorder* rc, double sigma, const double c[3], double T, double alpha,
                       float tk, int first, int count) {
  if (!rc) return;
  if (rc->ns == rc->cs) {
    rc->cs = rc->cs ? 2 * rc->cs : 1024;
    rc->s = (srec*)realloc(rc->s, sizeof(srec) * rc->cs);
  }
  srec* s = rc->s + rc->ns++;
  s->sigma = sigma; s->c[0] = c[0]; s->c[1] = c[1]; s->c[2] = c[2];
  s->T = T; s->alpha = alpha; s->tk = tk; s->first = first; s->count = count;
}

static void rec_contrib(recorder* rc, int l, double w) {
  if (!rc) return;
  if (rc->nc == rc->cc) {
    rc->cc = rc->cc ? 2 * rc->cc : 4096;
    rc->c = (contrib*)realloc(rc->c, sizeof(contrib) * rc->cc);
  }
  rc->c[rc->nc].l = l;
  rc->c[rc->nc].w = w;
  rc->nc++;
}

/* integrate one sample at t_k over a sorted contributor list (Eq. 4 P:95-101,
   Eq. 10-11, truncation per sample L2) */
static void do_sample(ctx_t* cx, int ray, const float o[3], const float d[3], const double dd[3],
                      float tk, const member* set, int n_set, double* C, double* T,
                      og_counters* cnt, recorder* rc) {
  const double x[3] = {(double)o[0] + (double)tk * (double)d[0],
                       (double)o[1] + (double)tk * (double)d[1],
                       (double)o[2] + (double)tk * (double)d[2]};
  double sigma = 0.0, sc[3] = {0.0, 0.0, 0.0};
  const int first = rc ? rc->nc : 0;
  int count = 0;
  for (int m = 0; m < n_set; ++m) {
    if (!(set[m].te <= tk && tk <= set[m].tx)) continue;
    const int l = set[m].l;
    const double w = weight_at(cx, l, x, NULL);
    const double* cl = color_of(cx, l, ray, dd);
    sigma += w;
    for (int ch = 0; ch < 3; ++ch) sc[ch] += w * cl[ch];
    rec_contrib(rc, l, w);
    ++count;
    if (cnt) cnt->evals++;
  }
  if (sigma > 0.0) {     /* O6: sigma_k = 0 skips the sample */
    const double e = exp(-sigma * (double)cx->cfg->dt);
    const double alpha = 1.0 - e;
    double c[3];
    for (int ch = 0; ch < 3; ++ch) c[ch] = sc[ch] / sigma;
    rec_sample(rc, sigma, c, *T, alpha, tk, first, count);
    for (int ch = 0; ch < 3; ++ch) C[ch] += (*T * alpha) * c[ch];
    *T = *T * e;
    if (cnt) cnt->samples++;
  }
}

/* Alg. 2 for one ray; returns terminal slab or -1 */
static void render_ray(ctx_t* cx, int ray, const float o[3], const float d[3], int force,
                       int32_t force_s, double rgb[3], double* Tout, int32_t* s_term,
                       og_counters* cnt, int32_t dump_cap, int32_t* dump_count, int32_t* dump,
                       recorder* rc) {
  const og_config* cf = cx->cfg;
  double C[3] = {0.0, 0.0, 0.0}, T = 1.0;
  *s_term = -1;
  if (dump_count) *dump_count = 0;
  float t0, t1;
  const int B = cf->slab_samples;
  const double dd[3] = {d[0], d[1], d[2]};
  if (og_clip(cx->root, o, d, cf->t_near, &t0, &t1)) {
    if (cnt) cnt->rays_hit++;
    if (cx->mode == 1 || cx->mode == 0) {
      for (int l = 0; l < cx->n; ++l) {
        cx->hit_all[l] = 0;
        if (!(cx->flags[l] & 2)) continue;
        float te, tx;
        if (og_isect(cx->M + 9 * (size_t)l, cx->r2[l], cx->mu + 3 * (size_t)l, o, d, &te, &tx)) {
          cx->hit_all[l] = 1; cx->te_all[l] = te; cx->tx_all[l] = tx;
        }
      }
    }
    for (int s = 0;; ++s) {
      const float tfirst = fmaf((float)(s * B) + 0.5f, cf->dt, t0);       /* ARITH-9 */
      if (!(tfirst < t1)) break;
      const float tlo = fmaf((float)(s * B), cf->dt, t0);
      const float thi = fminf(t1, fmaf((float)((s + 1) * B), cf->dt, t0));
      int n_set;
      if (cx->mode == 0) {
        /* plain per-sample definition: the "set" is all hit Gaussians; the
           per-sample test t_entry <= t_k <= t_exit decides (no truncation) */
        n_set = 0;
        for (int l = 0; l < cx->n; ++l)
          if (cx->hit_all[l]) {
            member m = {key64(cx->te_all[l], (uint32_t)l), l, cx->te_all[l], cx->tx_all[l]};
            set_push(cx, &n_set, m);
          }
        qsort(cx->set, n_set, sizeof(member), cmp_member);
        int nonempty = 0;
        for (int m = 0; m < n_set; ++m)
          if (cx->set[m].te <= thi && cx->set[m].tx >= tlo) {
            nonempty = 1;
            if (cnt && cx->pair_stamp[cx->set[m].l] != ray) { cnt->pairs++; cx->pair_stamp[cx->set[m].l] = ray; }
          }
        if (nonempty && cnt) cnt->slabs++;
      } else {
        n_set = slab_set(cx, o, d, tlo, thi);
        if (n_set == 0) continue;                                           /* Alg.2 l.20-23 */
        if (n_set > cf->hit_capacity) {                                      /* L7 */
          if (cnt) cnt->overflows++;
          n_set = cf->hit_capacity;
        }
        if (cnt) {
          cnt->slabs++;
          for (int m = 0; m < n_set; ++m)
            if (cx->pair_stamp[cx->set[m].l] != ray) { cnt->pairs++; cx->pair_stamp[cx->set[m].l] = ray; }
        }
        if (dump_count)
          for (int m = 0; m < n_set; ++m)
            if (*dump_count < dump_cap) {
              dump[2 * (*dump_count)] = s;
              dump[2 * (*dump_count) + 1] = cx->set[m].l;
              (*dump_count)++;
            }
      }
      for (int j = 0; j < B; ++j) {
        const float tk = fmaf((float)(s * B + j) + 0.5f, cf->dt, t0);
        if (!(tk < t1)) break;
        do_sample(cx, ray, o, d, dd, tk, cx->set, n_set, C, &T, cnt, rc);
      }
      if (force) {
        if (s == force_s) { *s_term = s; break; }
      } else if (T <= (double)cf->t_eps) {                                   /* L6 */
        *s_term = s;
        break;
      }
    }
  }
  for (int ch = 0; ch < 3; ++ch) rgb[ch] = C[ch] + T * (double)cf->background[ch];   /* L12 */
  *Tout = T;
}

static int ctx_init(ctx_t* cx, const og_gaussians* g, const og_gaussians* dec, const og_config* c,
                    int mode, const og_bvh* bvh) {
  memset(cx, 0, sizeof(*cx));
  const og_gaussians* gd = dec ? dec : g;
  const int n = g->n;
  const size_t n1 = n > 0 ? (size_t)n : 1;
  cx->g = g; cx->cfg = c; cx->mode = mode; cx->bvh = bvh; cx->n = n;
  if (mode == 2 && (!bvh || bvh->n != n)) return -1;
  cx->M = (float*)malloc(36 * n1); cx->r2 = (float*)malloc(4 * n1);
  cx->mu = (float*)malloc(12 * n1); cx->box = (float*)malloc(24 * n1);
  cx->flags = (int32_t*)malloc(4 * n1);
  cx->M64 = (double*)malloc(72 * n1); cx->R64 = (double*)malloc(72 * n1);
  cx->col = (double*)malloc(24 * n1); cx->col_stamp = (int32_t*)malloc(4 * n1);
  cx->pair_stamp = (int32_t*)malloc(4 * n1);
  cx->te_all = (float*)malloc(4 * n1); cx->tx_all = (float*)malloc(4 * n1);
  cx->hit_all = (uint8_t*)calloc(n1, 1);
  for (int a = 0; a < 3; ++a) { cx->root[a] = INFINITY; cx->root[3 + a] = -INFINITY; }
  for (int l = 0; l < n; ++l) {
    og_prim_setup(gd, c, l, cx->M + 9 * (size_t)l, cx->r2 + l, cx->box + 6 * (size_t)l, cx->flags + l);
    memcpy(cx->mu + 3 * (size_t)l, gd->mean + 3 * (size_t)l, 12);
    box_union(cx->root, cx->box + 6 * (size_t)l, cx->root);
    cx->col_stamp[l] = -1;
    cx->pair_stamp[l] = -1;
    /* fp64 value-path geometry from g */
    double q[4], R[9];
    for (int k = 0; k < 4; ++k) q[k] = g->quat[4 * (size_t)l + k];
    rotation_f64(q, R);
    memcpy(cx->R64 + 9 * (size_t)l, R, sizeof(R));
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b)
        cx->M64[9 * (size_t)l + 3 * a + b] = R[3 * b + a] / (double)g->scale[3 * (size_t)l + a];
  }
  if (mode == 2 && !dec) memcpy(cx->root, bvh->root, sizeof(cx->root));
  return 0;
}

static void ctx_free(ctx_t* cx) {
  free(cx->M); free(cx->r2); free(cx->mu); free(cx->box); free(cx->flags);
  free(cx->M64); free(cx->R64); free(cx->col); free(cx->col_stamp); free(cx->pair_stamp);
  free(cx->te_all); free(cx->tx_all); free(cx->hit_all); free(cx->set);
}

int32_t og_render(const og_gaussians* g, const og_gaussians* dec, const og_config* c, int32_t mode,
                  const og_bvh* bvh, int32_t n_rays, const float* ray_o, const float* ray_d,
                  const int32_t* force_s_term, double* rgb, double* T, int32_t* s_term,
                  og_counters* cnt, int32_t dump_cap, int32_t* dump_counts, int32_t* dump) {
  ctx_t cx;
  if (mode == 2 && dec) return -2;   /* frozen decisions use brute-force sets */
  if (ctx_init(&cx, g, dec, c, mode, bvh)) { ctx_free(&cx); return -1; }
  if (cnt) memset(cnt, 0, sizeof(*cnt));
  for (int r = 0; r < n_rays; ++r) {
    render_ray(&cx, r, ray_o + 3 * (size_t)r, ray_d + 3 * (size_t)r, force_s_term != NULL,
               force_s_term ? force_s_term[r] : -1, rgb + 3 * (size_t)r, T + r, s_term + r, cnt,
               dump_cap, dump_counts ? dump_counts + r : NULL,
               dump ? dump + 2 * (size_t)dump_cap * r : NULL, NULL);
  }
  ctx_free(&cx);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* backward: chain rule through Eq. 4 / Eq. 10-15 written per sample and per */
/* contributor (the derivatives of SURVEY.md O8, evaluated directly, without */
/* its moment factorisation).  dP/dc_k = T_k alpha_k; dP/dsigma_k =          */
/* dt (T_{k+1} c_k - S_k), S_k = sum_{j>k} T_j alpha_j c_j + T_end bg.        */
/* ------------------------------------------------------------------------ */
int32_t og_backward(const og_gaussians* g, const og_config* c, int32_t mode, const og_bvh* bvh,
                    int32_t n_rays, const float* ray_o, const float* ray_d, const double* d_rgb,
                    double* g_mean, double* g_quat, double* g_scale, double* g_density,
                    double* g_sh, double* g_sg_amp, double* g_sg_sharp, double* g_sg_axis) {
  ctx_t cx;
  if (ctx_init(&cx, g, NULL, c, mode, bvh)) { ctx_free(&cx); return -1; }
  recorder rc;
  memset(&rc, 0, sizeof(rc));
  const int nc = (g->sh_degree + 1) * (g->sh_degree + 1);
  const int G = g->sg_count;
  const double dt = c->dt;
  for (int r = 0; r < n_rays; ++r) {
    const float* o = ray_o + 3 * (size_t)r;
    const float* d = ray_d + 3 * (size_t)r;
    const double dd[3] = {d[0], d[1], d[2]};
    const double* gr = d_rgb + 3 * (size_t)r;
    rc.ns = 0; rc.nc = 0;
    double P[3], Tend;
    int32_t st;
    render_ray(&cx, r, o, d, 0, -1, P, &Tend, &st, NULL, 0, NULL, NULL, &rc);
    double Y[16];
    og_sh_basis(g->sh_degree, dd, Y);
    double S[3];
    for (int ch = 0; ch < 3; ++ch) S[ch] = Tend * (double)c->background[ch];
    for (int k = rc.ns - 1; k >= 0; --k) {
      const srec* sk = rc.s + k;
      const double Tk1 = sk->T * (1.0 - sk->alpha);
      double dLdc[3], gc = 0.0, gS = 0.0;
      for (int ch = 0; ch < 3; ++ch) {
        dLdc[ch] = gr[ch] * sk->T * sk->alpha;
        gc += gr[ch] * sk->c[ch];
        gS += gr[ch] * S[ch];
      }
      const double dLdsigma = dt * (Tk1 * gc - gS);
      const double x[3] = {(double)o[0] + (double)sk->tk * dd[0],
                           (double)o[1] + (double)sk->tk * dd[1],
                           (double)o[2] + (double)sk->tk * dd[2]};
      for (int m = 0; m < sk->count; ++m) {
        const contrib* ct = rc.c + sk->first + m;
        const int l = ct->l;
        const double w = ct->w;
        const double* cl = color_of(&cx, l, r, dd);
        double dLdw = dLdsigma;
        for (int ch = 0; ch < 3; ++ch) dLdw += dLdc[ch] * (cl[ch] - sk->c[ch]) / sk->sigma;
        double dLdcl[3];
        for (int ch = 0; ch < 3; ++ch) dLdcl[ch] = (w / sk->sigma) * dLdc[ch];
        /* colour parameters (Eq. 14-15) */
        for (int mm = 0; mm < nc; ++mm)
          for (int ch = 0; ch < 3; ++ch) g_sh[((size_t)l * nc + mm) * 3 + ch] += dLdcl[ch] * Y[mm];
        for (int j = 0; j < G; ++j) {
          const size_t lj = (size_t)l * G + j;
          const float* p = g->sg_axis + lj * 3;
          const float* kk = g->sg_amp + lj * 3;
          const double lam = g->sg_sharp[lj];
          const double dp = dd[0] * p[0] + dd[1] * p[1] + dd[2] * p[2];
          const double e = exp(lam * (dp - 1.0));
          double kd = 0.0;
          for (int ch = 0; ch < 3; ++ch) {
            g_sg_amp[lj * 3 + ch] += dLdcl[ch] * e;
            kd += dLdcl[ch] * kk[ch];
          }
          g_sg_sharp[lj] += kd * e * (dp - 1.0);
          for (int a = 0; a < 3; ++a) g_sg_axis[lj * 3 + a] += kd * e * lam * dd[a];
        }
        /* geometry: w = sigma~ exp(-|M(x-mu)|^2 / 2), M = S^-1 R^T */
        const double* M = cx.M64 + 9 * (size_t)l;
        const double* R = cx.R64 + 9 * (size_t)l;
        const float* mu = g->mean + 3 * (size_t)l;
        const float* sc = g->scale + 3 * (size_t)l;
        double y[3];
        const double wchk = weight_at(&cx, l, x, y);
        (void)wchk;
        const double psi = og_basis_psi(c->basis, (double)g->density[l],
                                        y[0] * y[0] + y[1] * y[1] + y[2] * y[2]);
        const double v[3] = {x[0] - mu[0], x[1] - mu[1], x[2] - mu[2]};
        for (int b = 0; b < 3; ++b) {     /* dw/dmu = psi M^T y (psi = w: Gaussian) */
          const double mty = M[b] * y[0] + M[3 + b] * y[1] + M[6 + b] * y[2];
          g_mean[3 * (size_t)l + b] += dLdw * psi * mty;
        }
        g_density[l] += dLdw * w / (double)g->density[l];
        double dLdR[9] = {0};
        for (int a = 0; a < 3; ++a) {
          const double sa = sc[a];
          for (int b = 0; b < 3; ++b) {
            const double dLdM = dLdw * (-psi * y[a] * v[b]);   /* dw/dM_ab = -psi y_a v_b */
            g_scale[3 * (size_t)l + a] += dLdM * (-R[3 * b + a] / (sa * sa));
            dLdR[3 * b + a] += dLdM / sa;                       /* M_ab = R_ba / s_a */
          }
        }
        double q[4], J[36];
        for (int kq = 0; kq < 4; ++kq) q[kq] = g->quat[4 * (size_t)l + kq];
        rotation_jacobian_f64(q, J);
        for (int kq = 0; kq < 4; ++kq) {
          double acc = 0.0;
          for (int e = 0; e < 9; ++e) acc += dLdR[e] * J[9 * kq + e];
          g_quat[4 * (size_t)l + kq] += acc;
        }
      }
      for (int ch = 0; ch < 3; ++ch) S[ch] += sk->T * sk->alpha * sk->c[ch];
    }
    (void)P; (void)st;
  }
  free(rc.s); free(rc.c);
  ctx_free(&cx);
  return 0;
}
