/*
 * rg_oracle.h -- plain, slow, single-threaded CPU ORACLE of the RayGauss hot path
 * (arXiv 2408.03356).  TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke()
 * and bench.py (cpu_baseline leg and --impl reference) may load it.  It shares no
 * code with the CUDA library (paper_2408_03356_b200/csrc) and includes none of its
 * headers; the product path never calls it.
 *
 * Precision policy (task rule "where floating point decides an
 * integer, both sides take that decision in the same precision"):
 *   - every quantity that DECIDES a set or an integer is computed in IEEE fp32
 *     with the explicit operation sequences of DESIGN.md "ARITH" (compiled with
 *     -ffp-contract=off, fmaf only where ARITH says fma): rotation R(q),
 *     M = S^-1 R^T, support radius r^2, padded AABBs, Morton codes, ray setup,
 *     scene-bbox clip, sample positions t_k, slab bounds, the per-(ray,Gaussian)
 *     support interval [t_entry, t_exit];
 *   - every VALUE (density weights, SH/SG colour, compositing, gradients) is fp64,
 *     written directly from the paper's equations.
 *
 * Parity pins for every function live in tests/test_oracle_*.py.
 */
#ifndef RG_ORACLE_H
#define RG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t n, sh_degree, sg_count, pad_;
  const float *mean;      /* [n,3] */
  const float *quat;      /* [n,4] (w,x,y,z) -- consumed as given (caller normalises) */
  const float *scale;     /* [n,3] */
  const float *density;   /* [n]   sigma-tilde */
  const float *sh;        /* [n,(deg+1)^2,3] */
  const float *sg_amp;    /* [n,G,3] */
  const float *sg_sharp;  /* [n,G] */
  const float *sg_axis;   /* [n,G,3] */
} og_gaussians;

typedef struct {
  float dt;              /* Delta t */
  int32_t slab_samples;  /* B */
  float sigma_eps;       /* sigma_eps (Eq.16) */
  float t_eps;           /* T_eps */
  int32_t hit_capacity;  /* n_max = K */
  int32_t radius_mode;   /* 0: r = phi^-1(sigma_eps/sigma); 1: r = k_sigma */
  float k_sigma;
  float t_near;
  float background[3];
  int32_t basis;         /* basis function phi: 0 Gaussian, 1 Bump, 2 Wendland,
                            3 inverse multiquadric, 4 inverse quadratic, 5 C0-Matern */
} og_config;

typedef struct {
  int64_t slabs;      /* non-empty slabs integrated */
  int64_t pairs;      /* distinct (ray, Gaussian) members of integrated slab sets */
  int64_t evals;      /* (sample, Gaussian) contributions: t_entry <= t_k <= t_exit */
  int64_t samples;    /* composited samples (sigma_k > 0) */
  int64_t overflows;  /* slabs whose hit set exceeded K */
  int64_t rays_hit;   /* rays with t0 < t1 */
} og_counters;

/* ---- fp32 decision path (ARITH-1..9) ---------------------------------- */
void og_rotation_f32(const float q[4], float R[9]);
/* per-Gaussian: M (9), r2, padded AABB lo/hi (6), flags (bit0 valid, bit1 active) */
void og_prim_setup(const og_gaussians* g, const og_config* c, int32_t i,
                   float M[9], float* r2, float box[6], int32_t* flags);
/* segment/ellipsoid support interval; returns 1 on hit and writes te, tx */
int32_t og_isect(const float M[9], float r2, const float mu[3], const float o[3],
                 const float d[3], float* te, float* tx);
/* Morton codes of the means (ARITH-6); codes of invalid Gaussians = 0xFFFFFFFF.
   fine: the next 7 bits per axis (floor(u 2^17) & 127) interleaved into 21 bits, the
   sort's tie-break inside an equal-code run (L34; 0 for invalid) */
void og_morton(const og_gaussians* g, const og_config* c, uint32_t* codes, uint32_t* fine,
               float lo[3], float hi[3]);
/* stable sort by (code, fine) -> order[pos] = original index; sorted codes out */
void og_sort(int32_t n, const uint32_t* codes, const uint32_t* fine, uint32_t* order,
             uint32_t* sorted);
/* Karras hierarchy (recursive top-down definition); children: >=0 internal,
   <0 leaf ~pos.  left/right have n-1 entries. */
void og_karras(int32_t n, const uint32_t* sorted_codes, int32_t* left, int32_t* right);
/* refit: node boxes [(n-1)*6] from leaf boxes in sorted order [n*6]; root[6] */
void og_refit(int32_t n, const int32_t* left, const int32_t* right,
              const float* leaf_boxes, float* node_boxes, float root[6]);
/* pinhole rays (ARITH-7); c2w row-major 3x4; pixel rect [x0,x1)x[y0,y1) row-major */
void og_camera_rays(int32_t width, int32_t height, float fx, float fy, float cx, float cy,
                    const float* c2w, int32_t x0, int32_t y0, int32_t x1, int32_t y1,
                    float* o, float* d);
/* RayGauss4x (L29): spp rays per pixel, spp = 1 (the centre,
   identical to og_camera_rays) or 4 (2x2 grid at offsets 1/4, 3/4 of the pixel);
   ray index = pixel index * spp + s, s = sx + 2 sy */
void og_camera_rays_spp(int32_t width, int32_t height, float fx, float fy, float cx, float cy,
                        const float* c2w, int32_t x0, int32_t y0, int32_t x1, int32_t y1,
                        int32_t spp, float* o, float* d);
/* scene-bbox clip (ARITH-8): returns 1 if t0 < t1 */
int32_t og_clip(const float box[6], const float o[3], const float d[3], float t_near,
                float* t0, float* t1);

/* basis function phi(r) at q = r^2 (fp64), and psi = -2 sigma~ dphi/dq
   (the weight's sensitivity to q; psi = w for the Gaussian) */
double og_basis_phi(int32_t basis, double q);
double og_basis_psi(int32_t basis, double sigma, double q);

/* ---- BVH (own implementation: O3) ------------------------------------- */
typedef struct og_bvh og_bvh;
og_bvh* og_build(const og_gaussians* g, const og_config* c);
void og_free(og_bvh* b);
/* views into the BVH: may pass NULL for any */
void og_bvh_views(const og_bvh* b, const uint32_t** codes_unsorted, const uint32_t** sorted_codes,
                  const uint32_t** order, const int32_t** left, const int32_t** right,
                  const float** leaf_boxes_sorted, const float** node_boxes, const float** root,
                  const float** mean_lo, const float** mean_hi, const uint32_t** fine);

/* ---- forward / backward (fp64 values) --------------------------------- */
/* mode 0: plain per-sample definition: every active Gaussian tested at every
           sample (no slabs for the sets, no BVH, no truncation), slab-granular
           termination -- SURVEY.md §8(c) "plain definition of the result";
   mode 1: Alg. 2 slab loop, per-slab hit set by brute force over all Gaussians;
   mode 2: Alg. 2 slab loop, per-slab hit set from the oracle's own BVH.
   dec: if non-NULL, every decision (sets, bbox, intervals) is taken from dec
        while values come from g (used by the finite-difference pins).
   force_s_term: if non-NULL, the termination slab of each ray is forced.
   dump: per ray up to dump_cap (slab, original index) records of the slab sets. */
int32_t og_render(const og_gaussians* g, const og_gaussians* dec, const og_config* c,
                  int32_t mode, const og_bvh* bvh, int32_t n_rays,
                  const float* ray_o, const float* ray_d, const int32_t* force_s_term,
                  double* rgb, double* T, int32_t* s_term, og_counters* cnt,
                  int32_t dump_cap, int32_t* dump_counts, int32_t* dump);

/* exact gradient (a.e.) of sum_r <d_rgb_r, rgb_r> w.r.t. the activated inputs,
   decisions held fixed (termination replayed).  grads are ACCUMULATED (+=). */
int32_t og_backward(const og_gaussians* g, const og_config* c, int32_t mode,
                    const og_bvh* bvh, int32_t n_rays, const float* ray_o,
                    const float* ray_d, const double* d_rgb,
                    double* g_mean, double* g_quat, double* g_scale, double* g_density,
                    double* g_sh, double* g_sg_amp, double* g_sg_sharp, double* g_sg_axis);

/* fp64 colour c_l(d) of Gaussian i (Eq. 14-15) */
void og_color(const og_gaussians* g, int32_t i, const double d[3], double rgb[3]);
/* fp64 real SH basis values (3DGS convention, L10); out[(deg+1)^2] */
void og_sh_basis(int32_t degree, const double d[3], double* out);

#ifdef __cplusplus
}
#endif
#endif
