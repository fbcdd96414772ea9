// rg_api.cu -- the C-ABI entry points of include/rg.h: argument validation
// (before anything is enqueued), workspace layout, launch, error mapping.
#include <cstdlib>
#include <cstring>

#include "rg_internal.cuh"

#include <atomic>
#include <mutex>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: a no-op unless a profiler injects

using namespace rg;

namespace {
// one NVTX range per C-ABI call that enqueues GPU work (SURVEY §5 tracing)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace
#define RG_NVTX(name) NvtxRange nvtx_range_(name)

namespace rg {
// diagnostic: number of kernels this library enqueued (process-wide)
static std::atomic<unsigned long long> g_launches{0};
void count_launches(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace rg

namespace {

// ---- rg_build_bvh as a CUDA graph: the ~30 launches and memsets of a
// build are captured once per (parameters, config, workspace, device) on a private
// stream and replayed with one cudaGraphLaunch on the caller's stream; parameter
// VALUES are read when the graph runs, so an optimiser updating them in place keeps
// hitting the cache.  A small round-robin cache under a mutex; RG_NO_GRAPH=1 in the
// environment (read once) launches the kernels directly.
struct GraphKey {
  rg_gaussians g;
  rg_config c;
  void* ws;
  int dev, pad_;
};
struct GraphEntry {
  GraphKey k;
  cudaGraphExec_t exec;
  unsigned launches;
};
constexpr int kGraphCache = 8;
std::mutex g_graph_mu;
GraphEntry g_graphs[kGraphCache];
int g_graph_n = 0, g_graph_next = 0;

bool graphs_enabled() {
  static const bool on = std::getenv("RG_NO_GRAPH") == nullptr;
  return on;
}

cudaError_t build_graph_launch(const rg_gaussians& g, const rg_config& c, char* w,
                               const BvhLayout& L, cudaStream_t st) {
  GraphKey k;
  std::memset(&k, 0, sizeof(k));
  k.g = g;
  k.c = c;
  k.ws = w;
  cudaGetDevice(&k.dev);
  std::lock_guard<std::mutex> lock(g_graph_mu);
  for (int i = 0; i < g_graph_n; ++i)
    if (std::memcmp(&g_graphs[i].k, &k, sizeof(k)) == 0) {
      count_launches(g_graphs[i].launches);
      return cudaGraphLaunch(g_graphs[i].exec, st);
    }
  cudaStream_t cap;
  if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    return launch_build(g, c, w, L, st);
  }
  const unsigned long long before = g_launches.load();
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed);
  if (e == cudaSuccess) {
    e = launch_build(g, c, w, L, cap);
    const cudaError_t e2 = cudaStreamEndCapture(cap, &graph);
    if (e == cudaSuccess) e = e2;
  }
  cudaStreamDestroy(cap);
  const unsigned n_launch = (unsigned)(g_launches.load() - before);
  g_launches.fetch_sub(n_launch, std::memory_order_relaxed);   // captured, not launched
  cudaGraphExec_t exec = nullptr;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (e != cudaSuccess) {      // capture unavailable: launch directly
    cudaGetLastError();
    return launch_build(g, c, w, L, st);
  }
  GraphEntry* slot;
  if (g_graph_n < kGraphCache) {
    slot = &g_graphs[g_graph_n++];
  } else {
    slot = &g_graphs[g_graph_next];
    g_graph_next = (g_graph_next + 1) % kGraphCache;
    cudaGraphExecDestroy(slot->exec);
  }
  slot->k = k;
  slot->exec = exec;
  slot->launches = n_launch;
  count_launches(n_launch);
  return cudaGraphLaunch(exec, st);
}

bool config_ok(const rg_config* c) {
  if (!c) return false;
  if (!(c->dt > 0.0f) || !isfinite(c->dt)) return false;
  if (c->slab_samples < 1 || c->slab_samples > 32) return false;
  if (!(c->sigma_eps > 0.0f) || !isfinite(c->sigma_eps)) return false;
  if (!(c->t_eps >= 0.0f && c->t_eps < 1.0f)) return false;
  if (c->hit_capacity < 1 || c->hit_capacity > 4096) return false;
  if (c->radius_mode != 0 && c->radius_mode != 1) return false;
  if (c->radius_mode == 1 && !(c->k_sigma > 0.0f)) return false;
  if (!isfinite(c->t_near)) return false;
  if (c->basis < 0 || c->basis > 5) return false;
  if (c->basis != 0 && c->radius_mode != 0) return false;
  if (c->list_capacity < 0) return false;
  return true;
}

bool gaussians_ok(const rg_gaussians* g) {
  if (!g || g->n < 0) return false;
  if (g->sh_degree < 0 || g->sh_degree > kMaxDeg) return false;
  if (g->sg_count < 0 || g->sg_count > kMaxLobes) return false;
  if (g->n == 0) return true;
  if (!g->mean || !g->quat || !g->scale || !g->density || !g->sh) return false;
  if (g->sg_count > 0 && (!g->sg_amp || !g->sg_sharp || !g->sg_axis)) return false;
  return true;
}

bool bvh_ok(const rg_bvh* b, const rg_gaussians* g) {
  if (!b || !b->root_box) return false;
  if (b->n != g->n || b->sh_degree != g->sh_degree || b->sg_count != g->sg_count) return false;
  if (b->n > 0 && (!b->geom || !b->app || !b->order || !b->wide || (b->n > 1 && !b->nodes)))
    return false;
  return true;
}

bool rays_ok(const rg_rays* r, const rg_camera* cam) {
  if ((r == nullptr) == (cam == nullptr)) return false;
  if (r) return r->n >= 0 && (r->n == 0 || (r->origin && r->dir));
  if (cam->x0 < 0 || cam->y0 < 0 || cam->x1 < cam->x0 || cam->y1 < cam->y0) return false;
  if (!(cam->fx != 0.0f) || !(cam->fy != 0.0f)) return false;
  if (cam->spp != 1 && cam->spp != 4) return false;
  if (cam->tile != 0) {
    if (cam->tile < 2 || cam->tile > 256 || (cam->tile & 1) || cam->spp != 1) return false;
    if (cam->shards < 1 || cam->shard < 0 || cam->shard >= cam->shards) return false;
  }
  if (camera_ray_slots(*cam) > 0x7FFFFFFF) return false;
  return true;
}

}  // namespace

extern "C" {

const char* rg_status_string(rg_status s) {
  switch (s) {
    case RG_OK: return "ok";
    case RG_ERR_INVALID_ARG: return "invalid argument";
    case RG_ERR_WORKSPACE_TOO_SMALL: return "workspace too small";
    case RG_ERR_CUDA: return "CUDA error";
    case RG_ERR_NOT_IMPLEMENTED: return "not implemented";
  }
  return "unknown status";
}

unsigned long long rg_kernel_launches(void) { return g_launches.load(); }

const char* rg_version(void) {
  return "libraygauss abi=1 sm_100a (LBVH + slab ray casting, fwd+bwd)";
}

size_t rg_bvh_workspace_bytes(int32_t n, int32_t sh_degree, int32_t sg_count) {
  if (n < 0 || sh_degree < 0 || sh_degree > kMaxDeg || sg_count < 0 || sg_count > kMaxLobes)
    return 0;
  return bvh_layout(n, sh_degree, sg_count).total;
}

rg_status rg_build_bvh(const rg_gaussians* g, const rg_config* cfg, void* ws, size_t ws_bytes,
                       rg_bvh* out, void* stream) {
  RG_NVTX("rg_build_bvh");
  if (!gaussians_ok(g) || !config_ok(cfg) || !ws || !out) return RG_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return RG_ERR_INVALID_ARG;
  if (g->n >= kMaxLeafPos) return RG_ERR_INVALID_ARG;   // leaf-range encoding
  const BvhLayout L = bvh_layout(g->n, g->sh_degree, g->sg_count);
  if (ws_bytes < L.total) return RG_ERR_WORKSPACE_TOO_SMALL;
  char* w = static_cast<char*>(ws);
  cudaGetLastError();   // clear sticky-free previous errors
  const cudaError_t e = graphs_enabled()
                            ? build_graph_launch(*g, *cfg, w, L, static_cast<cudaStream_t>(stream))
                            : launch_build(*g, *cfg, w, L, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return RG_ERR_CUDA;
  rg_bvh b;
  std::memset(&b, 0, sizeof(b));
  b.n = g->n;
  b.sh_degree = g->sh_degree;
  b.sg_count = g->sg_count;
  b.app_stride = app_stride(g->sh_degree, g->sg_count);
  b.geom = w + L.geom;
  b.app = reinterpret_cast<const float*>(w + L.app);
  b.nodes = w + L.nodes;
  b.wide = w + L.wide;
  b.wide_info = reinterpret_cast<const int32_t*>(w + L.wcounts);
  b.leaf_box = reinterpret_cast<const float*>(w + L.leaf_box);
  b.root_box = reinterpret_cast<const float*>(w + L.root_box);
  b.codes = reinterpret_cast<const uint32_t*>(w + L.codes);
  b.sorted_codes = reinterpret_cast<const uint32_t*>(w + L.keys_a);
  b.order = reinterpret_cast<const uint32_t*>(w + L.vals_a);
  *out = b;
  return RG_OK;
}

rg_status rg_refit_bvh(const rg_gaussians* g, const rg_config* cfg, void* ws, size_t ws_bytes,
                       rg_bvh* bvh, void* stream) {
  RG_NVTX("rg_refit_bvh");
  if (!gaussians_ok(g) || !config_ok(cfg) || !ws || !bvh) return RG_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return RG_ERR_INVALID_ARG;
  const BvhLayout L = bvh_layout(g->n, g->sh_degree, g->sg_count);
  if (ws_bytes < L.total) return RG_ERR_WORKSPACE_TOO_SMALL;
  char* w = static_cast<char*>(ws);
  // same topology: built by rg_build_bvh on this workspace with the same sizes
  if (bvh->n != g->n || bvh->sh_degree != g->sh_degree || bvh->sg_count != g->sg_count ||
      bvh->geom != static_cast<const void*>(w + L.geom) || bvh->wide != static_cast<const void*>(w + L.wide))
    return RG_ERR_INVALID_ARG;
  cudaGetLastError();
  const cudaError_t e = launch_refit(*g, *cfg, w, L, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RG_OK : RG_ERR_CUDA;
}

namespace {
bool arrays_ok(const rg_gaussian_grads* a, int32_t n, int32_t G) {
  if (!a) return false;
  if (n == 0) return true;
  if (!a->mean || !a->quat || !a->scale || !a->density || !a->sh) return false;
  if (G > 0 && (!a->sg_amp || !a->sg_sharp || !a->sg_axis)) return false;
  return true;
}
}  // namespace

rg_status rg_adam_step(const rg_adam_config* cfg, const rg_gaussian_grads* grad_act,
                       const rg_param_arrays* raw, const rg_param_arrays* m,
                       const rg_param_arrays* v, const rg_param_arrays* act_out, void* stream) {
  RG_NVTX("rg_adam_step");
  if (!cfg || cfg->n < 0 || cfg->sh_degree < 0 || cfg->sh_degree > kMaxDeg || cfg->sg_count < 0 ||
      cfg->sg_count > kMaxLobes || cfg->step < 1)
    return RG_ERR_INVALID_ARG;
  if (!(cfg->beta1 >= 0.f && cfg->beta1 < 1.f) || !(cfg->beta2 >= 0.f && cfg->beta2 < 1.f) ||
      !(cfg->eps > 0.f))
    return RG_ERR_INVALID_ARG;
  const int nc = (cfg->sh_degree + 1) * (cfg->sh_degree + 1);
  if (cfg->sh_active < 1 || cfg->sh_active > nc || cfg->sg_active < 0 ||
      cfg->sg_active > cfg->sg_count)
    return RG_ERR_INVALID_ARG;
  for (int k = 0; k < RG_LR_COUNT; ++k)
    if (!(cfg->lr[k] >= 0.f) || !isfinite(cfg->lr[k])) return RG_ERR_INVALID_ARG;
  for (const rg_gaussian_grads* a : {grad_act, raw, m, v, act_out})
    if (!arrays_ok(a, cfg->n, cfg->sg_count)) return RG_ERR_INVALID_ARG;
  cudaGetLastError();
  const cudaError_t e = launch_adam(*cfg, *grad_act, *raw, *m, *v, *act_out,
                                    static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RG_OK : RG_ERR_CUDA;
}

size_t rg_dssim_workspace_bytes(int32_t width, int32_t height) {
  if (width < 0 || height < 0) return 0;
  return dssim_workspace_bytes(height, width);
}

rg_status rg_l1_dssim_loss_grad(const float* rgb, const float* target, int32_t width,
                                int32_t height, float lambda, float* d_rgb, float* loss, void* ws,
                                size_t ws_bytes, void* stream) {
  RG_NVTX("rg_l1_dssim_loss_grad");
  if (width < 0 || height < 0 || !(lambda >= 0.f && lambda <= 1.f)) return RG_ERR_INVALID_ARG;
  if ((size_t)width * height == 0) return RG_OK;
  if (!rgb || !target || !d_rgb || !ws) return RG_ERR_INVALID_ARG;
  if (ws_bytes < dssim_workspace_bytes(height, width)) return RG_ERR_WORKSPACE_TOO_SMALL;
  cudaGetLastError();
  const cudaError_t e = launch_l1_dssim(rgb, target, height, width, lambda, d_rgb, loss,
                                        static_cast<float*>(ws), static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RG_OK : RG_ERR_CUDA;
}

rg_status rg_supersample_resolve(const float* rgb_rays, int64_t n_pixels, int32_t spp,
                                 float* rgb_px, void* stream) {
  RG_NVTX("rg_supersample_resolve");
  if (n_pixels < 0 || spp < 1 || (n_pixels > 0 && (!rgb_rays || !rgb_px))) return RG_ERR_INVALID_ARG;
  cudaGetLastError();
  return launch_ss_resolve(rgb_rays, n_pixels, spp, rgb_px, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess ? RG_OK : RG_ERR_CUDA;
}

rg_status rg_supersample_spread(const float* d_px, int64_t n_pixels, int32_t spp, float* d_rays,
                                void* stream) {
  RG_NVTX("rg_supersample_spread");
  if (n_pixels < 0 || spp < 1 || (n_pixels > 0 && (!d_px || !d_rays))) return RG_ERR_INVALID_ARG;
  cudaGetLastError();
  return launch_ss_spread(d_px, n_pixels, spp, d_rays, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess ? RG_OK : RG_ERR_CUDA;
}

rg_status rg_densify_accumulate(const float* grad_mean, int32_t n, float* acc, int32_t* cnt,
                                void* stream) {
  RG_NVTX("rg_densify_accumulate");
  if (n < 0 || (n > 0 && (!grad_mean || !acc || !cnt))) return RG_ERR_INVALID_ARG;
  cudaGetLastError();
  return launch_dens_acc(grad_mean, n, acc, cnt, static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? RG_OK : RG_ERR_CUDA;
}

size_t rg_densify_workspace_bytes(int32_t n) { return n < 0 ? 0 : densify_workspace_bytes(n); }

rg_status rg_densify_plan(const rg_gaussians* g, const float* acc, const int32_t* cnt,
                          float grad_eps, float extent, float sigma_eps, float percent_dense,
                          int32_t* action, void* ws, size_t ws_bytes, int32_t* counts,
                          void* stream) {
  RG_NVTX("rg_densify_plan");
  if (!gaussians_ok(g) || !counts || !ws) return RG_ERR_INVALID_ARG;
  if (g->n > 0 && (!acc || !cnt || !action)) return RG_ERR_INVALID_ARG;
  if (!isfinite(grad_eps) || !(extent >= 0.f) || !isfinite(sigma_eps) || !(percent_dense >= 0.f))
    return RG_ERR_INVALID_ARG;
  if (ws_bytes < densify_workspace_bytes(g->n)) return RG_ERR_WORKSPACE_TOO_SMALL;
  cudaGetLastError();
  return launch_dens_plan(*g, acc, cnt, grad_eps, extent, sigma_eps, percent_dense, action,
                          static_cast<char*>(ws), counts, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess ? RG_OK : RG_ERR_CUDA;
}

rg_status rg_densify_apply(const rg_gaussians* g, const rg_param_arrays* in,
                           const int32_t* action, const void* ws, const int32_t* counts,
                           const float* z, int32_t mode, const rg_param_arrays* out, void* stream) {
  RG_NVTX("rg_densify_apply");
  if (!gaussians_ok(g) || !out || !ws || !counts || mode < 0 || mode > 2) return RG_ERR_INVALID_ARG;
  if (g->n > 0 && (!action || !z)) return RG_ERR_INVALID_ARG;
  rg_gaussian_grads src;
  if (in) {
    src = *in;
  } else {
    if (mode != 0) return RG_ERR_INVALID_ARG;
    src = rg_gaussian_grads{const_cast<float*>(g->mean), const_cast<float*>(g->quat),
                            const_cast<float*>(g->scale), const_cast<float*>(g->density),
                            const_cast<float*>(g->sh), const_cast<float*>(g->sg_amp),
                            const_cast<float*>(g->sg_sharp), const_cast<float*>(g->sg_axis)};
  }
  if (!arrays_ok(&src, g->n, g->sg_count) || !arrays_ok(out, 1, g->sg_count)) return RG_ERR_INVALID_ARG;
  cudaGetLastError();
  return launch_dens_apply(*g, src, *out, action, static_cast<const char*>(ws), counts, z, mode,
                           static_cast<cudaStream_t>(stream)) == cudaSuccess ? RG_OK : RG_ERR_CUDA;
}

int64_t rg_camera_ray_count(const rg_camera* cam) {
  if (!cam || !rays_ok(nullptr, cam)) return 0;
  return camera_ray_slots(*cam);
}

rg_status rg_camera_rays(const rg_camera* cam, float* origin, float* dir, void* stream) {
  RG_NVTX("rg_camera_rays");
  if (!cam || !rays_ok(nullptr, cam)) return RG_ERR_INVALID_ARG;
  const int64_t n = camera_ray_slots(*cam);
  if (n > 0 && (!origin || !dir)) return RG_ERR_INVALID_ARG;
  return launch_camera_rays(*cam, origin, dir, static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? RG_OK
             : RG_ERR_CUDA;
}

rg_status rg_render_forward(const rg_gaussians* g, const rg_bvh* bvh, const rg_config* cfg,
                            const rg_rays* rays, const rg_camera* cam, float* rgb, float* T,
                            int32_t* replay, void* fetch_log, size_t log_bytes,
                            rg_stats* stats, int32_t debug_rays, int32_t debug_cap,
                            int32_t* debug_counts, int32_t* debug_records, void* stream) {
  RG_NVTX("rg_render_forward");
  if (!gaussians_ok(g) || !config_ok(cfg) || !bvh_ok(bvh, g) || !rays_ok(rays, cam))
    return RG_ERR_INVALID_ARG;
  if (cfg->basis != 0 && cfg->slab_samples < 5) return RG_ERR_NOT_IMPLEMENTED;
  const int64_t n = rays ? rays->n : camera_ray_slots(*cam);
  if (n > 0 && (!rgb || !T || !replay)) return RG_ERR_INVALID_ARG;
  if (debug_records && (debug_rays < 0 || debug_cap < 1 || !debug_counts))
    return RG_ERR_INVALID_ARG;
  if (fetch_log && (log_bytes < rg_fetch_log_bytes((int32_t)n, 1) ||
                    (reinterpret_cast<uintptr_t>(fetch_log) & 255) != 0))
    return RG_ERR_INVALID_ARG;
  const cudaError_t e = launch_forward(*g, *bvh, *cfg, rays, cam, rgb, T, replay, fetch_log,
                                       log_bytes, stats,
                                       debug_rays, debug_cap, debug_counts, debug_records,
                                       static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RG_OK : RG_ERR_CUDA;
}

size_t rg_fetch_log_bytes(int32_t n_rays, int32_t pairs_per_ray) {
  if (n_rays < 0) return 0;
  const size_t ppr = pairs_per_ray > 0 ? (size_t)pairs_per_ray : 48;
  // per pair: a 48-B slot plus 2 stored window samples of 16 B (rg_internal.cuh split)
  return fetch_log_header_bytes(n_rays) + 80 * ppr * (size_t)(n_rays > 0 ? n_rays : 1);
}

size_t rg_backward_workspace_bytes(int32_t n, int32_t sh_degree, int32_t sg_count) {
  if (n < 0 || sh_degree < 0 || sh_degree > kMaxDeg || sg_count < 0 || sg_count > kMaxLobes)
    return 0;
  return sizeof(float) * (size_t)grad_stride(sh_degree, sg_count) * (size_t)(n > 0 ? n : 1);
}

rg_status rg_render_backward(const rg_gaussians* g, const rg_bvh* bvh, const rg_config* cfg,
                             const rg_rays* rays, const rg_camera* cam, const float* rgb,
                             const float* T, const int32_t* replay, const void* fetch_log,
                             size_t log_bytes, const float* d_rgb,
                             const rg_gaussian_grads* grads, rg_stats* stats, void* ws,
                             size_t ws_bytes, void* stream) {
  RG_NVTX("rg_render_backward");
  if (!gaussians_ok(g) || !config_ok(cfg) || !bvh_ok(bvh, g) || !rays_ok(rays, cam) || !grads)
    return RG_ERR_INVALID_ARG;
  if (cfg->basis != 0 && cfg->slab_samples < 5) return RG_ERR_NOT_IMPLEMENTED;
  const int64_t n = rays ? rays->n : camera_ray_slots(*cam);
  if (n > 0 && (!rgb || !replay || !d_rgb)) return RG_ERR_INVALID_ARG;
  if (!ws || (reinterpret_cast<uintptr_t>(ws) & 15) != 0) return RG_ERR_INVALID_ARG;
  if (ws_bytes < rg_backward_workspace_bytes(g->n, g->sh_degree, g->sg_count))
    return RG_ERR_WORKSPACE_TOO_SMALL;
  if (fetch_log && (log_bytes < rg_fetch_log_bytes((int32_t)n, 1) ||
                    (reinterpret_cast<uintptr_t>(fetch_log) & 255) != 0))
    return RG_ERR_INVALID_ARG;
  const cudaError_t e = launch_backward(*g, *bvh, *cfg, rays, cam, rgb, T, replay, fetch_log,
                                        log_bytes, d_rgb, *grads,
                                        stats, static_cast<float*>(ws),
                                        static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? RG_OK : RG_ERR_CUDA;
}

rg_status rg_l1_loss_grad(const float* rgb, const float* target, int64_t n_values, float scale,
                          float* d_rgb, float* loss, void* stream) {
  RG_NVTX("rg_l1_loss_grad");
  if (n_values < 0 || (n_values > 0 && (!rgb || !target || !d_rgb || !loss)))
    return RG_ERR_INVALID_ARG;
  return launch_l1(rgb, target, n_values, scale, d_rgb, loss, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess
             ? RG_OK
             : RG_ERR_CUDA;
}

}  // extern "C"
