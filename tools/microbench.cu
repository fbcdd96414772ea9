// Microbenchmarks for the rates the roofline needs that MEASURED_PEAKS.json
// does not hold (SURVEY.md §8(d) "Peaks to use"): FP32 FMA, MUFU ex2,
// float / float4 reductions to global memory (RED through L2) and L2 read
// bandwidth.  Prints one JSON object.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && /tmp/mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int kIters = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;   // keep the chain alive
}

__global__ void k_ex2(float* out, float a) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = -(threadIdx.x & 7) * 1e-3f - i * 1e-4f;
  for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      x[i] = y * a;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;
}

// each warp reduces into a pseudo-random 16-B-aligned row (like the gradient
// scatter: one Gaussian row per pair, lanes on consecutive float4s)
__global__ void k_red4(float4* buf, size_t rows, int row_f4, int per_thread) {
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  uint32_t h = (uint32_t)warp * 2654435761u + 12345u;
  for (int i = 0; i < per_thread; ++i) {
    h = h * 1664525u + 1013904223u;
    const size_t r = h % rows;
    if (lane < row_f4) atomicAdd(buf + r * row_f4 + lane, make_float4(1.f, 1.f, 1.f, 1.f));
  }
}

__global__ void k_red1(float* buf, size_t rows, int row_f, int per_thread) {
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  uint32_t h = (uint32_t)warp * 2654435761u + 777u;
  for (int i = 0; i < per_thread; ++i) {
    h = h * 1664525u + 1013904223u;
    const size_t r = h % rows;
    if (lane < row_f) atomicAdd(buf + r * row_f + lane, 1.f);
  }
}

__global__ void k_l2read(const float4* __restrict__ buf, size_t n, int reps, float* out) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      const float4 v = __ldcg(buf + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[0] = acc.x;
}

template <class F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0, clk_khz = 0, l2 = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  float* out;
  CK(cudaMalloc(&out, 16));
  const int blocks = sms * 8, threads = 256;
  const double thr = (double)blocks * threads;
  const float t_fma = time_ms([&] { k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-4f); });
  const double fma_tflops = thr * kIters * 8 * 2 / (t_fma * 1e-3) / 1e12;
  const float t_ex2 = time_ms([&] { k_ex2<<<blocks, threads>>>(out, 0.999f); });
  const double ex2_tops = thr * (kIters / 4) * 8 / (t_ex2 * 1e-3) / 1e12;
  // reductions into a 144 MB buffer of 120-float rows (the C1 gradient rows)
  const int row_f4 = 30;
  const size_t rows = 300000;
  float4* buf;
  CK(cudaMalloc(&buf, rows * row_f4 * 16));
  CK(cudaMemset(buf, 0, rows * row_f4 * 16));
  const int per = 64;
  const int rblocks = sms * 16;
  const double warps = (double)rblocks * threads / 32;
  const float t_r4 = time_ms([&] { k_red4<<<rblocks, threads>>>(buf, rows, row_f4, per); });
  const double red4_g = warps * per * row_f4 / (t_r4 * 1e-3) / 1e9;
  const float t_r1 = time_ms([&] {
    k_red1<<<rblocks, threads>>>(reinterpret_cast<float*>(buf), rows * 4, 30, per);
  });
  const double red1_g = warps * per * 30 / (t_r1 * 1e-3) / 1e9;
  // L2-resident read bandwidth: 48 MB buffer read 20 times
  const size_t n4 = (48u << 20) / 16;
  const float t_l2 = time_ms([&] { k_l2read<<<sms * 8, 512>>>(buf, n4, 20, out); });
  const double l2_gbs = (double)n4 * 16 * 20 / (t_l2 * 1e-3) / 1e9;
  printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f, \"l2_bytes\": %d,\n"
         " \"ffma_tflops\": %.2f, \"ex2_tops\": %.3f,\n"
         " \"red_f32x4_gops\": %.2f, \"red_f32x4_gbs\": %.1f, \"red_f32_gops\": %.2f,\n"
         " \"l2_read_gbs\": %.0f,\n"
         " \"how\": \"best of 5 CUDA-event timings; FFMA 8 independent chains x 4096 iters x %d threads; "
         "ex2.approx 8 chains; RED: warps reduce float4 (30 lanes) or float (30 lanes) into pseudo-random "
         "120-float rows of a 144 MB buffer (the C1 gradient layout); L2: __ldcg float4 reads of a 48 MB buffer x 20\"}\n",
         sms, clk_khz / 1e3, l2, fma_tflops, ex2_tops, red4_g, red4_g * 16, red1_g, l2_gbs, (int)thr);
  return 0;
}
