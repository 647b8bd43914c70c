// Roofline denominators measured live on the device the solver runs on:
// FP32 FFMA throughput and MUFU.EX2 throughput (the SE edge kernel's co-bound).
// Only used by bench.py to report roofline fractions; not on the solve path.
#include <cuda_runtime.h>

#include "../../include/mgk.h"

namespace {

__global__ void k_ffma(float* out, float a, float b, int iters) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_ex2(float* out, float a, int iters) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
      asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
      asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x2));
      asm("ex2.approx.ftz.f32 %0, %0;" : "+f"(x3));
      x0 *= a; x1 *= a; x2 *= a; x3 *= a;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

}  // namespace

extern "C" int mgk_bench_peaks(int device, double* fp32_tflops, double* ex2_tops) {
  if (cudaSetDevice(device) != cudaSuccess) return MGK_E_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  float* out = nullptr;
  if (cudaMalloc(&out, (size_t)blocks * threads * sizeof(float)) != cudaSuccess) return MGK_E_CUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best_f = 1e30f, best_e = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    float ms;
    cudaEventRecord(e0);
    k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best_f = ms < best_f ? ms : best_f;
    cudaEventRecord(e0);
    k_ex2<<<blocks, threads>>>(out, 0.5f, iters / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) best_e = ms < best_e ? ms : best_e;
  }
  int rc = cudaGetLastError() == cudaSuccess ? MGK_OK : MGK_E_CUDA;
  if (fp32_tflops) *fp32_tflops = 2.0 * 8 * 16 * (double)iters * blocks * threads / (best_f * 1e-3) / 1e12;
  if (ex2_tops) *ex2_tops = 4.0 * 16 * (double)(iters / 4) * blocks * threads / (best_e * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return rc;
}
