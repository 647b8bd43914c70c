// Microbenchmarks for the roofline denominators of the FP32 CUDA-core path:
// FFMA throughput (reg-reg), MUFU.EX2 throughput, LDS gather throughput.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

__global__ void ffma_kernel(float* out, float a, float b, int iters) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  float y = b * 0.5f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      x0 = fmaf(x0, a, y); x1 = fmaf(x1, a, y); x2 = fmaf(x2, a, y); x3 = fmaf(x3, a, y);
      x4 = fmaf(x4, a, y); x5 = fmaf(x5, a, y); x6 = fmaf(x6, a, y); x7 = fmaf(x7, a, y);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void ex2_kernel(float* out, float a, int iters) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 0.1f, x2 = x0 + 0.2f, x3 = x0 + 0.3f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      x0 = exp2f(-x0 * a); x1 = exp2f(-x1 * a); x2 = exp2f(-x2 * a); x3 = exp2f(-x3 * a);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d smemPerSM %zu smemPerBlockOptin %zu regsPerSM %d clock_kHz %d\n", prop.name,
         prop.multiProcessorCount, prop.sharedMemPerMultiprocessor, prop.sharedMemPerBlockOptin,
         prop.regsPerMultiprocessor, clk);
  float* out; CK(cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    ffma_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("FFMA: %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    ex2_kernel<<<blocks, threads>>>(out, 0.5f, iters / 4);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 4.0 * 16 * (double)(iters / 4) * blocks * threads;
    printf("EX2 (with FMUL): %.3f ms  %.2f Tex2/s  per SM per clk @1965: %.2f\n", ms, ops / ms / 1e9,
           ops / (ms * 1e-3) / prop.multiProcessorCount / 1.965e9);
  }
  return 0;
}
