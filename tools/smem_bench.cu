// Shared-memory wavefront costs of the access shapes the warp solvers use: warp-uniform (broadcast)
// LDS.32 / LDS.64 / LDS.128, two-address LDS.128 (half-warps on adjacent records) and the
// conflict-free LDS.32 gather.  Reports warp-instructions per SM cycle (1.0 = one wavefront each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/smem_bench tools/smem_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_lds(float* out, int iters, int stride) {
  __shared__ __align__(16) float4 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float acc = 0.0f;
  int k = (threadIdx.x >> 5) * 7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = (k + u * stride) & 511;
      if constexpr (MODE == 0) {  // broadcast LDS.32
        acc += reinterpret_cast<const float*>(buf)[idx * 4];
      } else if constexpr (MODE == 1) {  // broadcast LDS.64
        const float2 v = reinterpret_cast<const float2*>(buf)[idx * 2];
        acc += v.x * v.y;
      } else if constexpr (MODE == 2) {  // broadcast LDS.128
        const float4 v = buf[idx];
        acc += v.x * v.y + v.z * v.w;
      } else if constexpr (MODE == 3) {  // LDS.128, two addresses (half-warps on adjacent records)
        const float4 v = buf[idx + (lane >> 4)];
        acc += v.x * v.y + v.z * v.w;
      } else if constexpr (MODE == 4) {  // conflict-free LDS.32 gather
        acc += reinterpret_cast<const float*>(buf)[idx * 32 % 4096 + lane];
      } else if constexpr (MODE == 5) {  // LDS.64 gather, consecutive 8-byte words
        const float2 v = reinterpret_cast<const float2*>(buf)[(idx * 32 + lane) & 2047];
        acc += v.x * v.y;
      }
    }
    k += static_cast<int>(acc) & 1;  // data dependence keeps the loads live
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE>
float run(float* out, int sms, int clk_khz) {
  const int blocks = sms * 4, threads = 256, iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_lds<MODE><<<blocks, threads>>>(out, 16, 1);
  cudaEventRecord(e0);
  k_lds<MODE><<<blocks, threads>>>(out, iters, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warp_instr = (double)blocks * (threads / 32) * iters * 16;
  const double sm_cycles = ms * 1e-3 * clk_khz * 1e3 * sms;
  return (float)(warp_instr / sm_cycles);
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, prop.multiProcessorCount * 4 * 256 * sizeof(float));
  const char* names[] = {"bcast LDS.32", "bcast LDS.64", "bcast LDS.128", "2-addr LDS.128", "gather LDS.32",
                         "gather LDS.64"};
  float r[6];
  for (int rep = 0; rep < 2; ++rep) {
    r[0] = run<0>(out, prop.multiProcessorCount, clk);
    r[1] = run<1>(out, prop.multiProcessorCount, clk);
    r[2] = run<2>(out, prop.multiProcessorCount, clk);
    r[3] = run<3>(out, prop.multiProcessorCount, clk);
    r[4] = run<4>(out, prop.multiProcessorCount, clk);
    r[5] = run<5>(out, prop.multiProcessorCount, clk);
  }
  for (int i = 0; i < 6; ++i) printf("%-16s %.3f warp-LDS per SM cycle (at the nominal clock %d kHz)\n", names[i], r[i], clk);
  return 0;
}
