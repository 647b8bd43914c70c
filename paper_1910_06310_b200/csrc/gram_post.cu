// Gram post-processing on the device: normalize_gram
// (gram.py:98-107) applied to the device-resident N x N matrix before the
// single D2H copy:  K[a,b] / sqrt(K[a,a] K[b,b]), unit diagonal, NaN
// propagates, and a non-NaN diagonal entry <= 0 is an error.
#include <algorithm>
#include <cmath>

#include "mgk_internal.h"

namespace mgk {

__global__ void k_gram_diag(const double* __restrict__ K, int64_t G, double* __restrict__ diag, int* __restrict__ bad) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= G) return;
  const double d = K[i * G + i];
  diag[i] = d;
  if (!isnan(d) && d <= 0.0) atomicExch(bad, 1);
}

__global__ void k_gram_normalize(double* __restrict__ K, int64_t G, const double* __restrict__ diag) {
  const int64_t total = G * G;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = e / G, b = e - a * G;
    const double da = diag[a], db = diag[b];
    K[e] = (a == b) ? (isnan(da) ? da : 1.0) : K[e] / sqrt(da * db);
  }
}

cudaError_t launch_gram_normalize(double* K, int64_t G, double* diag, int* bad, int num_sms, cudaStream_t stream,
                                  bool* nonpositive) {
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  k_gram_diag<<<(unsigned)((G + 255) / 256), 256, 0, stream>>>(K, G, diag, bad);
  int h = 0;
  e = cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return e;
  *nonpositive = h != 0;
  if (h) return cudaSuccess;
  k_gram_normalize<<<num_sms * 8, 256, 0, stream>>>(K, G, diag);
  return cudaGetLastError();
}

// Mirrored scatter of compact per-pair results into a device-resident Gram (gram.py:86-90): the
// collective-free assembly step of a sharded Gram once every rank's records sit on one device.
__global__ void k_gram_assemble(int64_t npairs, const int32_t* __restrict__ pa, const int32_t* __restrict__ pb,
                                const double* __restrict__ value, const int32_t* __restrict__ iters,
                                const uint8_t* __restrict__ conv, int64_t G, double* __restrict__ K,
                                int32_t* __restrict__ K_iters, uint8_t* __restrict__ K_conv) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < npairs; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = pa[k], b = pb[k];
    if (a < 0 || b < 0) continue;  // padding records
    const bool c = conv[k] != 0;
    const double v = c ? value[k] : __longlong_as_double(0x7ff8000000000000ll);
    if (K) K[a * G + b] = K[b * G + a] = v;
    if (K_iters) K_iters[a * G + b] = K_iters[b * G + a] = iters[k];
    if (K_conv) K_conv[a * G + b] = K_conv[b * G + a] = c;
  }
}

cudaError_t launch_gram_assemble(int64_t npairs, const int32_t* pa, const int32_t* pb, const double* value,
                                 const int32_t* iters, const uint8_t* conv, int64_t G, double* K, int32_t* K_iters,
                                 uint8_t* K_conv, int num_sms, cudaStream_t stream) {
  if (npairs <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((npairs + 255) / 256, (int64_t)num_sms * 16);
  k_gram_assemble<<<(unsigned)blocks, 256, 0, stream>>>(npairs, pa, pb, value, iters, conv, G, K, K_iters, K_conv);
  return cudaGetLastError();
}

}  // namespace mgk
