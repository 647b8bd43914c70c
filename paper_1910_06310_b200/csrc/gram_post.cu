// Gram post-processing on the device: normalize_gram
// (gram.py:98-107) applied to the device-resident N x N matrix before the
// single D2H copy:  K[a,b] / sqrt(K[a,a] K[b,b]), unit diagonal, NaN
// propagates, and a non-NaN diagonal entry <= 0 is an error.
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

}  // namespace mgk
