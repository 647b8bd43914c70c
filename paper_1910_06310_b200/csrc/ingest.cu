// Device graph ingestion: the spatial_graph cutoff builder
// (graphio.py:211-240) for a batch of point clouds.  Pairs i < j closer than
// the cutoff become edges in (i, j) lexicographic order with
// w = (1 - (d / cutoff)^2)^2 and label d.  Edges and d are bit-identical to the
// reference's float64 numpy evaluation, d = sqrt((dx*dx + dy*dy) + dz*dz) with
// every operation rounded separately (no FMA contraction, explicit _rn
// intrinsics); w uses correctly rounded squares, within 1e-13 of numpy's
// scalar ``** 2`` (libm pow, not correctly rounded; 1 - t^2 amplifies its ulp).
//
//   k_spatial_rows  warp per point (row i): ballot-count of j > i in range
//   host scan       row starts
//   k_spatial_fill  warp per row: ballot prefix places the row's edges in j order
#include <vector>

#include "../../include/mgk.h"
#include "mgk_internal.h"

namespace mgk {

__device__ __forceinline__ double pair_dist(const double* pi, const double* pj, int dim) {
  double acc = 0.0;
  for (int c = 0; c < dim; ++c) {
    const double x = __dsub_rn(pi[c], pj[c]);
    const double sq = __dmul_rn(x, x);
    acc = c == 0 ? sq : __dadd_rn(acc, sq);
  }
  return __dsqrt_rn(acc);
}

__global__ void k_spatial_rows(int64_t total, const int32_t* __restrict__ node_graph,
                               const int64_t* __restrict__ node_off, const double* __restrict__ pts, int dim,
                               double cutoff, int32_t* __restrict__ rowcount) {
  const int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= total) return;
  const int g = node_graph[v];
  const int64_t n0 = node_off[g], n1 = node_off[g + 1];
  const double* pi = pts + v * dim;
  int cnt = 0;
  for (int64_t base = v + 1; base < n1; base += 32) {
    const int64_t j = base + lane;
    const bool hit = j < n1 && pair_dist(pi, pts + j * dim, dim) < cutoff;
    cnt += __popc(__ballot_sync(0xffffffffu, hit));
  }
  (void)n0;
  if (lane == 0) rowcount[v] = cnt;
}

__global__ void k_spatial_fill(int64_t total, const int32_t* __restrict__ node_graph,
                               const int64_t* __restrict__ node_off, const double* __restrict__ pts, int dim,
                               double cutoff, const int64_t* __restrict__ rowstart, int32_t* __restrict__ ei,
                               int32_t* __restrict__ ej, double* __restrict__ w, double* __restrict__ d) {
  const int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= total) return;
  const int g = node_graph[v];
  const int64_t n0 = node_off[g], n1 = node_off[g + 1];
  const double* pi = pts + v * dim;
  int64_t pos = rowstart[v];
  for (int64_t base = v + 1; base < n1; base += 32) {
    const int64_t j = base + lane;
    double dist = 0.0;
    const bool hit = j < n1 && (dist = pair_dist(pi, pts + j * dim, dim)) < cutoff;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (hit) {
      const int64_t e = pos + __popc(m & ((1u << lane) - 1u));
      const double t = __ddiv_rn(dist, cutoff);
      const double u = __dsub_rn(1.0, __dmul_rn(t, t));
      ei[e] = (int32_t)(v - n0);
      ej[e] = (int32_t)(j - n0);
      w[e] = __dmul_rn(u, u);
      d[e] = dist;
    }
    pos += __popc(m);
  }
}

}  // namespace mgk

using namespace mgk;

extern "C" int mgk_spatial_edges(int device, int32_t N, const int64_t* node_off, int dim, const double* points,
                                 double cutoff, int64_t* edge_off, int32_t* ei, int32_t* ej, double* w, double* d) {
  extern int mgk_fail_ingest(int code, const char* msg);
  if (!(cutoff > 0)) return mgk_fail_ingest(MGK_E_INVALID, "cutoff must be positive");
  if (N <= 0 || !node_off || !edge_off) return mgk_fail_ingest(MGK_E_INVALID, "null or empty point-cloud batch");
  if (dim != 2 && dim != 3) return mgk_fail_ingest(MGK_E_INVALID, "points must be an (n, 2) or (n, 3) array");
  const int64_t total = node_off[N];
  if (total > 0 && !points) return mgk_fail_ingest(MGK_E_INVALID, "null points");
  if (cudaSetDevice(device) != cudaSuccess) return mgk_fail_ingest(MGK_E_CUDA, "no CUDA device");
  std::vector<int32_t> ng(total);
  for (int g = 0; g < N; ++g)
    for (int64_t v = node_off[g]; v < node_off[g + 1]; ++v) ng[v] = g;
  int32_t* d_ng = nullptr;
  int64_t *d_off = nullptr, *d_start = nullptr;
  double* d_pts = nullptr;
  int32_t* d_cnt = nullptr;
  int32_t *d_ei = nullptr, *d_ej = nullptr;
  double *d_w = nullptr, *d_d = nullptr;
  cudaError_t e = cudaSuccess;
  auto cleanup = [&]() {
    cudaFree(d_ng);
    cudaFree(d_off);
    cudaFree(d_start);
    cudaFree(d_pts);
    cudaFree(d_cnt);
    cudaFree(d_ei);
    cudaFree(d_ej);
    cudaFree(d_w);
    cudaFree(d_d);
  };
  const size_t tot = (size_t)std::max<int64_t>(total, 1);
  e = cudaMalloc(&d_ng, tot * 4);
  if (e == cudaSuccess) e = cudaMalloc(&d_off, (N + 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_start, (tot + 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_pts, tot * dim * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_cnt, tot * 4);
  if (e == cudaSuccess && total > 0) e = cudaMemcpy(d_ng, ng.data(), total * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_off, node_off, (N + 1) * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && total > 0) e = cudaMemcpy(d_pts, points, total * dim * 8, cudaMemcpyHostToDevice);
  const unsigned blocks = (unsigned)((total * 32 + 255) / 256);
  if (e == cudaSuccess && total > 0) {
    k_spatial_rows<<<blocks, 256>>>(total, d_ng, d_off, d_pts, dim, cutoff, d_cnt);
    e = cudaGetLastError();
  }
  std::vector<int32_t> cnt(total);
  if (e == cudaSuccess && total > 0) e = cudaMemcpy(cnt.data(), d_cnt, total * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    cleanup();
    return mgk_fail_ingest(MGK_E_CUDA, cudaGetErrorString(e));
  }
  // row starts (global) and per-graph edge offsets
  std::vector<int64_t> start(total + 1, 0);
  for (int64_t v = 0; v < total; ++v) start[v + 1] = start[v] + cnt[v];
  for (int g = 0; g <= N; ++g) edge_off[g] = start[node_off[g]];
  const int64_t ne = start[total];
  if (!ei && !ej && !w && !d) {
    cleanup();
    return MGK_OK;
  }
  if (!ei || !ej || !w || !d) {
    cleanup();
    return mgk_fail_ingest(MGK_E_INVALID, "edge outputs must be all set or all NULL");
  }
  const size_t nes = (size_t)std::max<int64_t>(ne, 1);
  e = cudaMemcpy(d_start, start.data(), (total + 1) * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&d_ei, nes * 4);
  if (e == cudaSuccess) e = cudaMalloc(&d_ej, nes * 4);
  if (e == cudaSuccess) e = cudaMalloc(&d_w, nes * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_d, nes * 8);
  if (e == cudaSuccess && total > 0) {
    k_spatial_fill<<<blocks, 256>>>(total, d_ng, d_off, d_pts, dim, cutoff, d_start, d_ei, d_ej, d_w, d_d);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && ne > 0) e = cudaMemcpy(ei, d_ei, ne * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && ne > 0) e = cudaMemcpy(ej, d_ej, ne * 4, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && ne > 0) e = cudaMemcpy(w, d_w, ne * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && ne > 0) e = cudaMemcpy(d, d_d, ne * 8, cudaMemcpyDeviceToHost);
  cleanup();
  if (e != cudaSuccess) return mgk_fail_ingest(MGK_E_CUDA, cudaGetErrorString(e));
  return MGK_OK;
}
