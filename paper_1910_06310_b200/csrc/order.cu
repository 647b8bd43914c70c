// Baseline node orderings on the device: reverse
// Cuthill-McKee (rcm_reorder, reorder.py:412-443) and Morton order
// (morton_keys / morton_reorder, reorder.py:448-478), bit-exact with the
// reference's pinned tie-breaks.
//
// Both reduce to ranking 64-bit keys inside each graph:
//   rank(u) = #{w : (key_w, w) < (key_u, u)}
// computed thread-per-node against shared-memory tiles of the graph's keys
// (k_rank_keys; the n^2 compares are ~10 ms even at n = 10^5, and need no
// segmented sort).  Morton's forward map IS that rank (lexsort by (key,
// index)); RCM's start order is the rank of (degree, index).
//
// RCM then runs one CTA per graph as a level-synchronous BFS that reproduces
// the reference's FIFO queue order exactly: a node v discovered in level L is
// owned by the EARLIEST queue position of L adjacent to it (atomicMin claim),
// the next level is the concatenation, in queue order, of every owner's
// children sorted by (degree, index), and each component's sequence is
// reversed in place.  Components start at the first unvisited node of the
// (degree, index) order, as `by_start` does.
#include <math_constants.h>

#include "mgk.h"
#include "mgk_internal.h"

namespace mgk {

constexpr int kOrderThreads = 256;
constexpr int kRankTile = 2048;  // keys per shared-memory tile (16 KB)

// ---- keys ---------------------------------------------------------------------------------------

// RCM start key (degree, index): degree = row length of the octile row expansion (unique neighbours,
// _adjacency_lists of reorder.py:27-35; duplicates and self-loops are rejected at upload).
__global__ void k_rcm_keys(int64_t ntotal, const int32_t* __restrict__ node_graph, const GraphDesc* __restrict__ graphs,
                           const int32_t* __restrict__ rowptr, uint64_t* __restrict__ keys) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= ntotal) return;
  const GraphDesc g = graphs[node_graph[v]];
  const int u = (int)(v - g.node_off);
  const int32_t* rp = rowptr + g.rowptr_off;
  keys[v] = ((uint64_t)(uint32_t)(rp[u + 1] - rp[u]) << 32) | (uint32_t)u;
}

__device__ double block_reduce_minmax(double v, bool is_min, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_min ? fmin(v, x) : fmax(v, x);
  }
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = red[0];
  for (int k = 1; k < (int)(blockDim.x >> 5); ++k) r = is_min ? fmin(r, red[k]) : fmax(r, red[k]);
  return r;
}

// morton_keys (reorder.py:448-468): coordinates quantised over the graph's bounding box with
// MORTON_BITS = 21, first coordinate in the least significant interleave slot.  Every float64 step
// is an explicitly rounded intrinsic (no FMA contraction), matching numpy's elementwise
// (pts - lo) * scale and floor.  One CTA per graph.
__global__ void __launch_bounds__(kOrderThreads)
k_morton_keys(const GraphDesc* __restrict__ graphs, const double* __restrict__ pts, int dim,
              uint64_t* __restrict__ keys) {
  __shared__ double red[kOrderThreads / 32];
  const GraphDesc g = graphs[blockIdx.x];
  const double* P = pts + g.node_off * dim;
  double lo[3], scale[3];
  for (int d = 0; d < dim; ++d) {
    double mn = CUDART_INF, mx = -CUDART_INF;
    for (int u = threadIdx.x; u < g.n; u += blockDim.x) {
      mn = fmin(mn, P[(int64_t)u * dim + d]);
      mx = fmax(mx, P[(int64_t)u * dim + d]);
    }
    mn = block_reduce_minmax(mn, true, red);
    mx = block_reduce_minmax(mx, false, red);
    double span = __dsub_rn(mx, mn);
    if (span == 0.0) span = 1.0;
    lo[d] = mn;
    scale[d] = __ddiv_rn(2097151.0, span);  // (2**21 - 1) / span
  }
  for (int u = threadIdx.x; u < g.n; u += blockDim.x) {
    uint64_t key = 0;
    for (int d = 0; d < dim; ++d) {
      const double f = floor(__dmul_rn(__dsub_rn(P[(int64_t)u * dim + d], lo[d]), scale[d]));
      int64_t qd = (f >= 0.0) ? (f < 2097151.0 ? (int64_t)f : 2097151) : 0;  // np.clip(.., 0, 2**21 - 1)
      for (int b = 0; b < 21; ++b) key |= (uint64_t)((qd >> b) & 1) << (b * dim + d);
    }
    keys[g.node_off + u] = key;
  }
}

// ---- per-graph ranking ---------------------------------------------------------------------------

// Block c ranks nodes [chunk_node[c], +blockDim) of graph chunk_graph[c] against all of that graph's
// keys; writes rank (local) to rank_out[node].
__global__ void __launch_bounds__(kOrderThreads)
k_rank_keys(const GraphDesc* __restrict__ graphs, const int32_t* __restrict__ chunk_graph,
            const int32_t* __restrict__ chunk_node, const uint64_t* __restrict__ keys, int64_t* __restrict__ rank_out) {
  __shared__ uint64_t tile[kRankTile];
  const GraphDesc g = graphs[chunk_graph[blockIdx.x]];
  const int u = chunk_node[blockIdx.x] + threadIdx.x;
  const uint64_t* K = keys + g.node_off;
  const bool live = u < g.n;
  const uint64_t ku = live ? K[u] : 0;
  int64_t r = 0;
  for (int t0 = 0; t0 < g.n; t0 += kRankTile) {
    const int len = min(kRankTile, g.n - t0);
    __syncthreads();
    for (int k = threadIdx.x; k < len; k += blockDim.x) tile[k] = K[t0 + k];
    __syncthreads();
    if (live) {
      for (int k = 0; k < len; ++k) {
        const uint64_t kw = tile[k];
        r += (kw < ku) || (kw == ku && t0 + k < u);
      }
    }
  }
  if (live) rank_out[g.node_off + u] = r;
}

// ---- RCM breadth-first search --------------------------------------------------------------------

// Exclusive scan of a[0..len) in place (block-wide, chunks of blockDim); returns the total.
__device__ int block_exclusive_scan(int* a, int len, int* warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int carry = 0;
  for (int c0 = 0; c0 < len; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const int x = i < len ? a[i] : 0;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    int before = carry, chunk = 0;
    for (int k = 0; k < nw; ++k) {
      if (k < w) before += warp_tot[k];
      chunk += warp_tot[k];
    }
    if (i < len) a[i] = before + incl - x;
    carry += chunk;
  }
  __syncthreads();
  return carry;
}

struct RcmScratch {
  int32_t* claim;    // [sum n] owner queue position of an unvisited node (INT_MAX: none)
  int32_t* visited;  // [sum n]
  int32_t* order;    // [sum n] Cuthill-McKee queue, components reversed at the end
  int32_t* start;    // [sum n] nodes by (degree, index)
  int32_t* cnt;      // [sum n] per queue position: children count, then their offset
};

__global__ void __launch_bounds__(kOrderThreads)
k_rcm_bfs(const GraphDesc* __restrict__ graphs, const int32_t* __restrict__ rowptr, const float4* __restrict__ rowent,
          RcmScratch s, int64_t* __restrict__ forward) {
  __shared__ int warp_tot[kOrderThreads / 32];
  __shared__ int sh_start, sh_cursor;
  const GraphDesc g = graphs[blockIdx.x];
  const int n = g.n;
  const int32_t* rp = rowptr + g.rowptr_off;
  const float4* re = rowent + g.nz_off;
  int32_t* claim = s.claim + g.node_off;
  int32_t* visited = s.visited + g.node_off;
  int32_t* order = s.order + g.node_off;
  const int32_t* start = s.start + g.node_off;
  int32_t* cnt = s.cnt + g.node_off;
  for (int u = threadIdx.x; u < n; u += blockDim.x) {
    claim[u] = INT_MAX;
    visited[u] = 0;
  }
  if (threadIdx.x == 0) sh_cursor = 0;
  __syncthreads();
  int tail = 0;
  for (;;) {
    if (threadIdx.x == 0) {  // first unvisited node of the (degree, index) order
      int c = sh_cursor;
      while (c < n && visited[start[c]]) ++c;
      sh_cursor = c;
      sh_start = c < n ? start[c] : -1;
      if (c < n) {
        order[tail] = start[c];
        visited[start[c]] = 1;
      }
    }
    __syncthreads();
    const int s0 = sh_start;
    if (s0 < 0) break;
    const int comp0 = tail;
    int lvl0 = tail, lvl1 = tail + 1;
    while (lvl0 < lvl1) {
      // claims: every unvisited neighbour is owned by the earliest level position adjacent to it
      for (int idx = lvl0 + (int)threadIdx.x; idx < lvl1; idx += blockDim.x) {
        const int u = order[idx];
        for (int k = rp[u]; k < rp[u + 1]; ++k) {
          const int v = __float_as_int(re[k].x);
          if (!visited[v]) atomicMin(&claim[v], idx);
        }
      }
      __syncthreads();
      for (int idx = lvl0 + (int)threadIdx.x; idx < lvl1; idx += blockDim.x) {
        const int u = order[idx];
        int c = 0;
        for (int k = rp[u]; k < rp[u + 1]; ++k) c += claim[__float_as_int(re[k].x)] == idx;
        cnt[idx - lvl0] = c;
      }
      __syncthreads();
      const int total = block_exclusive_scan(cnt, lvl1 - lvl0, warp_tot);
      // each owner writes its children in (degree, index) order
      for (int idx = lvl0 + (int)threadIdx.x; idx < lvl1; idx += blockDim.x) {
        const int u = order[idx];
        const int base = lvl1 + cnt[idx - lvl0];
        for (int k = rp[u]; k < rp[u + 1]; ++k) {
          const int v = __float_as_int(re[k].x);
          if (claim[v] != idx) continue;
          const int dv = rp[v + 1] - rp[v];
          int r = 0;
          for (int k2 = rp[u]; k2 < rp[u + 1]; ++k2) {
            const int x = __float_as_int(re[k2].x);
            if (claim[x] != idx) continue;
            const int dx = rp[x + 1] - rp[x];
            r += dx < dv || (dx == dv && x < v);
          }
          order[base + r] = v;
          visited[v] = 1;
        }
      }
      __syncthreads();
      lvl0 = lvl1;
      lvl1 += total;
    }
    tail = lvl1;
    // reverse this component's sequence in place (order.extend(reversed(component)))
    const int len = tail - comp0;
    for (int k = threadIdx.x; k < len / 2; k += blockDim.x) {
      const int a = order[comp0 + k];
      order[comp0 + k] = order[tail - 1 - k];
      order[tail - 1 - k] = a;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) forward[g.node_off + order[i]] = i;
}

__global__ void k_scatter_start(int64_t ntotal, const int32_t* __restrict__ node_graph,
                                const GraphDesc* __restrict__ graphs, const int64_t* __restrict__ rank,
                                int32_t* __restrict__ start) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= ntotal) return;
  const GraphDesc g = graphs[node_graph[v]];
  start[g.node_off + rank[v]] = (int32_t)(v - g.node_off);
}

// ---- host ---------------------------------------------------------------------------------------

static cudaError_t rank_all(int G, const std::vector<GraphDesc>& graphs, const GraphDesc* d_graphs,
                            const uint64_t* d_keys, int64_t* d_rank, cudaStream_t s) {
  std::vector<int32_t> cg, cn;
  for (int g = 0; g < G; ++g)
    for (int u = 0; u < graphs[g].n; u += kOrderThreads) {
      cg.push_back(g);
      cn.push_back(u);
    }
  if (cg.empty()) return cudaSuccess;
  int32_t* d_c = nullptr;
  cudaError_t e = cudaMalloc(&d_c, 2 * cg.size() * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_c, cg.data(), cg.size() * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_c + cg.size(), cn.data(), cn.size() * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    k_rank_keys<<<(unsigned)cg.size(), kOrderThreads, 0, s>>>(d_graphs, d_c, d_c + cg.size(), d_keys, d_rank);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d_c);
  return e;
}

int order_device(int method, int G, const std::vector<GraphDesc>& graphs, const GraphDesc* d_graphs,
                 const int32_t* d_node_graph, const int32_t* d_rowptr, const float4* d_rowent,
                 const std::vector<double>& coords, int dim, cudaStream_t s, std::vector<int64_t>& forward,
                 std::string& err) {
  int64_t nn = 0;
  for (const GraphDesc& g : graphs) nn += g.n;
  forward.assign(nn, 0);
  if (nn == 0) return MGK_OK;
  uint64_t* d_keys = nullptr;
  int64_t *d_rank = nullptr, *d_fwd = nullptr;
  double* d_pts = nullptr;
  int32_t* d_rs = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_keys);
    cudaFree(d_rank);
    cudaFree(d_fwd);
    cudaFree(d_pts);
    cudaFree(d_rs);
  };
  auto cuda_fail = [&](cudaError_t e) {
    cleanup();
    err = std::string("device reorder: ") + cudaGetErrorString(e);
    return MGK_E_CUDA;
  };
  cudaError_t e = cudaMalloc(&d_keys, nn * sizeof(uint64_t));
  if (e == cudaSuccess) e = cudaMalloc(&d_rank, nn * sizeof(int64_t));
  if (e != cudaSuccess) return cuda_fail(e);
  const unsigned nb = (unsigned)((nn + 255) / 256);
  if (method == MGK_REORDER_MORTON) {
    e = cudaMalloc(&d_pts, coords.size() * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d_pts, coords.data(), coords.size() * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e);
    k_morton_keys<<<G, kOrderThreads, 0, s>>>(d_graphs, d_pts, dim, d_keys);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = rank_all(G, graphs, d_graphs, d_keys, d_rank, s);
    if (e == cudaSuccess) e = cudaMemcpy(forward.data(), d_rank, nn * sizeof(int64_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e);
    cleanup();
    return MGK_OK;
  }
  // RCM
  k_rcm_keys<<<nb, 256, 0, s>>>(nn, d_node_graph, d_graphs, d_rowptr, d_keys);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = rank_all(G, graphs, d_graphs, d_keys, d_rank, s);
  if (e == cudaSuccess) e = cudaMalloc(&d_rs, 5 * nn * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&d_fwd, nn * sizeof(int64_t));
  if (e != cudaSuccess) return cuda_fail(e);
  RcmScratch sc{d_rs, d_rs + nn, d_rs + 2 * nn, d_rs + 3 * nn, d_rs + 4 * nn};
  k_scatter_start<<<nb, 256, 0, s>>>(nn, d_node_graph, d_graphs, d_rank, sc.start);
  k_rcm_bfs<<<G, kOrderThreads, 0, s>>>(d_graphs, d_rowptr, d_rowent, sc, d_fwd);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaMemcpy(forward.data(), d_fwd, nn * sizeof(int64_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e);
  cleanup();
  return MGK_OK;
}

}  // namespace mgk
