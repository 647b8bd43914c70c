// Internal declarations shared by the .cu translation units of libmgk.
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "mgk_dev.cuh"

namespace mgk {

// How a solver launch enumerates its pairs (all map a pair id to (a, b)).
enum PairMode : int32_t {
  PM_TRI = 0,   // all u <= v over list_a (row-major); list sorted by cost descending
  PM_RECT = 1,  // list_a x list_b
  PM_LIST = 2,  // explicit pairs: list_a[k], list_b[k]
  PM_RAGGED = 3,  // row u of list_a pairs with list_a[col0[u] .. col0[u] + len(u)); rows by prefix
};

struct PairJob {
  int32_t mode;
  int32_t na, nb;           // list lengths
  int64_t npairs;           // pairs this launch solves (after sharding)
  int64_t offset, stride;   // shard: local id q -> global id offset + q * stride
  const int32_t* list_a;
  const int32_t* list_b;
  const int64_t* row_prefix;  // PM_RAGGED: na + 1 prefix counts of row lengths
  const int32_t* row_col0;    // PM_RAGGED: first column of each row
};

struct SolveOut {
  // Gram matrix outputs (mirrored writes), any may be null
  double* K;                // [G*G]
  int32_t* K_iters;         // [G*G]
  uint8_t* K_conv;          // [G*G]
  int64_t G;
  // per-pair outputs (indexed by pair id), any may be null
  double* value;
  int32_t* iters;
  uint8_t* conv;
  float* residual;
  int32_t* pair_a;          // graph ids of each solved pair
  int32_t* pair_b;
  // nodewise field x[i * m + i'] per pair (float32), offsets per pair id
  float* nodewise;
  const int64_t* nodewise_off;
  // status bits raised by the solvers (kStatusNonPositiveKv: a floored vertex similarity <= 0)
  int32_t* status;
};
constexpr int32_t kStatusNonPositiveKv = 1;

struct SolveParams {
  double tol2;              // tol^2 (relative stopping rule r.r < tol^2 b.b)
  int64_t max_iter;         // 0 -> 10 * n * m (solver.py:87)
  float v_min;              // vertex-similarity floor (product.py:172-175)
  int32_t labeled;          // edge mode decided per dataset (product.py:153-161)
  int32_t tiny_nm;          // n*m at or below which the warp solver runs the pair in FP64
  int32_t panel_rpc;        // U rows per panel work item (0: automatic)
  int32_t lap_mode;         // Laplacian splitting (kappa_e = 1 pairs): 0 off, 1 by factor, 2 always
  int32_t fp64;             // every pair on the block solver with FP64 vectors (precise_tol)
  int32_t factor_ratio4;    // unlabeled panel / grid pairs use the factored A (P B^T) form when the direct
                            // form costs more than factor_ratio4 / 4 times as many contributions
};

// kappa_e = 1 systems solved to a relative residual below this bound run every pair with FP64
// vectors on the block solver.  Unlabeled product graphs are highly structured: FP32 vectors cost
// CG 3-8 extra iterations against the reference's float64 once the tolerance passes ~3e-7 (q = 5e-4)
// and at 1e-10 for any q (emulation in tools/precision_emulate.py), while labeled
// (kappa_e != 1) pairs keep iteration parity at the reference default 1e-10 in FP32.
constexpr double kPreciseTol = 5e-7;
// ... and so do kappa_e = 1 datasets whose largest self-pair cancellation factor max(d/q) / 2 exceeds
// kPreciseLap (q below ~1e-3): there even the Laplacian-split FP32 iteration flips a +-1 iteration
// count at tol 1e-6 (a q = 5e-4 self pair: 13 against the reference's 15).  Config-4 random geometric
// graphs at q = 0.05 peak at 143 (mean degree 32) and stay on the FP32 solvers.
constexpr float kPreciseLap = 256.0f;

// Laplacian splitting for this pair (mgk_dev.cuh kLapFactor); only the kappa_e = 1 solvers read it.
__host__ __device__ inline bool laplacian_pair(const SolveParams& prm, const GraphDesc& a, const GraphDesc& b) {
  if (prm.lap_mode <= 0) return false;
  if (prm.lap_mode >= 2) return true;
  return a.dqr * b.dqr > kLapFactor * (a.dqr + b.dqr);
}

// kv = max(kappa_v, v_min) with the reference's non-positive check (product.py:164-178)
__device__ __forceinline__ float floor_kv(float kv, const SolveParams& prm, const SolveOut& out) {
  kv = fmaxf(kv, prm.v_min);
  if (!(kv > 0.0f) && out.status) atomicOr(out.status, kStatusNonPositiveKv);
  return kv;
}

// Gram modes report a <= b (the reference's pair order, gram.py:38-54); lists keep the caller's order.
__host__ __device__ inline void decode_gram_pair(const PairJob& j, int64_t pid, int32_t& a, int32_t& b);

__host__ __device__ inline void decode_pair(const PairJob& j, int64_t q, int32_t& a, int32_t& b) {
  const int64_t pid = j.offset + q * j.stride;
  if (j.mode == PM_LIST) {
    a = j.list_a[pid];
    b = j.list_b[pid];
    return;
  }
  decode_gram_pair(j, pid, a, b);
  if (a > b) {
    const int32_t t = a;
    a = b;
    b = t;
  }
}

__host__ __device__ inline void decode_gram_pair(const PairJob& j, int64_t pid, int32_t& a, int32_t& b) {
  if (j.mode == PM_RAGGED) {
    int lo = 0, hi = j.na;  // largest u with row_prefix[u] <= pid
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (j.row_prefix[mid] <= pid) lo = mid; else hi = mid;
    }
    a = j.list_a[lo];
    b = j.list_a[j.row_col0[lo] + (pid - j.row_prefix[lo])];
  } else if (j.mode == PM_RECT) {
    a = j.list_a[pid / j.nb];
    b = j.list_b[pid % j.nb];
  } else {
    // row u holds (u, u..n-1); start(u) = u*n - u*(u-1)/2
    int64_t n = j.na;
    double disc = (double)(2 * n + 1) * (double)(2 * n + 1) - 8.0 * (double)pid;
    int64_t u = (int64_t)(((double)(2 * n + 1) - sqrt(disc > 0 ? disc : 0.0)) * 0.5);
    if (u < 0) u = 0;
    if (u > n - 1) u = n - 1;
    auto start = [n](int64_t r) { return r * n - r * (r - 1) / 2; };
    while (u > 0 && start(u) > pid) --u;
    while (u + 1 < n && start(u + 1) <= pid) ++u;
    int64_t v = pid - start(u) + u;
    a = j.list_a[u];
    b = j.list_a[v];
  }
}

// ---- tile builder kernels (tiles.cu)
__global__ void k_seg_count(int64_t, const int32_t*, const int32_t*, const int32_t*, const int64_t*, int32_t*);
__global__ void k_seg_scatter(int64_t, const int32_t*, const int32_t*, const int32_t*, const int64_t*,
                              const int64_t*, int32_t*, uint64_t*);
__global__ void k_seg_sort(int64_t, const int64_t*, const int32_t*, uint64_t*, uint64_t*);
__global__ void k_seg_ntiles(int64_t, const int64_t*, const int32_t*, const uint64_t*, int32_t*);
__global__ void k_seg_emit(int64_t, const int64_t*, const int32_t*, const int64_t*, const int32_t*,
                           const int32_t*, const uint64_t*, const GraphDesc*, const float*, const float*, int,
                           Octile*, float*, float*);
__global__ void k_degrees(int64_t, const int32_t*, const GraphDesc*, const Octile*, const int32_t*,
                          const float*, const double*, double*, float*);
__global__ void k_scan_exclusive(int64_t, const int32_t*, int64_t*);
__global__ void k_trow(int, const int64_t*, const int64_t*, GraphDesc*, int32_t*);
__global__ void k_rows_fill(int64_t, const int32_t*, const GraphDesc*, const Octile*, const int32_t*, const float*,
                            const float*, int, const int32_t*, float4*);
constexpr int kSortSmemBytes = 8192 * 8;
__global__ void k_sym_fill(int64_t, const int32_t*, const int32_t*, const int32_t*, const GraphDesc*, const int32_t*,
                           const float4*, int2*);
constexpr int kHistBins = 66;  // k_tile_hist: tiles per nonzero count 0..64, then non-empty tile rows
__global__ void k_tile_hist(const GraphDesc*, const Octile*, const int32_t*, int32_t*);

// per-pair FP32 vectors of the panel slab / grid buffer (pcg_panel.cu)
constexpr int kSlabVectors = 7;

// ---- solvers (pcg_warp.cu, pcg_block.cu)
struct SmallClass {
  static constexpr int NU = 24;      // max nodes of either graph
  static constexpr int SLOTS = 10;   // lane-side nonzeros <= 32 * SLOTS
  static constexpr int SMAX = 32 * SLOTS;
};
// narrow warp-solver instantiation: lane graphs of <= 32 * kNarrowSlots nonzeros
constexpr int kNarrowSlots = 4;

cudaError_t launch_pcg_warp(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                            const SolveParams& prm, const SolveOut& out, unsigned long long* queue,
                            int num_sms, int slots, cudaStream_t stream);
cudaError_t launch_pcg_tiny(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                            const SolveParams& prm, const SolveOut& out, unsigned long long* queue,
                            int num_sms, cudaStream_t stream);
// panel and grid classes (pcg_panel.cu, built as p256 and p512: 256- / 512-thread CTAs)
#define MGK_PANEL_DECLS                                                                                    \
  cudaError_t launch_pcg_panel(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek,         \
                               const PairJob& job, const SolveParams& prm, const SolveOut& out,          \
                               unsigned long long* queue, float* scratch, int64_t scratch_floats_per_cta, \
                               int nctas, int smem_vec_floats, cudaStream_t stream);                     \
  int panel_ctas_per_sm(int smem_vec_floats);                                                            \
  cudaError_t launch_pcg_grid(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek,          \
                              const PairJob& job, const SolveParams& prm, const SolveOut& out, float* vec,  \
                              int64_t vstride, double2* gbuf, int nblocks, cudaStream_t stream);         \
  int grid_blocks(int num_sms);
namespace p256 {
MGK_PANEL_DECLS
}
namespace p512 {
MGK_PANEL_DECLS
}
#undef MGK_PANEL_DECLS
// Gram post-processing (gram_post.cu)
cudaError_t launch_gram_normalize(double* K, int64_t G, double* diag, int* bad, int num_sms, cudaStream_t stream,
                                  bool* nonpositive);
cudaError_t launch_gram_assemble(int64_t npairs, const int32_t* pa, const int32_t* pb, const double* value,
                                 const int32_t* iters, const uint8_t* conv, int64_t G, double* K, int32_t* K_iters,
                                 uint8_t* K_conv, int num_sms, cudaStream_t stream);
cudaError_t launch_pcg_block(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                             const SolveParams& prm, const SolveOut& out, unsigned long long* queue,
                             float* scratch, int64_t scratch_floats_per_cta, int nctas, cudaStream_t stream);

// Baseline orderings (order.cu): method MGK_REORDER_RCM or MGK_REORDER_MORTON; forward maps
// (old -> new, local) of every graph; coords = the dataset's vector node labels (Morton).
int order_device(int method, int G, const std::vector<GraphDesc>& graphs, const GraphDesc* d_graphs,
                 const int32_t* d_node_graph, const int32_t* d_rowptr, const float4* d_rowent,
                 const std::vector<double>& coords, int dim, cudaStream_t s, std::vector<int64_t>& forward,
                 std::string& err);

}  // namespace mgk
