// K1: device octile builder (reference tiles.py:85-127, bit-exact).
//
// Every undirected edge (i, j) contributes the directed nonzeros (i, j) and
// (j, i).  A nonzero's key is (tile_row, tile_col, bit) with
// bit = (r % 8) * 8 + c % 8; octiles are the runs of equal (tile_row, tile_col)
// in key order, the bitmap is the OR of the run's bits and the compact values
// follow key order.  On the device this is a counting sort by tile row
// ("segment" = one tile row of one graph) followed by an in-segment sort on
// (tile_col << 6 | bit) and a run-length emit:
//
//   seg_count   thread / directed nonzero   atomic histogram over segments
//   scan        one CTA                     exclusive scan (segments are few)
//   seg_scatter thread / directed nonzero   (key, src) into its segment
//   seg_sort    CTA / segment               bitonic sort in shared memory
//                                           (global-memory fallback when large)
//   seg_emit    warp / segment              tile ids by ballot-scan, bitmaps,
//                                           compact w / labels, tile-row ptrs
//   degrees     thread / node               d_i = sum_j w_ij + q_i in column order
//
// Keys are unique (validate_graph rejects duplicate edges), so the result is
// deterministic regardless of the atomic order in seg_scatter.
#include "mgk_dev.cuh"
#include "mgk_internal.h"

namespace mgk {

__global__ void k_seg_count(int64_t nedges, const int32_t* __restrict__ ei, const int32_t* __restrict__ ej,
                            const int32_t* __restrict__ egraph, const int64_t* __restrict__ gseg,
                            int32_t* __restrict__ seg_count) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 2 * nedges) return;
  int64_t e = t >> 1;
  int r = (t & 1) ? ej[e] : ei[e];
  atomicAdd(&seg_count[gseg[egraph[e]] + (r >> 3)], 1);
}

__global__ void k_seg_scatter(int64_t nedges, const int32_t* __restrict__ ei, const int32_t* __restrict__ ej,
                              const int32_t* __restrict__ egraph, const int64_t* __restrict__ gseg,
                              const int64_t* __restrict__ seg_start, int32_t* __restrict__ seg_cursor,
                              uint64_t* __restrict__ keys) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 2 * nedges) return;
  int64_t e = t >> 1;
  int r = (t & 1) ? ej[e] : ei[e];
  int c = (t & 1) ? ei[e] : ej[e];
  int64_t seg = gseg[egraph[e]] + (r >> 3);
  int pos = atomicAdd(&seg_cursor[seg], 1);
  uint32_t key = ((uint32_t)(c >> 3) << 6) | (uint32_t)((r & 7) * 8 + (c & 7));
  keys[seg_start[seg] + pos] = ((uint64_t)key << 32) | (uint64_t)(uint32_t)t;
}

// In-place ascending bitonic sort of buf[0, P) (P a power of two) by the CTA.
__device__ void bitonic_sort(uint64_t* buf, int P) {
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        int ixj = i ^ j;
        if (ixj > i) {
          uint64_t a = buf[i], b = buf[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) {
            buf[i] = b;
            buf[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

constexpr int kSortSmem = 8192;  // keys per segment sorted in shared memory

__global__ void k_seg_sort(int64_t nseg, const int64_t* __restrict__ seg_start, const int32_t* __restrict__ seg_count,
                           uint64_t* __restrict__ keys, uint64_t* __restrict__ scratch) {
  extern __shared__ uint64_t sbuf[];
  for (int64_t seg = blockIdx.x; seg < nseg; seg += gridDim.x) {
    int cnt = seg_count[seg];
    if (cnt <= 1) continue;
    int P = 1;
    while (P < cnt) P <<= 1;
    uint64_t* src = keys + seg_start[seg];
    uint64_t* buf;
    if (P <= kSortSmem) {
      buf = sbuf;
    } else {
      buf = scratch + seg_start[seg] * 2;  // scratch holds 2x the keys: room for the pow2 pad
    }
    for (int i = threadIdx.x; i < P; i += blockDim.x) buf[i] = (i < cnt) ? src[i] : ~0ull;
    __syncthreads();
    bitonic_sort(buf, P);
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) src[i] = buf[i];
    __syncthreads();
  }
}

// Count distinct tile columns per segment (warp per segment).
__global__ void k_seg_ntiles(int64_t nseg, const int64_t* __restrict__ seg_start, const int32_t* __restrict__ seg_count,
                             const uint64_t* __restrict__ keys, int32_t* __restrict__ seg_ntiles) {
  int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t seg = warp; seg < nseg; seg += nwarps) {
    const uint64_t* k = keys + seg_start[seg];
    int cnt = seg_count[seg];
    int total = 0;
    for (int base = 0; base < cnt; base += 32) {
      int idx = base + lane;
      bool is_new = false;
      if (idx < cnt) {
        uint32_t tc = (uint32_t)(k[idx] >> 38);
        is_new = (idx == 0) || ((uint32_t)(k[idx - 1] >> 38) != tc);
      }
      total += __popc(__ballot_sync(0xffffffffu, is_new));
    }
    if (lane == 0) seg_ntiles[seg] = total;
  }
}

// Emit octiles + compact payload (warp per segment).
__global__ void k_seg_emit(int64_t nseg, const int64_t* __restrict__ seg_start, const int32_t* __restrict__ seg_count,
                           const int64_t* __restrict__ seg_tile, const int32_t* __restrict__ seg_graph,
                           const int32_t* __restrict__ seg_row, const uint64_t* __restrict__ keys,
                           const GraphDesc* __restrict__ graphs, const float* __restrict__ ew,
                           const float* __restrict__ elab, int el_dim, Octile* __restrict__ tiles,
                           float* __restrict__ nz_w, float* __restrict__ nz_label) {
  int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t seg = warp; seg < nseg; seg += nwarps) {
    const uint64_t* k = keys + seg_start[seg];
    int cnt = seg_count[seg];
    const GraphDesc g = graphs[seg_graph[seg]];
    int trow = seg_row[seg];
    int carry = -1;
    for (int base = 0; base < cnt; base += 32) {
      int idx = base + lane;
      bool valid = idx < cnt;
      uint64_t kv = valid ? k[idx] : 0;
      uint32_t tc = (uint32_t)(kv >> 38);
      bool is_new = valid && ((idx == 0) || ((uint32_t)(k[idx - 1] >> 38) != tc));
      uint32_t m = __ballot_sync(0xffffffffu, is_new);
      int local = carry + __popc(m & ((2u << lane) - 1u));  // inclusive count of run starts
      carry += __popc(m);
      if (valid) {
        int64_t tile = seg_tile[seg] + local;
        int64_t pos = seg_start[seg] + idx;  // global compact position
        uint32_t bit = (uint32_t)(kv >> 32) & 63u;
        if (is_new) {
          tiles[tile].row = (uint16_t)trow;
          tiles[tile].col = (uint16_t)tc;
          tiles[tile].nz_off = (uint32_t)(pos - g.nz_off);
        }
        atomicOr((unsigned long long*)&tiles[tile].bitmap, 1ull << bit);
        int64_t src = (int64_t)(uint32_t)kv;
        int64_t e = src >> 1;
        nz_w[pos] = ew[e];
        for (int c = 0; c < el_dim; ++c) nz_label[pos * el_dim + c] = elab[e * el_dim + c];
      }
    }
  }
}

// d_i = (sum_j w_ij accumulated in ascending column order) + q_i  (graphs.py:202-214)
__global__ void k_degrees(int64_t ntotal, const int32_t* __restrict__ node_graph, const GraphDesc* __restrict__ graphs,
                          const Octile* __restrict__ tiles, const int32_t* __restrict__ trow,
                          const float* __restrict__ nz_w, const double* __restrict__ q64, double* __restrict__ deg,
                          float* __restrict__ dm) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= ntotal) return;
  const GraphDesc g = graphs[node_graph[v]];
  int i = (int)(v - g.node_off);
  int I = i >> 3, r = i & 7;
  const int32_t* tr = trow + g.trow_off;
  double s = 0.0;
  for (int t = tr[I]; t < tr[I + 1]; ++t) {
    Octile o = tiles[g.tile_off + t];
    uint32_t byte = (uint32_t)(o.bitmap >> (8 * r)) & 0xffu;
    int base = __popcll(o.bitmap & ((1ull << (8 * r)) - 1ull));
    const float* w = nz_w + g.nz_off + o.nz_off + base;
    for (int c = 0; byte; ++c, byte &= byte - 1) s += (double)w[c];
  }
  deg[v] = s + q64[v];
  dm[v] = (float)s;  // d_i - q_i: the weight row sum (Laplacian splitting, mgk_dev.cuh)
}

// Exclusive scan of an int32 array into int64 (single CTA, chunked; n is the segment count).
__global__ void k_scan_exclusive(int64_t n, const int32_t* __restrict__ in, int64_t* __restrict__ out) {
  __shared__ int64_t part[1024];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n; base += blockDim.x) {
    int64_t idx = base + threadIdx.x;
    int64_t v = (idx < n) ? in[idx] : 0;
    part[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < (int)blockDim.x; off <<= 1) {
      int64_t add = (threadIdx.x >= (unsigned)off) ? part[threadIdx.x - off] : 0;
      __syncthreads();
      part[threadIdx.x] += add;
      __syncthreads();
    }
    if (idx < n) out[idx] = carry + part[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += part[threadIdx.x];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

// tile-row pointers: trow[g.trow_off + I] = seg_tile[seg] - g.tile_off for I in 0..ceil(n/8)
__global__ void k_trow(int G, const int64_t* __restrict__ gseg, const int64_t* __restrict__ seg_tile,
                       GraphDesc* __restrict__ graphs, int32_t* __restrict__ trow) {
  int gidx = blockIdx.x * blockDim.x + threadIdx.x;
  if (gidx >= G) return;
  GraphDesc g = graphs[gidx];
  int nrows = ceil8(g.n);
  int64_t s0 = gseg[gidx];
  int64_t base = seg_tile[s0];
  g.tile_off = base;
  g.ntiles = (int32_t)(seg_tile[s0 + nrows] - base);
  for (int I = 0; I <= nrows; ++I) trow[g.trow_off + I] = (int32_t)(seg_tile[s0 + I] - base);
  graphs[gidx] = g;
}

// Directed positions of both orientations of every undirected edge in the row expansion (rows
// ascending, columns ascending within a row): thread per edge, binary search of the two rows.  The
// solvers pair the two entries of an L edge on one lane (one edge-kernel evaluation for both).
__device__ __forceinline__ int row_find(const float4* ent, int lo, int hi, int col) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__float_as_int(ent[mid].x) < col) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_sym_fill(int64_t ne, const int32_t* __restrict__ ei, const int32_t* __restrict__ ej,
                           const int32_t* __restrict__ edge_graph, const GraphDesc* __restrict__ graphs,
                           const int32_t* __restrict__ rowptr, const float4* __restrict__ rowent,
                           int2* __restrict__ symk) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const GraphDesc g = graphs[edge_graph[e]];
  const int i = ei[e], j = ej[e];
  const int32_t* rp = rowptr + g.rowptr_off;
  const float4* ent = rowent + g.nz_off;
  symk[e] = make_int2(row_find(ent, rp[i], rp[i + 1], j), row_find(ent, rp[j], rp[j + 1], i));
}

// Per-graph octile density histogram for the reference's cost counters (product.py:224-266): hist[g][k] =
// tiles with k nonzeros (k = 1..64), hist[g][65] = non-empty tile rows.  One CTA per graph.
__global__ void k_tile_hist(const GraphDesc* __restrict__ graphs, const Octile* __restrict__ tiles,
                            const int32_t* __restrict__ trow, int32_t* __restrict__ hist) {
  __shared__ int h[kHistBins];
  const GraphDesc g = graphs[blockIdx.x];
  for (int k = threadIdx.x; k < kHistBins; k += blockDim.x) h[k] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < g.ntiles; t += blockDim.x) atomicAdd(&h[__popcll(tiles[g.tile_off + t].bitmap)], 1);
  const int32_t* tr = trow + g.trow_off;
  for (int I = threadIdx.x; I < ceil8(g.n); I += blockDim.x)
    if (tr[I + 1] > tr[I]) atomicAdd(&h[65], 1);
  __syncthreads();
  for (int k = threadIdx.x; k < kHistBins; k += blockDim.x) hist[(int64_t)blockIdx.x * kHistBins + k] = h[k];
}

// Row-ordered expansion of the octiles for the panel solver: node i's nonzeros
// (ascending column, the order its tile row implies) land at
// rowent[nz_off + rowptr[i] ..] as {col, w, label, log2 w}.  Thread per node.
__global__ void k_rows_fill(int64_t ntotal, const int32_t* __restrict__ node_graph, const GraphDesc* __restrict__ graphs,
                            const Octile* __restrict__ tiles, const int32_t* __restrict__ trow,
                            const float* __restrict__ nz_w, const float* __restrict__ nz_label, int el_dim,
                            const int32_t* __restrict__ rowptr, float4* __restrict__ rowent) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= ntotal) return;
  const GraphDesc g = graphs[node_graph[v]];
  const int i = (int)(v - g.node_off);
  const int I = i >> 3, r = i & 7;
  const int32_t* tr = trow + g.trow_off;
  float4* dst = rowent + g.nz_off + rowptr[g.rowptr_off + i];
  int pos = 0;
  for (int t = tr[I]; t < tr[I + 1]; ++t) {
    const Octile o = tiles[g.tile_off + t];
    uint32_t byte = (uint32_t)(o.bitmap >> (8 * r)) & 0xffu;
    const int64_t base = g.nz_off + o.nz_off + __popcll(o.bitmap & ((1ull << (8 * r)) - 1ull));
    for (int c = 0; byte; ++c, byte &= byte - 1) {
      const int64_t k = base + c;
      const float lab = el_dim > 0 ? nz_label[k * el_dim] : 0.0f;
      dst[pos++] = make_float4(__int_as_float(o.col * 8 + (__ffs(byte) - 1)), nz_w[k], lab, log2f(nz_w[k]));
    }
  }
}

}  // namespace mgk
