// K3 + K4 (medium class): one CTA solves one graph pair; PCG state in a
// per-CTA HBM/L2 scratch slab.  Same semantics as pcg_warp.cu (product.py:
// 351-419, solver.py:77-121) for any graph size / label dimension.
//
// XMV mapping: warp w takes U-rows i = w, w + nwarps, ...; lane l takes the
// L-nodes i' = l, l + 32, ...; each thread pulls its output element
//   AP[i][i'] = diag[i][i'] P[i][i'] - sum_{k in U(i)} sum_{k' in L(i')} kappa w w' P[j_k][j'_k']
// so there are no atomics.  U-row nonzeros are warp-uniform (broadcast loads),
// L-row nonzeros are per lane.  Both graphs are expanded from their octiles
// into row-ordered nonzero lists in the prologue (CSR derived from the tile
// bitmaps, ascending column).
#include "mgk_internal.h"

namespace mgk {

constexpr int kBlockThreads = 256;
constexpr int kBlockWarps = kBlockThreads / 32;

template <typename V>
struct BlockScratch {
  V* P;
  V* AP;
  V* R;
  V* X;
  V* DG;
  V* SD;        // Laplacian splitting: s = diag - rowsum(L)
  float4* UE;   // {col, w, label0, label1}
  float4* LE;
  float* ULAB;  // extra label dims (dim > 2): [S][el_dim]
  float* LLAB;
  int* urow;
  int* lrow;
};

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int k = 0; k < kBlockWarps; ++k) s += red[k];
  return s;
}

// Row-ordered nonzeros of graph g into dst (+ extra label dims into xlab), row pointers into rowptr.
__device__ void block_octiles_to_rows(const DatasetDev& ds, const GraphDesc& g, float4* dst, float* xlab, int* rowptr,
                                      int* sh_carry) {
  const int el_dim = ds.el_dim;
  const int32_t* tr = ds.trow + g.trow_off;
  const Octile* tiles = ds.tiles + g.tile_off;
  // pass 1: counts
  for (int i = threadIdx.x; i < g.n; i += blockDim.x) {
    int I = i >> 3, r = i & 7, cnt = 0;
    for (int t = tr[I]; t < tr[I + 1]; ++t) cnt += __popc((uint32_t)(tiles[t].bitmap >> (8 * r)) & 0xffu);
    rowptr[i + 1] = cnt;
  }
  __syncthreads();
  // pass 2: sequential-chunk scan (n can be large; chunked by blockDim)
  if (threadIdx.x == 0) {
    rowptr[0] = 0;
    *sh_carry = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 1; i <= g.n; ++i) {
      acc += rowptr[i];
      rowptr[i] = acc;
    }
  }
  __syncthreads();
  // pass 3: fill
  for (int i = threadIdx.x; i < g.n; i += blockDim.x) {
    int I = i >> 3, r = i & 7;
    int pos = rowptr[i];
    for (int t = tr[I]; t < tr[I + 1]; ++t) {
      Octile o = tiles[t];
      uint32_t byte = (uint32_t)(o.bitmap >> (8 * r)) & 0xffu;
      int base = o.nz_off + __popcll(o.bitmap & ((1ull << (8 * r)) - 1ull));
      for (int c = 0; byte; ++c, byte &= byte - 1) {
        int lc = __ffs(byte) - 1;
        int64_t k = g.nz_off + base + c;
        float l0 = el_dim > 0 ? ds.nz_label[k * el_dim] : 0.0f;
        float l1 = el_dim > 1 ? ds.nz_label[k * el_dim + 1] : 0.0f;
        dst[pos] = make_float4(__int_as_float(o.col * 8 + lc), ds.nz_w[k], l0, l1);
        for (int d = 2; d < el_dim; ++d) xlab[(int64_t)pos * el_dim + d] = ds.nz_label[k * el_dim + d];
        ++pos;
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float block_kappa(const KernelDesc& ek, int kind, const float4& a, const float4& b,
                                             const float* ax, const float* bx, int el_dim, bool cat) {
  if (kind == KK_NONE) return 1.0f;
  if (el_dim <= 1 && kind != KK_PROD && kind != KK_RCONV) {
    if (kind == KK_DELTA) return (__float_as_int(a.z) == __float_as_int(b.z)) ? 1.0f : ek.h;
    return kernel_scalar(ek, a.z, b.z);
  }
  float la[kMaxLabelDim], lb[kMaxLabelDim];
  la[0] = a.z;
  la[1] = el_dim > 1 ? a.w : 0.0f;
  lb[0] = b.z;
  lb[1] = el_dim > 1 ? b.w : 0.0f;
  for (int d = 2; d < el_dim; ++d) {
    la[d] = ax[d];
    lb[d] = bx[d];
  }
  return kernel_vec(ek, la, lb, el_dim, cat);
}

__device__ __forceinline__ float vfma(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double vfma(double a, double b, double c) { return fma(a, b, c); }

template <typename V>
__device__ __forceinline__ void solve_block_pair(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek,
                                                 const SolveParams& prm, const SolveOut& out, float* base,
                                                 unsigned long long pid, int32_t ga, int32_t gb, double* red,
                                                 int* sh_carry) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int el_dim = ds.el_dim;
  const bool ecat = ds.el_kind == LK_CAT;
  int ekind = prm.labeled ? ek.kind : KK_NONE;
  if (ekind == KK_CONST1) ekind = KK_NONE;
  {
    const GraphDesc U = ds.graphs[ga], L = ds.graphs[gb];
    const int n = U.n, m = L.n;
    const int64_t nm = (int64_t)n * m;
    const int SU = 2 * U.ne, SL = 2 * L.ne;

    // carve the slab (block_slab in capi.cu reserves room for FP64 vectors of tiny pairs)
    BlockScratch<V> s;
    s.P = reinterpret_cast<V*>((((uintptr_t)base) + 15) & ~(uintptr_t)15);
    s.AP = s.P + nm;
    s.R = s.AP + nm;
    s.X = s.R + nm;
    s.DG = s.X + nm;
    s.SD = s.DG + nm;
    float* tail = reinterpret_cast<float*>(s.SD + nm);
    tail = (float*)(((uintptr_t)tail + 15) & ~(uintptr_t)15);
    s.UE = (float4*)tail;
    s.LE = s.UE + SU;
    s.ULAB = (float*)(s.LE + SL);
    s.LLAB = s.ULAB + (el_dim > 2 ? (int64_t)SU * el_dim : 0);
    s.urow = (int*)(s.LLAB + (el_dim > 2 ? (int64_t)SL * el_dim : 0));
    s.lrow = s.urow + n + 1;

    block_octiles_to_rows(ds, U, s.UE, s.ULAB, s.urow, sh_carry);
    block_octiles_to_rows(ds, L, s.LE, s.LLAB, s.lrow, sh_carry);

    // kappa_e = 1 pairs with a large diag / s (mgk_dev.cuh kLapFactor): A p = s p - sum L (p_j - p_i)
    const bool lap = ekind == KK_NONE && laplacian_pair(prm, U, L);
    // diag, b, r, z, p
    const bool vlab = (vk.kind != KK_CONST1 && vk.kind != KK_NONE && ds.nl_kind != LK_NONE);
    double bu = 0.0, bl = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double dq = ds.deg[U.node_off + i] * ds.q64[U.node_off + i];
      bu += dq * dq;
    }
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      double dq = ds.deg[L.node_off + i] * ds.q64[L.node_off + i];
      bl += dq * dq;
    }
    const double bb = block_sum(bu, red) * block_sum(bl, red);
    const double eps = prm.tol2 * bb;
    double rho_l = 0.0, rr_l = 0.0;
    for (int64_t e = threadIdx.x; e < nm; e += blockDim.x) {
      int i = (int)(e / m), l = (int)(e - (int64_t)i * m);
      int64_t vu = U.node_off + i, vl = L.node_off + l;
      float kv = 1.0f;
      if (vlab)
        kv = floor_kv(kernel_vec(vk, ds.vlabel + vu * ds.nl_dim, ds.vlabel + vl * ds.nl_dim, ds.nl_dim,
                                 ds.nl_kind == LK_CAT), prm, out);
      const double dg64 = ds.deg[vu] * ds.deg[vl] / (double)kv;
      V dg = (V)dg64;
      s.SD[e] = lap ? (V)(dg64 - (ds.deg[vu] - ds.q64[vu]) * (ds.deg[vl] - ds.q64[vl])) : dg;
      V b = (V)((ds.deg[vu] * ds.q64[vu]) * (ds.deg[vl] * ds.q64[vl]));
      V z = b / dg;
      s.DG[e] = dg;
      s.R[e] = b;
      s.X[e] = V(0);
      s.P[e] = z;
      rho_l += (double)b * z;
      rr_l += (double)b * b;
    }
    double rho = block_sum(rho_l, red);
    double rr = block_sum(rr_l, red);
    bool conv = rr < eps;
    const int64_t max_iter = prm.max_iter > 0 ? prm.max_iter : 10ll * nm;
    int64_t it = 0;
    __syncthreads();

    while (!conv && it < max_iter) {
      // XMV (pull per output element)
      for (int i = warp; i < n; i += kBlockWarps) {
        const int k0 = s.urow[i], k1 = s.urow[i + 1];
        for (int l = lane; l < m; l += 32) {
          const int q0 = s.lrow[l], q1 = s.lrow[l + 1];
          const int64_t e = (int64_t)i * m + l;
          const V pc = lap ? s.P[e] : V(0);
          V acc = V(0);
          for (int k = k0; k < k1; ++k) {
            const float4 ea = s.UE[k];
            const V* prow = s.P + (int64_t)__float_as_int(ea.x) * m;
            V part = V(0);
            for (int q = q0; q < q1; ++q) {
              const float4 eb = s.LE[q];
              float kap = block_kappa(ek, ekind, ea, eb, s.ULAB + (int64_t)k * el_dim,
                                      s.LLAB + (int64_t)q * el_dim, el_dim, ecat);
              part = vfma((V)kap * (V)eb.y, prow[__float_as_int(eb.x)] - pc, part);
            }
            acc = vfma((V)ea.y, part, acc);
          }
          s.AP[e] = s.SD[e] * s.P[e] - acc;
        }
      }
      __syncthreads();
      if (ga == gb) {  // self pair: keep the iterate exactly symmetric (see pcg_warp.cu)
        for (int64_t e = threadIdx.x; e < nm; e += blockDim.x) {
          int i = (int)(e / m), l = (int)(e - (int64_t)i * m);
          if (i < l) {
            V v = V(0.5) * (s.AP[e] + s.AP[(int64_t)l * m + i]);
            s.AP[e] = v;
            s.AP[(int64_t)l * m + i] = v;
          }
        }
        __syncthreads();
      }
      ++it;
      double pap_l = 0.0;
      for (int64_t e = threadIdx.x; e < nm; e += blockDim.x) pap_l += (double)s.P[e] * (double)s.AP[e];
      const double alpha = rho / block_sum(pap_l, red);
      const V af = (V)alpha;
      double rr2 = 0.0, rz = 0.0;
      for (int64_t e = threadIdx.x; e < nm; e += blockDim.x) {
        s.X[e] = vfma(af, s.P[e], s.X[e]);
        V r = vfma(-af, s.AP[e], s.R[e]);
        s.R[e] = r;
        V z = r / s.DG[e];
        rr2 += (double)r * r;
        rz += (double)r * z;
      }
      rr = block_sum(rr2, red);
      const double rho_next = block_sum(rz, red);
      if (rr < eps) {
        conv = true;
        break;
      }
      const V beta = (V)(rho_next / rho);
      for (int64_t e = threadIdx.x; e < nm; e += blockDim.x) s.P[e] = vfma(beta, s.P[e], s.R[e] / s.DG[e]);
      rho = rho_next;
      __syncthreads();
    }
    __syncthreads();
    double v_l = 0.0;
    for (int64_t e = threadIdx.x; e < nm; e += blockDim.x) {
      int i = (int)(e / m), l = (int)(e - (int64_t)i * m);
      v_l += (double)ds.p[U.node_off + i] * (double)ds.p[L.node_off + l] * (double)s.X[e];
    }
    const double val = block_sum(v_l, red);
    if (out.nodewise) {
      float* nw = out.nodewise + out.nodewise_off[pid];
      for (int64_t e = threadIdx.x; e < nm; e += blockDim.x) nw[e] = s.X[e];
    }
    if (threadIdx.x == 0) {
      if (out.value) out.value[pid] = val;
      if (out.iters) out.iters[pid] = (int32_t)it;
      if (out.conv) out.conv[pid] = conv ? 1 : 0;
      if (out.residual) out.residual[pid] = (float)sqrt(rr);
      if (out.pair_a) out.pair_a[pid] = ga;
      if (out.pair_b) out.pair_b[pid] = gb;
      if (out.K) {
        double kval = conv ? val : __longlong_as_double(0x7ff8000000000000ll);
        out.K[(int64_t)ga * out.G + gb] = kval;
        out.K[(int64_t)gb * out.G + ga] = kval;
      }
      if (out.K_iters) {
        out.K_iters[(int64_t)ga * out.G + gb] = (int32_t)it;
        out.K_iters[(int64_t)gb * out.G + ga] = (int32_t)it;
      }
      if (out.K_conv) {
        out.K_conv[(int64_t)ga * out.G + gb] = conv;
        out.K_conv[(int64_t)gb * out.G + ga] = conv;
      }
    }
  }
}

__global__ void __launch_bounds__(kBlockThreads)
k_pcg_block(DatasetDev ds, KernelDesc vk, KernelDesc ek, PairJob job, SolveParams prm, SolveOut out,
            unsigned long long* queue, float* scratch, int64_t slab) {
  __shared__ double red[kBlockWarps];
  __shared__ unsigned long long sh_pid;
  __shared__ int sh_carry;
  for (;;) {
    if (threadIdx.x == 0) sh_pid = atomicAdd(queue, 1ull);
    __syncthreads();
    const unsigned long long pid = sh_pid;
    __syncthreads();
    if (pid >= (unsigned long long)job.npairs) break;
    int32_t ga, gb;
    decode_pair(job, (int64_t)pid, ga, gb);
    const int64_t nm = (int64_t)ds.graphs[ga].n * ds.graphs[gb].n;
    // pairs at or below the tiny threshold run with FP64 vectors (CG there ends by Krylov exhaustion,
    // which FP32 rounding delays; see pcg_warp.cu k_pcg_tiny), and so does every pair of a precise
    // kappa_e = 1 solve (kPreciseTol); the rest with FP32 vectors
    if (nm <= prm.tiny_nm || prm.fp64)
      solve_block_pair<double>(ds, vk, ek, prm, out, scratch + (int64_t)blockIdx.x * slab, pid, ga, gb, red, &sh_carry);
    else
      solve_block_pair<float>(ds, vk, ek, prm, out, scratch + (int64_t)blockIdx.x * slab, pid, ga, gb, red, &sh_carry);
    __syncthreads();
  }
}

cudaError_t launch_pcg_block(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                             const SolveParams& prm, const SolveOut& out, unsigned long long* queue, float* scratch,
                             int64_t slab, int nctas, cudaStream_t stream) {
  if (nctas < 1) nctas = 1;
  if ((int64_t)nctas > job.npairs) nctas = (int)job.npairs;
  if (nctas < 1) return cudaSuccess;
  k_pcg_block<<<nctas, kBlockThreads, 0, stream>>>(ds, vk, ek, job, prm, out, queue, scratch, slab);
  return cudaGetLastError();
}

}  // namespace mgk
