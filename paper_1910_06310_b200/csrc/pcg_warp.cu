// K3 + K4 (small-pair class): one warp solves one graph pair end to end.
//
// Replaces, per pair: ProductOperator.__init__ (product.py:184-222: diag,
// vertex similarity), apply / apply_offdiag (product.py:351-419: the
// on-the-fly tensor-product matvec "XMV") and solve_pcg (solver.py:77-121).
//
// Persistent: every warp pops pair ids from a global atomic queue whose order
// is cost-descending (longest job first, gram.py:38-54) and keeps solving until
// the queue is drained.  Nothing about the product graph is materialised: each
// PCG iteration re-streams both graphs' nonzeros and evaluates the edge base
// kernel for every fused contribution.
//
// Roles.  Of the two graphs, U ("uniform") is walked row by row by the whole
// warp in lock step, L ("lanes") is spread over the 32 lanes: lane l owns the
// L-nonzeros k' = l + 32 t (t < NS, registers, for the whole solve) and the
// L-node i' = l for the vector operations.  The PCG direction P lives in
// shared memory as [i][32] (i = U node, column = lane), so the XMV gather
// P[j][col_L(k')] is bank-conflict free (bank = column).  For U-row i:
//
//   acc[t] = sum_{k in U(i)} kappa(e_k, e'_t) * w_k * P[j_k][col_L(t)]   (registers)
//   SEG[k'] = acc[t] * w'_t;  OFF[i][i'] = sum_{k' in L(i')} SEG[k']
//
// i.e. OFF = sum_{j, j'} w_ij w'_i'j' ke(e_ij, e'_i'j') p[j, j'] (product.py:454-478),
// and the vector phase forms A p = diag * p - OFF.  NS = ceil(S_L / 32) is a
// template parameter (switch per pair) so no lane issues dead slots.
// Unlabeled pairs use the factorised form OFF = A (P B^T) (the paper's dense x
// dense unlabeled primitive, product.py:94): n*S_L + S_U*m work instead of
// S_U*S_L.  The value px.x is accumulated as sum_k alpha_k (px.p_k), so the
// Gram path keeps no x vector.
//
// The graphs come from the dataset's row expansion of the device octiles
// (k_rows_fill, tiles.cu: one popc/bit-scan pass over every tile row per
// dataset), read per pair as coalesced 16-byte records.
#include <cstdio>

#include "mgk_internal.h"

namespace mgk {

constexpr int kWarpsPerBlock = 2;
constexpr int NU = SmallClass::NU;
constexpr int SLOTS = SmallClass::SLOTS;
constexpr int SMAX = SmallClass::SMAX;

// Per-warp shared memory.  The residual and the diagonal live in registers
// (lane = L node, one register per U row), so only the XMV operands are here.
template <bool UNLAB, bool NODEWISE, int SLM>
struct WarpSmem {
  float P[NU][32];        // P + OFF: staging area for the L nonzeros during the prologue
  float OFF[NU][32];
  float T[UNLAB ? NU : 1][32];
  float X[NODEWISE ? NU : 1][32];
  float4 UE[SMAX];        // U nonzeros in row order: {weight form, label, byte offset of P row j, -}
  float SEG[2 * 32 * SLM];  // segment sums of two U-rows
  int urow[NU + 8];
  int lrow[40];
  float upq[NU];          // p_i of U nodes
  float udq[NU];          // d_i q_i of U nodes
  float udm[UNLAB ? NU : 1];  // d_i - q_i of U nodes (Laplacian splitting: preconditioner = s + udm * ldm)
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

__device__ __forceinline__ void write_pair_outputs(const SolveOut& out, unsigned long long pid, int ga, int gb,
                                                   double val, int64_t it, bool conv, double rr, int lane) {
  if (lane != 0) return;
  if (out.value) out.value[pid] = val;
  if (out.iters) out.iters[pid] = (int32_t)it;
  if (out.conv) out.conv[pid] = conv ? 1 : 0;
  if (out.residual) out.residual[pid] = (float)sqrt(rr);
  if (out.pair_a) out.pair_a[pid] = ga;
  if (out.pair_b) out.pair_b[pid] = gb;
  const double kval = conv ? val : __longlong_as_double(0x7ff8000000000000ll);
  if (out.K) {
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

// diag[i][l] = d_i d'_l / max(kv, v_min)  (product.py:164-178, 210); kept out of
// line so the vertex-kernel code exists once per kernel (instruction-cache footprint)
__device__ __noinline__ double diag_of(const DatasetDev& ds, const KernelDesc& vk, const SolveParams& prm,
                                       const SolveOut& out, bool vlab, int64_t vu, int64_t vl) {
  float kv = 1.0f;
  if (vlab)
    kv = floor_kv(kernel_vec(vk, ds.vlabel + vu * ds.nl_dim, ds.vlabel + vl * ds.nl_dim, ds.nl_dim,
                             ds.nl_kind == LK_CAT), prm, out);
  return ds.deg[vu] * ds.deg[vl] / (double)kv;
}

// s = diag - rowsum(L) for kappa_e = 1: rowsum = (d - q)(d' - q'), both in FP64 (Laplacian splitting)
__device__ __forceinline__ double shifted_diag(const DatasetDev& ds, double diag, int64_t vu, int64_t vl) {
  return diag - (ds.deg[vu] - ds.q64[vu]) * (ds.deg[vl] - ds.q64[vl]);
}

// ---------------------------------------------------------------------------
// Tiny product systems (n*m <= prm.tiny_nm, default 128): CG terminates there
// by Krylov exhaustion, which FP32 rounding in the matvec delays by a few
// iterations.  These pairs run the same algorithm with FP64 vectors and FP64
// accumulation (edge-kernel coefficients stay FP32), which restores the
// reference's iteration counts.
//
// The matvec uses the warp solver's lane-slot mapping: the warp walks the
// rows of U in lock step, lane l owns the nonzeros l + 32 t of L (t < NS), so
// every lane runs the same trip counts -- no divergent per-element loops.  U is
// the graph with FEWER nodes (n m <= 128 gives n_U <= 11): few row passes (each
// ends in a warp sync and a segment sum) and up to NS = 10 independent slot
// chains per U nonzero.
// The field lives compactly as [i * m + l] (a warp-uniform row j gathers
// P[j * m + col_L(t)], consecutive banks); the vector phase gives lane e % 32
// the elements e (<= 4 per lane).
// ---------------------------------------------------------------------------
constexpr int kTinyMax = 128;
constexpr int kTinySlots = SLOTS;  // lane graph of <= 320 nonzeros (the small class)
constexpr int kTinyRows = 11;      // n_U <= floor(128 / 11)... U is the smaller graph: n_U^2 <= n_U n_L <= 128

struct TinySmem {
  double P[kTinyMax];
  double AP[kTinyMax];
  double RD[kTinyMax];  // 1 / diag (Jacobi preconditioner)
  double SS[kTinyMax];
  double R[kTinyMax];   // residual and iterate (shared memory keeps the matvec's registers free)
  double X[kTinyMax];
  double SEG[2 * 32 * kTinySlots];  // slot products of two U rows, segment-summed per L row
  float4 UE[kTinyRows * (kTinyRows - 1)];  // U nonzeros: {weight form, label, P row offset j * m, -}
  int urow[kTinyRows + 1];
  int lrow[NU + 8];
};

// AP = SS * P - OFF for all U rows; OFF[i][l] = sum_{k in U(i)} sum_{t in L(l)} kappa w_k w'_t P[j_k][col_t]
// (Laplacian splitting: P[j_k][col_t] - P[i][l] instead of P[j_k][col_t]).  Lane slot t holds an
// undirected L edge {l_t, c_t}: one edge-kernel value (MUFU.EX2 + F2F) feeds the contributions of
// both directed entries l_t -> c_t (gathers P[j][c_t], lands on OFF[i][l_t]) and c_t -> l_t
// (gathers P[j][l_t], lands on OFF[i][c_t]); the per-entry accumulation order is unchanged.
template <int NS, int EK, bool LAP>
__device__ __forceinline__ void tiny_xmv(TinySmem& S, const KernelDesc& ek, int nu, int m, int lane,
                                         const int (&lcol)[kTinySlots], const int (&lrw)[kTinySlots],
                                         const int (&lkab)[kTinySlots], const float (&lw)[kTinySlots],
                                         const float (&llab)[kTinySlots], int nund, int lr0, int lr1) {
  for (int i = 0; i < nu; i += 2) {
    const bool two = i + 1 < nu;
    double acc[2][NS], accb[2][NS];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int t = 0; t < NS; ++t) acc[r][t] = accb[r][t] = 0.0;
      if (r == 1 && !two) break;
      const int row = i + r;
      double pca[NS], pcb[NS];
#pragma unroll
      for (int t = 0; t < NS; ++t) {
        pca[t] = LAP ? S.P[row * m + lrw[t]] : 0.0;  // l -> c lands on (row, l)
        pcb[t] = LAP ? S.P[row * m + lcol[t]] : 0.0;  // c -> l lands on (row, c)
      }
      const int k1 = S.urow[row + 1];
      for (int k = S.urow[row]; k < k1; ++k) {
        const float4 e0 = S.UE[k];
        const double* p0 = S.P + __float_as_int(e0.z);
#pragma unroll
        for (int t = 0; t < NS; ++t) {
          const double c = (double)edge_kappa_w<EK>(ek, e0.y, llab[t], e0.x);
          const double va = LAP ? p0[lcol[t]] - pca[t] : p0[lcol[t]];
          const double vb = LAP ? p0[lrw[t]] - pcb[t] : p0[lrw[t]];
          acc[r][t] = fma(c, va, acc[r][t]);
          accb[r][t] = fma(c, vb, accb[r][t]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      if (lane + 32 * t < nund) {
        const int ka = lkab[t] & 0xffff, kb = lkab[t] >> 16;
        const double w = (double)lw[t];
        S.SEG[ka] = acc[0][t] * w;
        S.SEG[kb] = accb[0][t] * w;
        S.SEG[32 * kTinySlots + ka] = acc[1][t] * w;
        S.SEG[32 * kTinySlots + kb] = accb[1][t] * w;
      }
    }
    __syncwarp();
    if (lane < m) {
      double s0 = 0.0, s1 = 0.0;
      for (int q = lr0; q < lr1; ++q) {
        s0 += S.SEG[q];
        s1 += S.SEG[32 * kTinySlots + q];
      }
      const int e0 = i * m + lane;
      S.AP[e0] = S.SS[e0] * S.P[e0] - s0;
      if (two) S.AP[e0 + m] = S.SS[e0 + m] * S.P[e0 + m] - s1;
    }
    __syncwarp();
  }
}

template <int EK, bool LAP>
__device__ __forceinline__ void tiny_xmv_dispatch(TinySmem& S, const KernelDesc& ek, int nu, int m, int lane,
                                                  const int (&lcol)[kTinySlots], const int (&lrw)[kTinySlots],
                                                  const int (&lkab)[kTinySlots], const float (&lw)[kTinySlots],
                                                  const float (&llab)[kTinySlots], int nund, int lr0, int lr1) {
  switch ((nund + 31) >> 5) {
#define MGK_TINY_CASE(N) \
    case N: tiny_xmv<N, EK, LAP>(S, ek, nu, m, lane, lcol, lrw, lkab, lw, llab, nund, lr0, lr1); break;
    MGK_TINY_CASE(1) MGK_TINY_CASE(2) MGK_TINY_CASE(3) MGK_TINY_CASE(4) MGK_TINY_CASE(5)
#undef MGK_TINY_CASE
    default:  // edgeless L: OFF = 0 (an edgeless U has no rows to walk either)
      for (int e = lane; e < nu * m; e += 32) S.AP[e] = S.SS[e] * S.P[e];
      __syncwarp();
  }
}

template <int EK>
__device__ __forceinline__ void solve_tiny(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek,
                                        const SolveParams& prm, const SolveOut& out, const GraphDesc& U,
                                        const GraphDesc& L, TinySmem& S, int lane, double& value_out, int64_t& it_out,
                                        bool& conv_out, double& rr_out, float* nw, bool swap) {
  const int nu = U.n, m = L.n, nm = nu * m;
  const bool vlab = (vk.kind != KK_CONST1 && vk.kind != KK_NONE && ds.nl_kind != LK_NONE);
  // kappa_e = 1 with a large diag / s: A p = s p - sum c (p_j - p_i), s in FP64 (mgk_dev.cuh kLapFactor)
  const bool lap = EK == KK_NONE && laplacian_pair(prm, U, L);
  // lane slots of L: undirected edge u = lane + 32 t = {l, c} (l < c) -> columns c and l, weight, label and
  // the directed positions of l -> c and c -> l (upper entries compacted by ballot into SEG first)
  const int SL = 2 * L.ne, nund = SL >> 1;
  int lcol[kTinySlots], lrw[kTinySlots], lkab[kTinySlots];
  float lw[kTinySlots], llab[kTinySlots];
  {
    const float4* lr = ds.rowent + L.nz_off;
    int* upos = reinterpret_cast<int*>(S.SEG);
    int base = 0;
    for (int k0 = 0; k0 < SL; k0 += 32) {
      const int k = k0 + lane;
      bool up = false;
      if (k < SL) {
        int r = 0;
        while (S.lrow[r + 1] <= k) ++r;
        up = r < __float_as_int(lr[k].x);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, up);
      if (up) upos[base + __popc(bal & ((1u << lane) - 1u))] = k;
      base += __popc(bal);
    }
    __syncwarp();
#pragma unroll
    for (int t = 0; t < kTinySlots; ++t) {
      const int u = lane + 32 * t;
      lcol[t] = 0;
      lrw[t] = 0;
      lkab[t] = 0;
      lw[t] = 0.0f;
      llab[t] = 0.0f;
      if (u < nund) {
        const int ka = upos[u];
        const float4 e = lr[ka];
        int l = 0;
        while (S.lrow[l + 1] <= ka) ++l;
        const int c = __float_as_int(e.x);
        int kb = S.lrow[c];
        while (__float_as_int(lr[kb].x) != l) ++kb;
        lcol[t] = c;
        lrw[t] = l;
        lw[t] = e.y;
        llab[t] = e.z;
        lkab[t] = ka | (kb << 16);
      }
    }
    __syncwarp();
  }
  const int lr0 = lane < m ? S.lrow[lane] : 0, lr1 = lane < m ? S.lrow[lane + 1] : 0;
  double bb_u = 0.0, bb_l = 0.0;
  if (lane < nu) {
    double dq = ds.deg[U.node_off + lane] * ds.q64[U.node_off + lane];
    bb_u = dq * dq;
  }
  if (lane < m) {
    double dq = ds.deg[L.node_off + lane] * ds.q64[L.node_off + lane];
    bb_l = dq * dq;
  }
  double rho = 0.0, rr = 0.0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int e = lane + 32 * s;
    if (e < nm) {
      const int i = e / m, l = e - i * m;
      const int64_t vu = U.node_off + i, vl = L.node_off + l;
      const double dg = diag_of(ds, vk, prm, out, vlab, vu, vl);
      const double b = (ds.deg[vu] * ds.q64[vu]) * (ds.deg[vl] * ds.q64[vl]);
      S.RD[e] = 1.0 / dg;
      S.SS[e] = lap ? shifted_diag(ds, dg, vu, vl) : dg;
      S.R[e] = b;
      S.X[e] = 0.0;
      const double z = b / dg;
      S.P[e] = z;
      rho += b * z;
      rr += b * b;
    }
  }
  const double eps = prm.tol2 * warp_sum(bb_u) * warp_sum(bb_l);
  rho = warp_sum(rho);
  rr = warp_sum(rr);
  bool conv = rr < eps;
  const int64_t max_iter = prm.max_iter > 0 ? prm.max_iter : 10ll * nm;
  int64_t it = 0;
  __syncwarp();
  while (!conv && it < max_iter) {
    if (lap)
      tiny_xmv_dispatch<EK, true>(S, ek, nu, m, lane, lcol, lrw, lkab, lw, llab, nund, lr0, lr1);
    else
      tiny_xmv_dispatch<EK, false>(S, ek, nu, m, lane, lcol, lrw, lkab, lw, llab, nund, lr0, lr1);
    ++it;
    double pap = 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int e = lane + 32 * s;
      if (e < nm) pap += S.P[e] * S.AP[e];
    }
    const double alpha = rho / warp_sum(pap);
    double rr_l = 0.0, rz_l = 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int e = lane + 32 * s;
      if (e < nm) {
        S.X[e] += alpha * S.P[e];
        const double r = S.R[e] - alpha * S.AP[e];
        S.R[e] = r;
        rr_l += r * r;
        rz_l += r * (r * S.RD[e]);
      }
    }
    rr = warp_sum(rr_l);
    const double rho_next = warp_sum(rz_l);
    if (rr < eps) {
      conv = true;
      break;
    }
    const double beta = rho_next / rho;
    __syncwarp();
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int e = lane + 32 * s;
      if (e < nm) S.P[e] = S.R[e] * S.RD[e] + beta * S.P[e];
    }
    rho = rho_next;
    __syncwarp();
  }
  double val = 0.0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int e = lane + 32 * s;
    if (e < nm) {
      const int i = e / m, l = e - i * m;
      val += (double)ds.p[U.node_off + i] * (double)ds.p[L.node_off + l] * S.X[e];
      if (nw) nw[swap ? (int64_t)l * nu + i : (int64_t)e] = (float)S.X[e];
    }
  }
  value_out = warp_sum(val);
  it_out = it;
  conv_out = conv;
  rr_out = rr;
}

// ---------------------------------------------------------------------------
// XMV, labeled: OFF[i][l] for all U-rows i, undirected L slots per lane.
// ---------------------------------------------------------------------------
// acc[t], acc_b[t] += kappa(e_k, e'_t) w_k P[j_k][c_t] and ... P[j_k][l_t]: undirected L edge t = {l_t, c_t}
// (one edge-kernel value for both directed entries; the per-entry accumulation order is unchanged)
template <int NSU, int EK, int SLM, class Smem>
__device__ __forceinline__ void accumulate_row_sym(const Smem& S, const KernelDesc& ek, int i, const char* pbase,
                                                   const int (&lcoff)[SLM], const int (&lroff)[SLM],
                                                   const float (&llab)[SLM], float (&acc)[NSU],
                                                   float (&accb)[NSU]) {
  const int k1 = S.urow[i + 1];
  int k = S.urow[i];
  for (; k + 1 < k1; k += 2) {
    const float4 e0 = S.UE[k], e1 = S.UE[k + 1];
    const char* r0 = pbase + __float_as_int(e0.z);
    const char* r1 = pbase + __float_as_int(e1.z);
    float pa0[NSU], pb0[NSU], pa1[NSU], pb1[NSU];
#pragma unroll
    for (int t = 0; t < NSU; ++t) {
      pa0[t] = *reinterpret_cast<const float*>(r0 + lcoff[t]);
      pb0[t] = *reinterpret_cast<const float*>(r0 + lroff[t]);
      pa1[t] = *reinterpret_cast<const float*>(r1 + lcoff[t]);
      pb1[t] = *reinterpret_cast<const float*>(r1 + lroff[t]);
    }
#pragma unroll
    for (int t = 0; t < NSU; ++t) {
      const float c0 = edge_kappa_w<EK>(ek, e0.y, llab[t], e0.x);
      const float c1 = edge_kappa_w<EK>(ek, e1.y, llab[t], e1.x);
      acc[t] = fmaf(c0, pa0[t], acc[t]);
      accb[t] = fmaf(c0, pb0[t], accb[t]);
      acc[t] = fmaf(c1, pa1[t], acc[t]);
      accb[t] = fmaf(c1, pb1[t], accb[t]);
    }
  }
  if (k < k1) {
    const float4 e0 = S.UE[k];
    const char* r0 = pbase + __float_as_int(e0.z);
#pragma unroll
    for (int t = 0; t < NSU; ++t) {
      const float c0 = edge_kappa_w<EK>(ek, e0.y, llab[t], e0.x);
      acc[t] = fmaf(c0, *reinterpret_cast<const float*>(r0 + lcoff[t]), acc[t]);
      accb[t] = fmaf(c0, *reinterpret_cast<const float*>(r0 + lroff[t]), accb[t]);
    }
  }
}

// Labeled XMV over undirected L slots (NSU = ceil(S_L / 64)): each pass accumulates two U rows, writes
// the slot products to the directed positions of the segment buffer, and sums the L-row segments.
template <int NSU, int EK, int SLM, class Smem>
__device__ __forceinline__ void xmv_labeled_sym(Smem& S, const KernelDesc& ek, int nu, int m, int lane,
                                                const int (&lcoff)[SLM], const int (&lroff)[SLM],
                                                const int (&lkab)[SLM], const float (&lw)[SLM],
                                                const float (&llab)[SLM], int lr0, int lr1, int nund) {
  const char* pbase = reinterpret_cast<const char*>(&S.P[0][0]);
  for (int i = 0; i < nu; i += 2) {
    const bool two = i + 1 < nu;
    float a0[NSU], b0[NSU], a1[NSU], b1[NSU];
#pragma unroll
    for (int t = 0; t < NSU; ++t) a0[t] = b0[t] = a1[t] = b1[t] = 0.0f;
    accumulate_row_sym<NSU, EK, SLM>(S, ek, i, pbase, lcoff, lroff, llab, a0, b0);
    if (two) accumulate_row_sym<NSU, EK, SLM>(S, ek, i + 1, pbase, lcoff, lroff, llab, a1, b1);
#pragma unroll
    for (int t = 0; t < NSU; ++t) {
      if (lane + 32 * t < nund) {
        const int ka = lkab[t] & 0xffff, kb = lkab[t] >> 16;
        S.SEG[ka] = a0[t] * lw[t];
        S.SEG[kb] = b0[t] * lw[t];
        S.SEG[32 * SLM + ka] = a1[t] * lw[t];
        S.SEG[32 * SLM + kb] = b1[t] * lw[t];
      }
    }
    __syncwarp();
    if (lane < m) {
      float s0 = 0.0f, s1 = 0.0f;
#pragma unroll 2
      for (int q = lr0; q < lr1; ++q) {
        s0 += S.SEG[q];
        s1 += S.SEG[32 * SLM + q];
      }
      S.OFF[i][lane] = s0;
      if (two) S.OFF[i + 1][lane] = s1;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// XMV, unlabeled (kappa = 1): T = P B^T (slots + segment sums), OFF = A T.
// LAP (Laplacian splitting, mgk_dev.cuh kLapFactor): OFF = sum L (p_jj' - p_ii') instead, in the same
// factorised form via p_jj' - p_ii' = (p_jj' - p_ji') + (p_ji' - p_ii'):
//   T[j][i'] = sum_j' B_i'j' (p_jj' - p_ji'),  OFF[i][i'] = sum_j A_ij T[j][i'] + b_i' sum_j A_ij (p_ji' - p_ii')
// with b_i' = d'_i' - q'_i' (a coefficient of differences: its FP32 rounding is harmless).
template <int NS, int SLM, bool LAP, class Smem>
__device__ __forceinline__ void xmv_unlabeled(Smem& S, int nu, int m, int lane, const int (&lcoff)[SLM],
                                              const float (&lw)[SLM], const int (&lroff)[SLM], int lr0, int lr1,
                                              float lbm) {
  const char* pbase = reinterpret_cast<const char*>(&S.P[0][0]);
  for (int j = 0; j < nu; ++j) {
    const char* row = pbase + j * 128;
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      float v = *reinterpret_cast<const float*>(row + lcoff[t]);
      if constexpr (LAP) v -= *reinterpret_cast<const float*>(row + lroff[t]);
      S.SEG[lane + 32 * t] = lw[t] * v;
    }
    __syncwarp();
    if (lane < m) {
      float s = 0.0f;
#pragma unroll 1
      for (int q = lr0; q < lr1; ++q) s += S.SEG[q];
      S.T[j][lane] = s;
    }
    __syncwarp();
  }
  for (int i = 0; i < nu; ++i) {
    float s = 0.0f, s2 = 0.0f;
    const float pi = LAP ? S.P[i][lane] : 0.0f;
    for (int k = S.urow[i]; k < S.urow[i + 1]; ++k) {
      const float4 e = S.UE[k];
      const int j = __float_as_int(e.z) >> 7;
      s = fmaf(e.x, S.T[j][lane], s);
      if constexpr (LAP) s2 = fmaf(e.x, S.P[j][lane] - pi, s2);
    }
    if (lane < m) S.OFF[i][lane] = LAP ? fmaf(lbm, s2, s) : s;
  }
  __syncwarp();
}

template <int EK, int SLM, class Smem>
__device__ __forceinline__ void xmv_dispatch(int ns, Smem& S, const KernelDesc& ek, int nu, int m, int lane,
                                             const int (&lcoff)[SLM], const float (&lw)[SLM],
                                             const float (&llab)[SLM], const int (&lroff)[SLM],
                                             const int (&lkab)[SLM], int nund, int lr0, int lr1, bool lap,
                                             float lbm) {
  if constexpr (EK != KK_NONE) {
    switch ((nund + 31) >> 5) {
      case 1: xmv_labeled_sym<1, EK, SLM>(S, ek, nu, m, lane, lcoff, lroff, lkab, lw, llab, lr0, lr1, nund); return;
      case 2: xmv_labeled_sym<2, EK, SLM>(S, ek, nu, m, lane, lcoff, lroff, lkab, lw, llab, lr0, lr1, nund); return;
      case 3:
        if constexpr (SLM >= 5) xmv_labeled_sym<3, EK, SLM>(S, ek, nu, m, lane, lcoff, lroff, lkab, lw, llab, lr0, lr1, nund);
        return;
      case 4:
        if constexpr (SLM >= 7) xmv_labeled_sym<4, EK, SLM>(S, ek, nu, m, lane, lcoff, lroff, lkab, lw, llab, lr0, lr1, nund);
        return;
      case 5:
        if constexpr (SLM >= 9) xmv_labeled_sym<5, EK, SLM>(S, ek, nu, m, lane, lcoff, lroff, lkab, lw, llab, lr0, lr1, nund);
        return;
      default:  // edgeless lane graph: OFF = 0
        for (int i = 0; i < nu; ++i) S.OFF[i][lane] = 0.0f;
        __syncwarp();
        return;
    }
  } else {
#define MGK_XMV_CASE(N)                                                                  \
  case N:                                                                                \
    if constexpr (N <= SLM) {                                                            \
      if (lap)                                                                           \
        xmv_unlabeled<N, SLM, true>(S, nu, m, lane, lcoff, lw, lroff, lr0, lr1, lbm);    \
      else                                                                               \
        xmv_unlabeled<N, SLM, false>(S, nu, m, lane, lcoff, lw, lroff, lr0, lr1, lbm);   \
    }                                                                                    \
    break;
  switch (ns) {
    MGK_XMV_CASE(1)
    MGK_XMV_CASE(2)
    MGK_XMV_CASE(3)
    MGK_XMV_CASE(4)
    MGK_XMV_CASE(5)
    MGK_XMV_CASE(6)
    MGK_XMV_CASE(7)
    MGK_XMV_CASE(8)
    MGK_XMV_CASE(9)
    MGK_XMV_CASE(10)
    default:  // ns == 0: edgeless lane graph, OFF = 0
      for (int i = 0; i < nu; ++i) S.OFF[i][lane] = 0.0f;
      __syncwarp();
  }
#undef MGK_XMV_CASE
  }
  static_assert(SLOTS == 10 && SLM <= SLOTS, "xmv_dispatch covers 1..10 slots");
}

// SLM: lane-side slot capacity of this instantiation.  SLM = 4 (S_L <= 128)
// covers ~95% of QM7-shaped pairs with a third of the registers; the host
// routes the pairs whose graphs both exceed 128 nonzeros to the SLM = 10
// instantiation (gram_jobs: the wide-prefix triangle), so every pair of a
// narrow job has a narrow graph for the lane side.
template <int EK, bool NODEWISE, int SLM>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, SLM <= 4 ? 8 : 6)
k_pcg_warp(DatasetDev ds, KernelDesc vk, KernelDesc ek, PairJob job, SolveParams prm, SolveOut out,
           unsigned long long* queue) {
  constexpr bool UNLAB = (EK == KK_NONE);
  using Smem = WarpSmem<UNLAB, NODEWISE, SLM>;
  static_assert(sizeof(float) * 2 * NU * 32 >= sizeof(float4) * SMAX, "staging area too small");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  Smem& S = reinterpret_cast<Smem*>(smem_raw)[threadIdx.x >> 5];
  float4* stage = reinterpret_cast<float4*>(&S.P[0][0]);
  const int el_dim = ds.el_dim;
  const bool vlab = (vk.kind != KK_CONST1 && vk.kind != KK_NONE && ds.nl_kind != LK_NONE);

  for (;;) {
    unsigned long long pid = 0;
    if (lane == 0) pid = atomicAdd(queue, 1ull);
    pid = __shfl_sync(0xffffffffu, pid, 0);
    if (pid >= (unsigned long long)job.npairs) break;
    int32_t ga, gb;
    decode_pair(job, (int64_t)pid, ga, gb);
    const GraphDesc A = ds.graphs[ga], B = ds.graphs[gb];
    // orientation: L takes the graph that minimises S_U * ceil(S_L / 32), within SLM slots
    const int SA = 2 * A.ne, SB = 2 * B.ne;
    const int nsA = (SA + 31) >> 5, nsB = (SB + 31) >> 5;
#ifndef MGK_ORIENT
#define MGK_ORIENT 0
#endif
    // MGK_ORIENT 1 (labeled, undirected slots): shared-memory wavefronts per U nonzero ~ 2 (row entry)
    // + 2 ceil(S_L / 64) (two gathers per undirected slot)
    const long costAB = (MGK_ORIENT && EK != KK_NONE) ? (long)SA * (2 + 2 * ((SB + 63) >> 6)) + 4 * A.n
                                                       : (long)SA * nsB + A.n;  // U = A, L = B
    const long costBA = (MGK_ORIENT && EK != KK_NONE) ? (long)SB * (2 + 2 * ((SA + 63) >> 6)) + 4 * B.n
                                                       : (long)SB * nsA + B.n;
    bool swap = (costBA < costAB);
    if (SLM < SLOTS) {
      if ((swap ? nsA : nsB) > SLM) swap = !swap;
      if ((swap ? nsA : nsB) > SLM) continue;  // not routed here by the host (both graphs wide)
    }
    const GraphDesc U = swap ? B : A;
    const GraphDesc L = swap ? A : B;
    const int nu = U.n, m = L.n;
    const int SL = 2 * L.ne;
    const int ns = (SL + 31) >> 5;

    // ---- prologue: octiles -> rows (U into UE, L staged then held in registers)
    // rows from the dataset's row expansion of the octiles (k_rows_fill: {col, w, label, log2 w},
    // ascending column per row): independent coalesced 16-byte loads, no per-pair bit scans
    {
      const float4* ur = ds.rowent + U.nz_off;
      const float4* lr = ds.rowent + L.nz_off;
      const int SU = 2 * U.ne;
      for (int k = lane; k < SU; k += 32) {
        const float4 e = ur[k];
        S.UE[k] = make_float4(EK == KK_SE ? e.w : e.y, e.z, __int_as_float(__float_as_int(e.x) * 128), 0.0f);
      }
      for (int k = lane; k < SL; k += 32) stage[k] = lr[k];
      if (lane <= nu) S.urow[lane] = ds.rowptr[U.rowptr_off + lane];
      if (lane <= m) S.lrow[lane] = ds.rowptr[L.rowptr_off + lane];
    }
    __syncwarp();
    int lcoff[SLM], lroff[SLM];
    float lw[SLM], llab[SLM];
    int lkab[SLM];  // labeled: SEG positions of the two directed entries of an undirected L edge (16 + 16 bits)
    if constexpr (UNLAB) {
#pragma unroll
      for (int t = 0; t < SLM; ++t) {
        const int k = lane + 32 * t;
        lcoff[t] = 0;
        lroff[t] = 0;
        lw[t] = 0.0f;
        llab[t] = 0.0f;
        lkab[t] = 0;
        if (k < SL) {
          const float4 e = stage[k];
          lcoff[t] = __float_as_int(e.x) * 4;
          lw[t] = e.y;
          llab[t] = e.z;
          int r = 0;  // L row of the slot (Laplacian splitting)
          while (S.lrow[r + 1] <= k) ++r;
          lroff[t] = r * 4;
        }
      }
    } else {
      // Undirected L edges on the lanes: edge {l, c} (l < c) owns both directed entries l->c and c->l,
      // whose contributions share one edge-kernel value -- one MUFU.EX2 feeds two accumulators.
      // Upper entries (l < c) in row order, compacted by ballot: UPOS[u] = directed position.
      int* upos = reinterpret_cast<int*>(S.SEG);
      int base = 0;
      for (int k0 = 0; k0 < SL; k0 += 32) {
        const int k = k0 + lane;
        bool up = false;
        if (k < SL) {
          int r = 0;
          while (S.lrow[r + 1] <= k) ++r;
          up = r < __float_as_int(stage[k].x);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, up);
        if (up) upos[base + __popc(bal & ((1u << lane) - 1u))] = k;
        base += __popc(bal);
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < SLM; ++t) {
        const int u = lane + 32 * t;
        lcoff[t] = 0;
        lroff[t] = 0;
        lw[t] = 0.0f;
        llab[t] = 0.0f;
        lkab[t] = 0;
        if (u < (SL >> 1)) {
          const int ka = upos[u];
          const float4 e = stage[ka];
          int l = 0;
          while (S.lrow[l + 1] <= ka) ++l;
          const int c = __float_as_int(e.x);
          int kb = S.lrow[c];  // the reverse entry c -> l in row c
          while (__float_as_int(stage[kb].x) != l) ++kb;
          lcoff[t] = c * 4;  // l -> c gathers P[j][c]
          lroff[t] = l * 4;  // c -> l gathers P[j][l]
          lw[t] = e.y;
          llab[t] = e.z;
          lkab[t] = ka | (kb << 16);
        }
      }
    }
    int lr0 = 0, lr1 = 0;
    if (lane < m) {
      lr0 = S.lrow[lane];
      lr1 = S.lrow[lane + 1];
    }

    __syncwarp();  // staging (P/OFF) is free again

    // ---- node data: L on lanes, U in shared memory; vectors as [U node][lane]
    double ldq = 0.0;
    float lp = 0.0f, lbm = 0.0f;
    if (lane < m) {
      const int64_t v = L.node_off + lane;
      ldq = ds.deg[v] * ds.q64[v];
      lp = ds.p[v];
      lbm = ds.dm[v];
    }
    // kappa_e = 1 pairs with a large diag / s: Laplacian splitting (dv = s, preconditioner s + udm lbm)
    const bool lap = UNLAB && laplacian_pair(prm, U, L);
    double bb_u = 0.0;
    if (lane < nu) {
      const int64_t v = U.node_off + lane;
      const double dq = ds.deg[v] * ds.q64[v];
      S.udq[lane] = (float)dq;
      S.upq[lane] = ds.p[v];
      if constexpr (UNLAB) S.udm[lane] = ds.dm[v];
      bb_u = dq * dq;
    }
    // b = (d q) (x) (d' q');  eps = tol^2 b.b  (solver.py:69-74, 88) -- b.b is separable
    const double bb = warp_sum(bb_u) * warp_sum(ldq * ldq);
    const double eps = prm.tol2 * bb;
    const int64_t max_iter = prm.max_iter > 0 ? prm.max_iter : 10ll * nu * m;
    __syncwarp();

    // x = 0, r = b, z = r / diag, p = z  (solver.py:91-97); R and diag in registers.
    // Scalar categorical delta / no vertex kernel (the common case) inline: diag = d d' / kv with
    // kv in {1, h}; anything else goes through the generic diag_of.
    const bool active = lane < m;
    const bool vfast = !vlab || (vk.kind == KK_DELTA && ds.nl_dim == 1);
    double ldeg = 1.0;
    int llabel = 0;
    if (vfast && active) {
      ldeg = ds.deg[L.node_off + lane];
      if (vlab) llabel = __float_as_int(ds.vlabel[L.node_off + lane]);
    }
    const double inv_h = vlab ? 1.0 / (double)fmaxf(vk.h, prm.v_min) : 1.0;
    float rv[NU], dv[NU];
    double rho = 0.0, rr = 0.0;
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      rv[i] = 0.0f;
      dv[i] = 1.0f;
      if (i < nu) {
        float p0 = 0.0f;
        if (active) {
          const int64_t vu = U.node_off + i, vl = L.node_off + lane;
          double dg;
          if (vfast) {
            const bool same = !vlab || __float_as_int(ds.vlabel[vu]) == llabel;
            dg = ds.deg[vu] * ldeg * (same ? 1.0 : inv_h);
          } else {
            dg = diag_of(ds, vk, prm, out, vlab, vu, vl);
          }
          dv[i] = (float)(lap ? shifted_diag(ds, dg, vu, vl) : dg);
          rv[i] = (float)((double)S.udq[i] * ldq);
          p0 = rv[i] * rcp_approx((float)dg);
          rho += (double)rv[i] * (double)p0;
          rr += (double)rv[i] * (double)rv[i];
        }
        S.P[i][lane] = p0;
        if constexpr (NODEWISE) S.X[i][lane] = 0.0f;
      }
    }
    rho = warp_sum(rho);
    rr = warp_sum(rr);
    bool conv = rr < eps;
    int64_t it = 0;
    double value = 0.0;
    const bool self_pair = (ga == gb);
    __syncwarp();

    while (!conv && it < max_iter) {
      // ---------------- off-diagonal product OFF = (A (x) A' . ke) P
      xmv_dispatch<EK, SLM>(ns, S, ek, nu, m, lane, lcoff, lw, llab, lroff, lkab, SL >> 1, lr0, lr1, lap, lbm);
      if (self_pair) {
        // self pair: the exact operator maps symmetric fields to symmetric fields;
        // symmetrising keeps the FP32 Krylov space in that subspace as the FP64
        // reference does (diag * P is exactly symmetric already)
        for (int i = 0; i < lane && active; ++i) {
          const float v = 0.5f * (S.OFF[i][lane] + S.OFF[lane][i]);
          S.OFF[i][lane] = v;
          S.OFF[lane][i] = v;
        }
        __syncwarp();
      }
      ++it;
      // ---------------- PCG update (solver.py:98-110); A p = diag * p - OFF
      // Dot products: FP32 partial sums of two rows, promoted to FP64 once per pair of rows (halves the
      // F2F conversions, which share the XU pipe with MUFU.EX2); px . p (value only) in FP32 per lane.
      double pap = 0.0;
      float pend = 0.0f, pxp32 = 0.0f;
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        if (i >= nu) break;  // warp-uniform: no issue slots spent on absent rows
        if (active) {
          const float p = S.P[i][lane];
          const float ap = fmaf(dv[i], p, -S.OFF[i][lane]);
          S.OFF[i][lane] = ap;
          if (i & 1) {
            pap += (double)fmaf(p, ap, pend);
            pend = 0.0f;
          } else {
            pend = p * ap;
          }
          pxp32 = fmaf(S.upq[i], p, pxp32);
        }
      }
      pap = warp_sum(pap + (double)pend);
      const double pxp = warp_sum((double)pxp32 * (double)lp);
      const double alpha = rho / pap;
      value += alpha * pxp;  // px . x accumulated as sum_k alpha_k (px . p_k)
      const float af = (float)alpha;
      double rr_l = 0.0, rz_l = 0.0;
      float rr_p = 0.0f, rz_p = 0.0f;
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        if (i >= nu) break;  // warp-uniform: no issue slots spent on absent rows
        if (active) {
          if constexpr (NODEWISE) S.X[i][lane] = fmaf(af, S.P[i][lane], S.X[i][lane]);
          const float r = fmaf(-af, S.OFF[i][lane], rv[i]);
          // preconditioner: the full diagonal (Laplacian splitting: s + (d - q)(d' - q'))
          const float z = r * rcp_approx(UNLAB && lap ? fmaf(S.udm[i], lbm, dv[i]) : dv[i]);
          rv[i] = r;
          S.OFF[i][lane] = z;
          if (i & 1) {
            rr_l += (double)fmaf(r, r, rr_p);
            rz_l += (double)fmaf(r, z, rz_p);
            rr_p = rz_p = 0.0f;
          } else {
            rr_p = r * r;
            rz_p = r * z;
          }
        }
      }
      rr = warp_sum(rr_l + (double)rr_p);
      const double rho_next = warp_sum(rz_l + (double)rz_p);
      if (rr < eps) {
        conv = true;
        break;
      }
      const float beta = (float)(rho_next / rho);
      if (active) {
#pragma unroll 4
        for (int i = 0; i < nu; ++i) S.P[i][lane] = fmaf(beta, S.P[i][lane], S.OFF[i][lane]);
      }
      rho = rho_next;
      __syncwarp();
    }

    if constexpr (NODEWISE) {
      if (out.nodewise && active) {
        float* nw = out.nodewise + out.nodewise_off[pid];
        // field is [n_a][n_b] with a = first graph of the pair
        for (int i = 0; i < nu; ++i) {
          const int64_t idx = swap ? (int64_t)lane * nu + i : (int64_t)i * m + lane;
          nw[idx] = S.X[i][lane];
        }
      }
    }
    write_pair_outputs(out, pid, ga, gb, value, it, conv, rr, lane);
    __syncwarp();
  }
}

// Tiny-pair kernel: warp per pair, FP64 vectors (see solve_tiny).
template <int EK>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 8)
k_pcg_tiny(DatasetDev ds, KernelDesc vk, KernelDesc ek, PairJob job, SolveParams prm, SolveOut out,
           unsigned long long* queue) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  TinySmem& S = reinterpret_cast<TinySmem*>(smem_raw)[threadIdx.x >> 5];
  for (;;) {
    unsigned long long pid = 0;
    if (lane == 0) pid = atomicAdd(queue, 1ull);
    pid = __shfl_sync(0xffffffffu, pid, 0);
    if (pid >= (unsigned long long)job.npairs) break;
    int32_t ga, gb;
    decode_pair(job, (int64_t)pid, ga, gb);
    const GraphDesc A = ds.graphs[ga], B = ds.graphs[gb];
    // U = the graph with fewer nodes (rows walked by the warp), L = the other (lane slots, small class)
    const bool swap = (B.n < A.n) || (B.n == A.n && B.ne < A.ne);
    const GraphDesc U = swap ? B : A, L = swap ? A : B;
    {  // rows from the dataset's row expansion of the octiles (see k_pcg_warp)
      const float4* ur = ds.rowent + U.nz_off;
      for (int k = lane; k < 2 * U.ne; k += 32) {
        const float4 e = ur[k];
        S.UE[k] = make_float4(EK == KK_SE ? e.w : e.y, e.z, __int_as_float(__float_as_int(e.x) * L.n), 0.0f);
      }
      if (lane <= U.n) S.urow[lane] = ds.rowptr[U.rowptr_off + lane];
      if (lane <= L.n) S.lrow[lane] = ds.rowptr[L.rowptr_off + lane];
    }
    __syncwarp();
    double val, rr;
    int64_t it;
    bool conv;
    float* nw = out.nodewise ? out.nodewise + out.nodewise_off[pid] : nullptr;
    solve_tiny<EK>(ds, vk, ek, prm, out, U, L, S, lane, val, it, conv, rr, nw, swap);
    write_pair_outputs(out, pid, ga, gb, val, it, conv, rr, lane);
    __syncwarp();
  }
}

template <int EK>
static cudaError_t launch_tiny_ek(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek,
                                  const PairJob& job, const SolveParams& prm, const SolveOut& out,
                                  unsigned long long* queue, int num_sms, cudaStream_t stream) {
  auto kern = k_pcg_tiny<EK>;
  const size_t smem = sizeof(TinySmem) * kWarpsPerBlock;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarpsPerBlock * 32, smem);
  if (e != cudaSuccess) return e;
  int64_t blocks = (int64_t)(per_sm < 1 ? 1 : per_sm) * num_sms;
  const int64_t need = (job.npairs + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, kWarpsPerBlock * 32, smem, stream>>>(ds, vk, ek, job, prm, out, queue);
  return cudaGetLastError();
}

cudaError_t launch_pcg_tiny(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                            const SolveParams& prm, const SolveOut& out, unsigned long long* queue, int num_sms,
                            cudaStream_t stream) {
  int kind = prm.labeled ? ek.kind : KK_NONE;
  if (kind == KK_CONST1) kind = KK_NONE;
  switch (kind) {
    case KK_SE: return launch_tiny_ek<KK_SE>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
    case KK_DELTA: return launch_tiny_ek<KK_DELTA>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
    case KK_POLY: return launch_tiny_ek<KK_POLY>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
    default: return launch_tiny_ek<KK_NONE>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
  }
}

template <int EK, bool NODEWISE, int SLM>
static cudaError_t launch_ek(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                             const SolveParams& prm, const SolveOut& out, unsigned long long* queue, int num_sms,
                             cudaStream_t stream) {
  using Smem = WarpSmem<EK == KK_NONE, NODEWISE, SLM>;
  auto kern = k_pcg_warp<EK, NODEWISE, SLM>;
  const size_t smem = sizeof(Smem) * kWarpsPerBlock;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarpsPerBlock * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)per_sm * num_sms;
  const int64_t need = (job.npairs + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, kWarpsPerBlock * 32, smem, stream>>>(ds, vk, ek, job, prm, out, queue);
  return cudaGetLastError();
}

template <bool NODEWISE, int SLM>
static cudaError_t launch_nw(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                             const SolveParams& prm, const SolveOut& out, unsigned long long* queue, int num_sms,
                             cudaStream_t stream) {
  int kind = prm.labeled ? ek.kind : KK_NONE;
  if (kind == KK_CONST1) kind = KK_NONE;
  switch (kind) {
    case KK_SE: return launch_ek<KK_SE, NODEWISE, SLM>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
    case KK_DELTA: return launch_ek<KK_DELTA, NODEWISE, SLM>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
    case KK_POLY: return launch_ek<KK_POLY, NODEWISE, SLM>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
    default: return launch_ek<KK_NONE, NODEWISE, SLM>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
  }
}

cudaError_t launch_pcg_warp(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                            const SolveParams& prm, const SolveOut& out, unsigned long long* queue, int num_sms,
                            int slots, cudaStream_t stream) {
  if (slots <= kNarrowSlots) {
    if (out.nodewise) return launch_nw<true, kNarrowSlots>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
    return launch_nw<false, kNarrowSlots>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
  }
  if (out.nodewise) return launch_nw<true, SLOTS>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
  return launch_nw<false, SLOTS>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
}

}  // namespace mgk
