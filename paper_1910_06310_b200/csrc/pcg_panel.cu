// K3 + K4 (panel class): one CTA solves one graph pair of any size.
//
// Replaces, per pair, ProductOperator.__init__ (product.py:184-222), apply /
// apply_offdiag (product.py:351-419) and solve_pcg (solver.py:77-121) for the
// pairs the warp solver cannot hold in one warp (configs 3-5: 24 < n <= 5000).
//
// Same on-the-fly XMV as pcg_warp.cu, generalised from "the whole lane graph in
// one warp's registers" to row panels: the lane graph L is cut (once per
// dataset, on the host from the degree sequence) into panels of consecutive
// rows holding at most 128 nonzeros; a warp holds one panel in registers
// (lane l owns panel nonzeros l + 32 t, t < NS) and walks a chunk of U rows:
//
//   acc[t]  = sum_{k in U(i)} kappa(e_k, e'_t) w_k P[j_k][col_L(t)]
//   OFF[i][r] = sum_{t in L(r)} acc[t] w'_t          (segment sum in shared memory)
//   AP[i][r]  = diag[i][r] P[i][r] - OFF[i][r]
//
// Every (panel, U-row chunk) item writes a disjoint block of AP, so there are
// no atomics and the result is independent of the warp schedule.  Small lane
// graphs (S_L <= 64) use a single panel with 2 slots per lane.
//
// PCG state: P and AP live in shared memory when 2 n m floats fit the per-CTA
// budget chosen at launch (mid-size pairs), otherwise in a per-CTA slab in HBM
// (read through L1/L2; the gathers P[j][col] of one warp touch a narrow column
// window of a few rows, which is what the PBR ordering buys).  R, diag and the
// nodewise iterate always sit in the slab (streamed once per iteration).
// Dot products are FP64 block reductions in a fixed order (deterministic).
#include <cooperative_groups.h>

#include "mgk_internal.h"

namespace mgk {

// This file is compiled twice: CTAs of 256 threads (namespace p256: mid-size pairs, two CTAs per SM)
// and of 512 threads (p512: large pairs, one CTA per SM so the resident P vectors stay in L2).
#ifndef MGK_PANEL_NS
#define MGK_PANEL_NS p256
#endif
namespace MGK_PANEL_NS {

namespace cg = cooperative_groups;

#ifndef MGK_PANEL_THREADS
#define MGK_PANEL_THREADS 256
#endif
constexpr int kPT = MGK_PANEL_THREADS;  // threads per CTA
constexpr int kPW = kPT / 32;     // warps per CTA
constexpr int kSegFloats = 2 * kPanelCap;  // per-warp segment buffer (two U rows)
// Per-CTA cache of small graphs' row expansions (U up to kCacheU nonzeros, a single-panel L), so the
// XMV's row entries come from shared memory instead of L1/L2 on mid-size pairs.
constexpr int kCacheU = 1024;
constexpr int kCacheRows = 256;
constexpr int kCacheFloats = 4 * (kCacheU + kPanelCap) + 2 * (kCacheRows + 1) + 2;
constexpr int kPanelStaticSmem = (kPW * kSegFloats + kCacheFloats) * 4;
// Per-pair vectors in the panel slab / grid buffer: R, DG, X, P, AP, T (unlabeled: P B^T), SD (the
// shifted diagonal s of the Laplacian splitting).  capi.cu sizes both with kSlabVectors (mgk_internal.h).
static_assert(kSlabVectors == 7, "slab layout");

// Streaming (evict-first) access to the per-pair vectors that are read / written once per phase (R,
// the diagonals, X): they should not displace the P vectors whose scattered gathers feed the XMV from
// L2 (MGK_PANEL_STREAM=0 builds the plain accesses for A/B runs).
#ifndef MGK_PANEL_STREAM
#define MGK_PANEL_STREAM 1
#endif
__device__ __forceinline__ float ld_stream(const float* p) {
#if MGK_PANEL_STREAM
  return __ldcs(p);
#else
  return *p;
#endif
}
__device__ __forceinline__ void st_stream(float* p, float v) {
#if MGK_PANEL_STREAM
  __stcs(p, v);
#else
  *p = v;
#endif
}

// PCG vector passes over the elements e0, e0 + es, ... (es = the CTA's / grid's thread count), four
// elements per step with every load issued before the arithmetic (the streamed vectors come from
// HBM: four independent loads in flight per thread instead of one); per-thread accumulation order unchanged.
// A/B on the box: 4 for the 512-thread panel CTAs and the grid solver (config 3 +1.6 %, config-4 buckets
// +5-7 %); 1 for the 256-thread CTAs (the extra registers spill there: config 5 -7 % at 4).
#ifndef MGK_VEC_UNROLL
#define MGK_VEC_UNROLL (MGK_PANEL_THREADS >= 512 ? 4 : 1)
#endif
// x += alpha p, r -= alpha Ap, z = r / diag (stored over Ap); returns (r.r, r.z) partials
template <bool NODEWISE, class I>
__device__ __forceinline__ double2 pcg_pass2(I e0, I es, I nm, float af, const float* P, float* AP, float* R,
                                             const float* DG, float* X) {
  constexpr int U = MGK_VEC_UNROLL;
  double2 acc = make_double2(0.0, 0.0);
  for (I eb = e0; eb < nm; eb += U * es) {
    float ap[U], rv[U], dg[U], xv[U], pv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const I e = eb + u * es;
      if (e < nm) {
        ap[u] = AP[e];
        rv[u] = ld_stream(R + e);
        dg[u] = ld_stream(DG + e);
        if constexpr (NODEWISE) {
          xv[u] = ld_stream(X + e);
          pv[u] = P[e];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const I e = eb + u * es;
      if (e < nm) {
        if constexpr (NODEWISE) st_stream(X + e, fmaf(af, pv[u], xv[u]));
        const float r = fmaf(-af, ap[u], rv[u]);
        const float z = r * rcp_approx(dg[u]);
        st_stream(R + e, r);
        AP[e] = z;
        acc.x += (double)r * (double)r;
        acc.y += (double)r * (double)z;
      }
    }
  }
  return acc;
}

// p = z + beta p (z stored over Ap)
template <class I>
__device__ __forceinline__ void pcg_update_p(I e0, I es, I nm, float beta, float* P, const float* AP) {
  constexpr int U = MGK_VEC_UNROLL;
  for (I eb = e0; eb < nm; eb += U * es) {
    float pv[U], zv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const I e = eb + u * es;
      if (e < nm) {
        pv[u] = P[e];
        zv[u] = AP[e];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const I e = eb + u * es;
      if (e < nm) P[e] = fmaf(beta, pv[u], zv[u]);
    }
  }
}

__device__ __forceinline__ double2 block_sum2(double2 v, double2* buf) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  if (lane == 0) buf[w] = v;
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < kPW; ++k) {
    s.x += buf[k].x;
    s.y += buf[k].y;
  }
  return s;
}

// Gather addressing: each lane keeps a pointer to P[0][col(t)] per slot (made opaque to the compiler, so
// it is not re-associated into (j m + col) << 2 + P with a sign extension and a 64-bit carry chain), and a
// gather P[j][col(t)] is one IMAD.WIDE.U32 (lane pointer + 4 j m) + the load.  MGK_PANEL_LP=0: P + j m + col.
#ifndef MGK_PANEL_LP
#define MGK_PANEL_LP 1
#endif
__device__ __forceinline__ const float* opaque_ptr(const float* p) {
#if MGK_PANEL_LP
  const float* r;
  asm("mov.b64 %0, %1;" : "=l"(r) : "l"(p));
  return r;
#else
  return p;
#endif
}

// acc[t] += sum_{k in [k0, k1)} kappa(e_k, e'_t) w_k P[j_k][lcol[t]]   (U row, warp-uniform)
// LAP (kappa_e = 1, Laplacian splitting): the gathered values enter as differences P[j_k][lcol[t]] - pc[t]
// with pc[t] = P[i][row(t)] the element the contribution lands on (mgk_dev.cuh kLapFactor).
template <int NS, int EK, bool LAP = false>
__device__ __forceinline__ void row_accumulate(const KernelDesc& ek, const float4* __restrict__ ue, int k0, int k1,
                                               const float* const (&lp)[NS], int m,
                                               const float (&llab)[NS], float (&acc)[NS],
                                               const float (&pc)[NS]) {
  int k = k0;
#ifndef MGK_PANEL_UNROLL4
#define MGK_PANEL_UNROLL4 1
#endif
  if constexpr (MGK_PANEL_UNROLL4 != 0) {  // four nonzeros per step: 4 NS gathers in flight per warp
    for (; k + 3 < k1; k += 4) {
      float4 e[4];
      float pv[4][NS];
#pragma unroll
      for (int u = 0; u < 4; ++u) e[u] = ue[k + u];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned off = (unsigned)(__float_as_int(e[u].x) * m);
#pragma unroll
        for (int t = 0; t < NS; ++t) pv[u][t] = LAP ? lp[t][off] - pc[t] : lp[t][off];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int t = 0; t < NS; ++t)
          acc[t] = fmaf(edge_kappa_w<EK>(ek, e[u].z, llab[t], EK == KK_SE ? e[u].w : e[u].y), pv[u][t], acc[t]);
    }
  }
  for (; k + 1 < k1; k += 2) {
    const float4 e0 = ue[k], e1 = ue[k + 1];
    const unsigned o0 = (unsigned)(__float_as_int(e0.x) * m), o1 = (unsigned)(__float_as_int(e1.x) * m);
    float p0[NS], p1[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      p0[t] = lp[t][o0];
      p1[t] = lp[t][o1];
      if constexpr (LAP) {
        p0[t] -= pc[t];
        p1[t] -= pc[t];
      }
    }
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      acc[t] = fmaf(edge_kappa_w<EK>(ek, e0.z, llab[t], EK == KK_SE ? e0.w : e0.y), p0[t], acc[t]);
      acc[t] = fmaf(edge_kappa_w<EK>(ek, e1.z, llab[t], EK == KK_SE ? e1.w : e1.y), p1[t], acc[t]);
    }
  }
  if (k < k1) {
    const float4 e0 = ue[k];
    const unsigned o0 = (unsigned)(__float_as_int(e0.x) * m);
#pragma unroll
    for (int t = 0; t < NS; ++t)
      acc[t] = fmaf(edge_kappa_w<EK>(ek, e0.z, llab[t], EK == KK_SE ? e0.w : e0.y),
                    LAP ? lp[t][o0] - pc[t] : lp[t][o0], acc[t]);
  }
}

// L row of every slot of a panel (Laplacian splitting): lrow[t] = r with lrp[r] <= kbeg + lane + 32 t < lrp[r+1]
template <int NS>
__device__ __forceinline__ void slot_rows(const int32_t* lrp, int rbeg, int rend, int kbeg, int kend, int lane,
                                          int (&lrow)[NS]) {
#pragma unroll
  for (int t = 0; t < NS; ++t) {
    const int k = kbeg + lane + 32 * t;
    int lo = rbeg, hi = rend;  // largest r in [rbeg, rend) with lrp[r] <= k
    if (k >= kend) {
      lrow[t] = rbeg;
      continue;
    }
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (lrp[mid] <= k) lo = mid; else hi = mid;
    }
    lrow[t] = lo;
  }
}


struct PairView {
  const int32_t* urp;   // U row pointers (relative to ue)
  const float4* ue;     // U row entries
  const int32_t* lrp;
  const float4* le;
  const int32_t* prow;  // L panel row boundaries (null: single panel = all rows)
  const int2* lsym;     // L's undirected edges: directed positions (i -> j, j -> i) in le (ds.symk)
  int n, m, np, rpc, nund;
};

// Largest U-row chunk of a panel-solver item (A/B on config 3 with chunk-major items: 8 rows +5 % over 32)
#ifndef MGK_PANEL_RPC_MAX
#define MGK_PANEL_RPC_MAX 8
#endif
constexpr int kPanelRpcMax = MGK_PANEL_RPC_MAX;

// Prefetch of the epilogue diagonal (A/B on the box: config 3 +3 % on the 512-thread CTAs; config 5's
// 256-thread CTAs -1.4 %, so off there)
#ifndef MGK_PANEL_DGPF
#define MGK_PANEL_DGPF (MGK_PANEL_THREADS >= 512)
#endif

// Item order: chunk-major (consecutive warps take the panels of one U-row chunk, so the CTA's gathers
// share the P rows of that chunk's neighbourhood in L1; A/B on the box: +16 % on config 3, +22 % on the
// SE grid buckets of config 4) or panel-major (MGK_PANEL_CMAJOR=0).
#ifndef MGK_PANEL_CMAJOR
#define MGK_PANEL_CMAJOR 1
#endif
__device__ __forceinline__ void item_coords(int64_t item, int np, int nchunks, int& p, int& c) {
#if MGK_PANEL_CMAJOR
  c = (int)(item / np);
  p = (int)(item - (int64_t)c * np);
#else
  p = (int)(item / nchunks);
  c = (int)(item - (int64_t)p * nchunks);
#endif
}

// AP = diag * P - XMV(P) over the (panel, chunk) items w0, w0 + wstride, ...
// When part != nullptr the warp also accumulates (p.Ap, px.p) over the
// elements it wrote (every element is written by exactly one item).
// LAP: AP = s * P - sum L (P_jj' - P_ii') with DG = s (the caller passes the shifted diagonal).
template <int NS, int EK, bool LAP = false>
__device__ void xmv_panels(const KernelDesc& ek, const PairView& v, const float* P, float* AP, const float* DG,
                           float* SEG, int lane, int64_t w0, int64_t wstride, const float* pu, const float* pl,
                           double2* part) {
  const int n = v.n, m = v.m;
  const int nchunks = (n + v.rpc - 1) / v.rpc;
  const int64_t items = (int64_t)v.np * nchunks;
  double pap = 0.0, pxp = 0.0;
  for (int64_t item = w0; item < items; item += wstride) {
    int p, c;
    item_coords(item, v.np, nchunks, p, c);
    const int rbeg = v.prow ? v.prow[p] : 0;
    const int rend = v.prow ? v.prow[p + 1] : m;
    const int kbeg = v.lrp[rbeg], kend = v.lrp[rend];
    int lcol[NS];
    float lw[NS], llab[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const int k = kbeg + lane + 32 * t;
      lcol[t] = 0;
      lw[t] = 0.0f;
      llab[t] = 0.0f;
      if (k < kend) {
        const float4 e = v.le[k];
        lcol[t] = __float_as_int(e.x);
        lw[t] = e.y;
        llab[t] = e.z;
      }
    }
    int lrw[NS];
    if constexpr (LAP) slot_rows<NS>(v.lrp, rbeg, rend, kbeg, kend, lane, lrw);
    const float* lp[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) lp[t] = opaque_ptr(P + lcol[t]);
    // this lane's first two panel rows, cached
    const int ra = rbeg + lane, rb = rbeg + lane + 32;
    int qa0 = 0, qa1 = 0, qb0 = 0, qb1 = 0;
    float pla = 0.0f, plb = 0.0f;
    if (ra < rend) {
      qa0 = v.lrp[ra] - kbeg;
      qa1 = v.lrp[ra + 1] - kbeg;
      if (part) pla = pl[ra];
    }
    if (rb < rend) {
      qb0 = v.lrp[rb] - kbeg;
      qb1 = v.lrp[rb + 1] - kbeg;
      if (part) plb = pl[rb];
    }
    const int i0 = c * v.rpc, i1 = min(n, i0 + v.rpc);
    for (int i = i0; i < i1; i += 2) {
      const bool two = i + 1 < i1;
      float acc0[NS], acc1[NS], pc0[NS], pc1[NS];
#pragma unroll
      for (int t = 0; t < NS; ++t) {
        acc0[t] = acc1[t] = 0.0f;
        pc0[t] = pc1[t] = 0.0f;
        if constexpr (LAP) {
          pc0[t] = P[i * m + lrw[t]];
          if (two) pc1[t] = P[(i + 1) * m + lrw[t]];
        }
      }
      // the epilogue's streamed diagonal of the lane's first panel row, loaded before the accumulation
      // so its HBM latency overlaps the gathers
      float dga0 = 0.0f, dga1 = 0.0f;
#if MGK_PANEL_DGPF
      if (ra < rend) {
        dga0 = ld_stream(DG + i * m + ra);
        if (two) dga1 = ld_stream(DG + (i + 1) * m + ra);
      }
#endif
      row_accumulate<NS, EK, LAP>(ek, v.ue, v.urp[i], v.urp[i + 1], lp, m, llab, acc0, pc0);
      if (two) row_accumulate<NS, EK, LAP>(ek, v.ue, v.urp[i + 1], v.urp[i + 2], lp, m, llab, acc1, pc1);
#pragma unroll
      for (int t = 0; t < NS; ++t) {
        SEG[lane + 32 * t] = acc0[t] * lw[t];
        SEG[kPanelCap + lane + 32 * t] = acc1[t] * lw[t];
      }
      __syncwarp();
      const int base = i * m;
      float pu0 = 0.0f, pu1 = 0.0f;
      if (part) {
        pu0 = pu[i];
        pu1 = two ? pu[i + 1] : 0.0f;
      }
      for (int r = ra; r < rend; r += 32) {
        int q0, q1;
        float plr;
        if (r == ra) {
          q0 = qa0;
          q1 = qa1;
          plr = pla;
        } else if (r == rb) {
          q0 = qb0;
          q1 = qb1;
          plr = plb;
        } else {
          q0 = v.lrp[r] - kbeg;
          q1 = v.lrp[r + 1] - kbeg;
          plr = part ? pl[r] : 0.0f;
        }
        float s0 = 0.0f, s1 = 0.0f;
        for (int q = q0; q < q1; ++q) {
          s0 += SEG[q];
          s1 += SEG[kPanelCap + q];
        }
        const int e0 = base + r;
        const float p0 = P[e0];
        const bool pf = MGK_PANEL_DGPF && r == ra;
        const float a0 = fmaf(pf ? dga0 : ld_stream(DG + e0), p0, -s0);
        AP[e0] = a0;
        if (part) {
          pap += (double)p0 * (double)a0;
          pxp += (double)(pu0 * plr) * (double)p0;
        }
        if (two) {
          const float p1 = P[e0 + m];
          const float a1 = fmaf(pf ? dga1 : ld_stream(DG + e0 + m), p1, -s1);
          AP[e0 + m] = a1;
          if (part) {
            pap += (double)p1 * (double)a1;
            pxp += (double)(pu1 * plr) * (double)p1;
          }
        }
      }
      __syncwarp();
    }
  }
  if (part) {
    part->x += pap;
    part->y += pxp;
  }
}

// Single-panel labeled XMV over undirected L slots: slot t = L edge {l, c}; one edge-kernel evaluation
// feeds both directed entries (gathers P[j][c] -> lands on row l, P[j][l] -> lands on row c), the slot
// products go to both directed positions of the segment buffer, and the L-row segment sums are as in
// xmv_panels (same per-entry accumulation order: results identical to the directed slots).
template <int NSU, int EK>
__device__ void xmv_panels_sym(const KernelDesc& ek, const PairView& v, const float* P, float* AP, const float* DG,
                               float* SEG, int lane, int64_t w0, int64_t wstride, const float* pu, const float* pl,
                               double2* part) {
  const int n = v.n, m = v.m;
  const int nchunks = (n + v.rpc - 1) / v.rpc;
  int lca[NSU], lcb[NSU], lkab[NSU];
  float lw[NSU], llab[NSU];
#pragma unroll
  for (int t = 0; t < NSU; ++t) {
    const int u = lane + 32 * t;
    lca[t] = lcb[t] = lkab[t] = 0;
    lw[t] = llab[t] = 0.0f;
    if (u < v.nund) {
      const int2 kk = v.lsym[u];
      const float4 e = v.le[kk.x];
      lca[t] = __float_as_int(e.x);           // l -> c gathers P[j][c]
      lcb[t] = __float_as_int(v.le[kk.y].x);  // c -> l gathers P[j][l]
      lw[t] = e.y;
      llab[t] = e.z;
      lkab[t] = kk.x | (kk.y << 16);
    }
  }
  const float* lpa[NSU];
  const float* lpb[NSU];
#pragma unroll
  for (int t = 0; t < NSU; ++t) {
    lpa[t] = opaque_ptr(P + lca[t]);
    lpb[t] = opaque_ptr(P + lcb[t]);
  }
  const int ra = lane, rb = lane + 32;
  int qa0 = 0, qa1 = 0, qb0 = 0, qb1 = 0;
  float pla = 0.0f, plb = 0.0f;
  if (ra < m) {
    qa0 = v.lrp[ra];
    qa1 = v.lrp[ra + 1];
    if (part) pla = pl[ra];
  }
  if (rb < m) {
    qb0 = v.lrp[rb];
    qb1 = v.lrp[rb + 1];
    if (part) plb = pl[rb];
  }
  double pap = 0.0, pxp = 0.0;
  for (int64_t c = w0; c < nchunks; c += wstride) {
    const int i0 = (int)c * v.rpc, i1 = min(n, i0 + v.rpc);
    for (int i = i0; i < i1; i += 2) {
      const bool two = i + 1 < i1;
      float a[2][NSU], b[2][NSU];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
#pragma unroll
        for (int t = 0; t < NSU; ++t) a[r][t] = b[r][t] = 0.0f;
        if (r == 1 && !two) break;
        const int k1 = v.urp[i + r + 1];
        int k = v.urp[i + r];
        for (; k + 1 < k1; k += 2) {
          const float4 e0 = v.ue[k], e1 = v.ue[k + 1];
          const unsigned o0 = (unsigned)(__float_as_int(e0.x) * m), o1 = (unsigned)(__float_as_int(e1.x) * m);
#pragma unroll
          for (int t = 0; t < NSU; ++t) {
            const float x0a = lpa[t][o0], x0b = lpb[t][o0], x1a = lpa[t][o1], x1b = lpb[t][o1];
            const float c0 = edge_kappa_w<EK>(ek, e0.z, llab[t], EK == KK_SE ? e0.w : e0.y);
            const float c1 = edge_kappa_w<EK>(ek, e1.z, llab[t], EK == KK_SE ? e1.w : e1.y);
            a[r][t] = fmaf(c0, x0a, a[r][t]);
            b[r][t] = fmaf(c0, x0b, b[r][t]);
            a[r][t] = fmaf(c1, x1a, a[r][t]);
            b[r][t] = fmaf(c1, x1b, b[r][t]);
          }
        }
        if (k < k1) {
          const float4 e0 = v.ue[k];
          const unsigned o0 = (unsigned)(__float_as_int(e0.x) * m);
#pragma unroll
          for (int t = 0; t < NSU; ++t) {
            const float c0 = edge_kappa_w<EK>(ek, e0.z, llab[t], EK == KK_SE ? e0.w : e0.y);
            a[r][t] = fmaf(c0, lpa[t][o0], a[r][t]);
            b[r][t] = fmaf(c0, lpb[t][o0], b[r][t]);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < NSU; ++t) {
        if (lane + 32 * t < v.nund) {
          const int ka = lkab[t] & 0xffff, kb = lkab[t] >> 16;
          SEG[ka] = a[0][t] * lw[t];
          SEG[kb] = b[0][t] * lw[t];
          SEG[kPanelCap + ka] = a[1][t] * lw[t];
          SEG[kPanelCap + kb] = b[1][t] * lw[t];
        }
      }
      __syncwarp();
      const int base = i * m;
      float pu0 = 0.0f, pu1 = 0.0f;
      if (part) {
        pu0 = pu[i];
        pu1 = two ? pu[i + 1] : 0.0f;
      }
      for (int r = ra; r < m; r += 32) {
        int q0, q1;
        float plr;
        if (r == ra) {
          q0 = qa0;
          q1 = qa1;
          plr = pla;
        } else if (r == rb) {
          q0 = qb0;
          q1 = qb1;
          plr = plb;
        } else {
          q0 = v.lrp[r];
          q1 = v.lrp[r + 1];
          plr = part ? pl[r] : 0.0f;
        }
        float s0 = 0.0f, s1 = 0.0f;
        for (int q = q0; q < q1; ++q) {
          s0 += SEG[q];
          s1 += SEG[kPanelCap + q];
        }
        const int e0 = base + r;
        const float p0 = P[e0];
        const float a0 = fmaf(ld_stream(DG + e0), p0, -s0);
        AP[e0] = a0;
        if (part) {
          pap += (double)p0 * (double)a0;
          pxp += (double)(pu0 * plr) * (double)p0;
        }
        if (two) {
          const float p1 = P[e0 + m];
          const float a1 = fmaf(ld_stream(DG + e0 + m), p1, -s1);
          AP[e0 + m] = a1;
          if (part) {
            pap += (double)p1 * (double)a1;
            pxp += (double)(pu1 * plr) * (double)p1;
          }
        }
      }
      __syncwarp();
    }
  }
  if (part) {
    part->x += pap;
    part->y += pxp;
  }
}

template <int EK>
__device__ __forceinline__ void xmv_dispatch(int ns, const KernelDesc& ek, const PairView& v, const float* P,
                                             float* AP, const float* DG, float* SEG, int lane, int64_t w0,
                                             int64_t wstride, const float* pu, const float* pl, double2* part,
                                             bool lap) {
  if constexpr (EK != KK_NONE) {
    if (!v.prow && v.nund > 0) {  // single panel (S_L <= 128): undirected slots, one kappa per L edge
      if (v.nund <= 32)
        xmv_panels_sym<1, EK>(ek, v, P, AP, DG, SEG, lane, w0, wstride, pu, pl, part);
      else
        xmv_panels_sym<2, EK>(ek, v, P, AP, DG, SEG, lane, w0, wstride, pu, pl, part);
      return;
    }
  }
  if constexpr (EK == KK_NONE) {
    if (lap) {
      switch (ns) {
        case 2: xmv_panels<2, EK, true>(ek, v, P, AP, DG, SEG, lane, w0, wstride, pu, pl, part); break;
        case 4: xmv_panels<4, EK, true>(ek, v, P, AP, DG, SEG, lane, w0, wstride, pu, pl, part); break;
        default: xmv_panels<kPanelSlots, EK, true>(ek, v, P, AP, DG, SEG, lane, w0, wstride, pu, pl, part); break;
      }
      return;
    }
  }
  switch (ns) {
    case 2: xmv_panels<2, EK>(ek, v, P, AP, DG, SEG, lane, w0, wstride, pu, pl, part); break;
    case 4: xmv_panels<4, EK>(ek, v, P, AP, DG, SEG, lane, w0, wstride, pu, pl, part); break;
    default: xmv_panels<kPanelSlots, EK>(ek, v, P, AP, DG, SEG, lane, w0, wstride, pu, pl, part); break;
  }
}

// Unlabeled pairs (kappa_e = 1): the off-diagonal block is A (x) B, so
// XMV(P) = A P B^T (the factorisation of the reference's unlabeled dense x dense
// micro-kernel, product.py:94) at n S_L + S_U m work instead of S_U S_L:
//   phase T:  T[j][r] = sum_{t in L(r)} w'_t P[j][col(t)]  (warp items over P rows x L panels,
//             the panel's slots in registers, segment sums as in xmv_panels)
//   phase AP: AP[i][r] = diag P - sum_{k in U(i)} w_k T[j_k][r]  (thread per element, coalesced over r)
// The caller places a block / grid barrier between the phases.
// LAP: T[j][r] = sum_{t in L(r)} w'_t (P[j][col(t)] - P[j][r])  (Laplacian splitting, see factored_AP)
template <int NS, bool LAP>
__device__ void factored_T(const PairView& v, const float* P, float* T, float* SEG, int lane, int64_t w0,
                           int64_t wstride) {
  const int n = v.n, m = v.m;
  const int nchunks = (n + v.rpc - 1) / v.rpc;
  const int64_t items = (int64_t)v.np * nchunks;
  for (int64_t item = w0; item < items; item += wstride) {
    int p, c;
    item_coords(item, v.np, nchunks, p, c);
    const int rbeg = v.prow ? v.prow[p] : 0;
    const int rend = v.prow ? v.prow[p + 1] : m;
    const int kbeg = v.lrp[rbeg], kend = v.lrp[rend];
    int lcol[NS];
    float lw[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const int k = kbeg + lane + 32 * t;
      lcol[t] = 0;
      lw[t] = 0.0f;
      if (k < kend) {
        const float4 e = v.le[k];
        lcol[t] = __float_as_int(e.x);
        lw[t] = e.y;
      }
    }
    int lrw[NS];
    if constexpr (LAP) slot_rows<NS>(v.lrp, rbeg, rend, kbeg, kend, lane, lrw);
    const int j0 = c * v.rpc, j1 = min(n, j0 + v.rpc);
    for (int j = j0; j < j1; j += 2) {
      const bool two = j + 1 < j1;
      const float* r0 = P + j * m;
      const float* r1 = two ? r0 + m : r0;
#pragma unroll
      for (int t = 0; t < NS; ++t) {
        float x0 = r0[lcol[t]], x1 = r1[lcol[t]];
        if constexpr (LAP) {
          x0 -= r0[lrw[t]];
          x1 -= r1[lrw[t]];
        }
        SEG[lane + 32 * t] = lw[t] * x0;
        SEG[kPanelCap + lane + 32 * t] = lw[t] * x1;
      }
      __syncwarp();
      for (int r = rbeg + lane; r < rend; r += 32) {
        const int q0 = v.lrp[r] - kbeg, q1 = v.lrp[r + 1] - kbeg;
        float s0 = 0.0f, s1 = 0.0f;
        for (int q = q0; q < q1; ++q) {
          s0 += SEG[q];
          s1 += SEG[kPanelCap + q];
        }
        T[j * m + r] = s0;
        if (two) T[(j + 1) * m + r] = s1;
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ void factored_T_dispatch(int ns, const PairView& v, const float* P, float* T, float* SEG,
                                                    int lane, int64_t w0, int64_t wstride, bool lap) {
  if (lap) {
    switch (ns) {
      case 2: factored_T<2, true>(v, P, T, SEG, lane, w0, wstride); break;
      case 4: factored_T<4, true>(v, P, T, SEG, lane, w0, wstride); break;
      default: factored_T<kPanelSlots, true>(v, P, T, SEG, lane, w0, wstride); break;
    }
    return;
  }
  switch (ns) {
    case 2: factored_T<2, false>(v, P, T, SEG, lane, w0, wstride); break;
    case 4: factored_T<4, false>(v, P, T, SEG, lane, w0, wstride); break;
    default: factored_T<kPanelSlots, false>(v, P, T, SEG, lane, w0, wstride); break;
  }
}

// AP = diag P - A T over elements e0, e0 + estride, ...; accumulates (p.Ap, px.p) when part != nullptr.
// Laplacian splitting (ldm != nullptr, DG = s): AP = s P - (A T + b (x) sum_j A_ij (P[j][l] - P[i][l]))
// with T from factored_T<LAP> and b = ldm = d' - q' of the L nodes.
__device__ void factored_AP(const PairView& v, const float* P, const float* T, float* AP, const float* DG,
                            int64_t e0, int64_t estride, const float* pu, const float* pl, double2* part,
                            const float* ldm) {
  const int m = v.m;
  const int64_t nm = (int64_t)v.n * m;
  const int64_t di = estride / m, dl = estride % m;
  int64_t i = e0 / m, l = e0 % m;
  double pap = 0.0, pxp = 0.0;
  for (int64_t e = e0; e < nm; e += estride) {
    float acc = 0.0f;
    if (ldm) {
      const float pi = P[e];
      float acc2 = 0.0f;
      for (int k = v.urp[i]; k < v.urp[i + 1]; ++k) {
        const float4 u = v.ue[k];
        const int64_t f = (int64_t)__float_as_int(u.x) * m + l;
        acc = fmaf(u.y, T[f], acc);
        acc2 = fmaf(u.y, P[f] - pi, acc2);
      }
      acc = fmaf(ldm[l], acc2, acc);
    } else {
      for (int k = v.urp[i]; k < v.urp[i + 1]; ++k) {
        const float4 u = v.ue[k];
        acc = fmaf(u.y, T[(int64_t)__float_as_int(u.x) * m + l], acc);
      }
    }
    const float p = P[e];
    const float ap = fmaf(ld_stream(DG + e), p, -acc);
    AP[e] = ap;
    if (part) {
      pap += (double)p * (double)ap;
      pxp += (double)(pu[i] * pl[l]) * (double)p;
    }
    l += dl;
    i += di;
    if (l >= m) {
      l -= m;
      ++i;
    }
  }
  if (part) {
    part->x += pap;
    part->y += pxp;
  }
}

// Lane-side cost of a graph (slot-rounded nonzeros a warp streams per U nonzero).
__device__ __forceinline__ int64_t lane_cost(const GraphDesc& g) {
  const int S = 2 * g.ne;
  if (S <= 64) return 64;
  if (S <= 128) return 128;
  if (g.npanels <= 0) return (int64_t)1 << 40;
  return (int64_t)g.npanels * kPanelCap;
}

template <int EK, bool NODEWISE>
__global__ void __launch_bounds__(kPT, 512 / kPT)
k_pcg_panel(DatasetDev ds, KernelDesc vk, KernelDesc ek, PairJob job, SolveParams prm, SolveOut out,
            unsigned long long* queue, float* scratch, int64_t slab, int smem_vec) {
  extern __shared__ __align__(16) float psm[];
  __shared__ double2 red[2][kPW];
  __shared__ unsigned long long sh_pid;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* SEG = psm + warp * kSegFloats;
  float4* c_ue = reinterpret_cast<float4*>(psm + kPW * kSegFloats);
  float4* c_le = c_ue + kCacheU;
  int32_t* c_urp = reinterpret_cast<int32_t*>(c_le + kPanelCap);
  int32_t* c_lrp = c_urp + kCacheRows + 1;
  float* svec = psm + kPW * kSegFloats + kCacheFloats;
  const bool vlab = (vk.kind != KK_CONST1 && vk.kind != KK_NONE && ds.nl_kind != LK_NONE);
  const int64_t vstride = slab / kSlabVectors;

  for (;;) {
    if (threadIdx.x == 0) sh_pid = atomicAdd(queue, 1ull);
    __syncthreads();
    const unsigned long long pid = sh_pid;
    if (pid >= (unsigned long long)job.npairs) break;
    int32_t ga, gb;
    decode_pair(job, (int64_t)pid, ga, gb);
    const GraphDesc A = ds.graphs[ga], B = ds.graphs[gb];
    // orientation: L is the graph with the cheaper lane side (fewest streamed slots)
    const int64_t costAB = (int64_t)(2 * A.ne) * lane_cost(B) + A.n;
    const int64_t costBA = (int64_t)(2 * B.ne) * lane_cost(A) + B.n;
    const bool swap = costBA < costAB;
    const GraphDesc U = swap ? B : A;
    const GraphDesc L = swap ? A : B;
    const int n = U.n, m = L.n, nm = n * m;
    const int SL = 2 * L.ne;
    const int ns = SL <= 64 ? 2 : (SL <= 128 ? 4 : kPanelSlots);
    const bool lap = EK == KK_NONE && laplacian_pair(prm, U, L);

    PairView v;
    v.urp = ds.rowptr + U.rowptr_off;
    v.ue = ds.rowent + U.nz_off;
    v.lrp = ds.rowptr + L.rowptr_off;
    v.le = ds.rowent + L.nz_off;
    v.prow = SL > 128 ? ds.panel_row + L.panel_off : nullptr;
    v.lsym = ds.symk + L.edge_off;
    v.nund = L.ne;
    v.n = n;
    v.m = m;
    v.np = SL > 128 ? L.npanels : 1;
    {
      int rpc = (n * v.np) / (4 * kPW);
      rpc = rpc < 2 ? 2 : (rpc > kPanelRpcMax ? kPanelRpcMax : rpc);
      if (prm.panel_rpc > 0) rpc = prm.panel_rpc;
      v.rpc = (rpc + 1) & ~1;
    }
    // stage the row expansions in shared memory when they fit (the previous pair is done with them:
    // the pair loop ends on a barrier)
    {
      const int SU = 2 * U.ne;
      const bool cu = SU <= kCacheU && n < kCacheRows;
      const bool cl = v.np == 1 && SL <= kPanelCap && m < kCacheRows;
      if (cu) {
        for (int k = threadIdx.x; k < SU; k += kPT) c_ue[k] = v.ue[k];
        for (int r = threadIdx.x; r <= n; r += kPT) c_urp[r] = v.urp[r];
      }
      if (cl) {
        for (int k = threadIdx.x; k < SL; k += kPT) c_le[k] = v.le[k];
        for (int r = threadIdx.x; r <= m; r += kPT) c_lrp[r] = v.lrp[r];
      }
      __syncthreads();
      if (cu) {
        v.ue = c_ue;
        v.urp = c_urp;
      }
      if (cl) {
        v.le = c_le;
        v.lrp = c_lrp;
      }
    }

    float* base = scratch + (int64_t)blockIdx.x * slab;
    float* R = base;
    float* DG = base + vstride;
    float* X = base + 2 * vstride;
    float* P = base + 3 * vstride;
    float* AP = base + 4 * vstride;
    float* T = base + 5 * vstride;  // unlabeled: P B^T
    float* SD = base + 6 * vstride;  // Laplacian splitting: s = diag - rowsum(L)
    if (2 * nm <= smem_vec) {
      P = svec;
      AP = svec + nm;
    }
    const int di = kPT / m, dl = kPT % m;

    // ---- setup (solver.py:69-74, 91-97): diag, b, x = 0, r = b, z = r / diag, p = z
    double2 acc = make_double2(0.0, 0.0);
    for (int i = threadIdx.x; i < n; i += kPT) {
      const double dq = ds.deg[U.node_off + i] * ds.q64[U.node_off + i];
      acc.x += dq * dq;
    }
    for (int i = threadIdx.x; i < m; i += kPT) {
      const double dq = ds.deg[L.node_off + i] * ds.q64[L.node_off + i];
      acc.y += dq * dq;
    }
    int flip = 0;
    double2 s = block_sum2(acc, red[flip]);
    flip ^= 1;
    const double eps = prm.tol2 * s.x * s.y;
    acc = make_double2(0.0, 0.0);
    {
      int i = threadIdx.x / m, l = threadIdx.x % m;
      for (int e = threadIdx.x; e < nm; e += kPT) {
        const int64_t vu = U.node_off + i, vl = L.node_off + l;
        float kv = 1.0f;
        if (vlab)
          kv = floor_kv(kernel_vec(vk, ds.vlabel + vu * ds.nl_dim, ds.vlabel + vl * ds.nl_dim, ds.nl_dim,
                                   ds.nl_kind == LK_CAT), prm, out);
        const double dg64 = ds.deg[vu] * ds.deg[vl] / (double)kv;
        const float dg = (float)dg64;
        const float b = (float)((ds.deg[vu] * ds.q64[vu]) * (ds.deg[vl] * ds.q64[vl]));
        const float z = b * rcp_approx(dg);
        if (lap) SD[e] = (float)(dg64 - (ds.deg[vu] - ds.q64[vu]) * (ds.deg[vl] - ds.q64[vl]));
        DG[e] = dg;
        R[e] = b;
        P[e] = z;
        if constexpr (NODEWISE) X[e] = 0.0f;
        acc.x += (double)b * (double)z;
        acc.y += (double)b * (double)b;
        l += dl;
        i += di;
        if (l >= m) {
          l -= m;
          ++i;
        }
      }
    }
    s = block_sum2(acc, red[flip]);
    flip ^= 1;
    double rho = s.x, rr = s.y;
    bool conv = rr < eps;
    const int64_t max_iter = prm.max_iter > 0 ? prm.max_iter : 10ll * nm;
    int64_t it = 0;
    double value = 0.0;
    const bool self_pair = (ga == gb);
    // unlabeled: factorise when it saves work beyond its extra pass (not for degree-4 sparsity)
    const bool factor = (int64_t)(2 * U.ne) * SL * 4 > prm.factor_ratio4 * ((int64_t)n * SL + (int64_t)(2 * U.ne) * m);
    __syncthreads();

    while (!conv && it < max_iter) {
      double2 part = make_double2(0.0, 0.0);
      if (EK == KK_NONE && factor) {
        factored_T_dispatch(ns, v, P, T, SEG, lane, warp, kPW, lap);
        __syncthreads();
        factored_AP(v, P, T, AP, lap ? SD : DG, threadIdx.x, kPT, ds.p + U.node_off, ds.p + L.node_off,
                    self_pair ? nullptr : &part, lap ? ds.dm + L.node_off : nullptr);
      } else {
        xmv_dispatch<EK>(ns, ek, v, P, AP, lap ? SD : DG, SEG, lane, warp, kPW, ds.p + U.node_off,
                         ds.p + L.node_off, self_pair ? nullptr : &part, lap);
      }
      __syncthreads();
      if (self_pair) {
        // self pair: keep the iterate exactly symmetric (see pcg_warp.cu)
        for (int e = threadIdx.x; e < nm; e += kPT) {
          const int i = e / m, l = e - i * m;
          if (i < l) {
            const int f = l * m + i;
            const float a = AP[e], b = AP[f];
            const float sym = 0.5f * (a + b);
            AP[e] = sym;
            AP[f] = sym;
          }
        }
        __syncthreads();
        // pass 1: p.Ap and px.p (value = sum_k alpha_k px.p_k)
        int i = threadIdx.x / m, l = threadIdx.x % m;
        for (int e = threadIdx.x; e < nm; e += kPT) {
          const float p = P[e];
          part.x += (double)p * (double)AP[e];
          part.y += (double)(ds.p[U.node_off + i] * ds.p[L.node_off + l]) * (double)p;
          l += dl;
          i += di;
          if (l >= m) {
            l -= m;
            ++i;
          }
        }
      }
      ++it;
      // lanes of a warp hold partial sums: fold them into the block reduction
      s = block_sum2(part, red[flip]);
      flip ^= 1;
      const double alpha = rho / s.x;
      value += alpha * s.y;
      const float af = (float)alpha;
      // pass 2: x += alpha p, r -= alpha Ap, z = r / diag (stored over Ap)
      acc = pcg_pass2<NODEWISE, int>((int)threadIdx.x, kPT, nm, af, P, AP, R, DG, X);
      s = block_sum2(acc, red[flip]);
      flip ^= 1;
      rr = s.x;
      const double rho_next = s.y;
      if (rr < eps) {
        conv = true;
        break;
      }
      const float beta = (float)(rho_next / rho);
      pcg_update_p<int>((int)threadIdx.x, kPT, nm, beta, P, AP);
      rho = rho_next;
      __syncthreads();
    }

    if constexpr (NODEWISE) {
      if (out.nodewise) {
        float* nw = out.nodewise + out.nodewise_off[pid];
        int i = threadIdx.x / m, l = threadIdx.x % m;
        for (int e = threadIdx.x; e < nm; e += kPT) {
          nw[swap ? l * n + i : e] = X[e];
          l += dl;
          i += di;
          if (l >= m) {
            l -= m;
            ++i;
          }
        }
      }
    }
    if (threadIdx.x == 0) {
      if (out.value) out.value[pid] = value;
      if (out.iters) out.iters[pid] = (int32_t)it;
      if (out.conv) out.conv[pid] = conv ? 1 : 0;
      if (out.residual) out.residual[pid] = (float)sqrt(rr);
      if (out.pair_a) out.pair_a[pid] = ga;
      if (out.pair_b) out.pair_b[pid] = gb;
      const double kval = conv ? value : __longlong_as_double(0x7ff8000000000000ll);
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
    __syncthreads();
  }
}

template <int EK, bool NODEWISE>
static cudaError_t launch_panel_ek(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek,
                                   const PairJob& job, const SolveParams& prm, const SolveOut& out,
                                   unsigned long long* queue, float* scratch, int64_t slab, int nctas, int smem_vec,
                                   cudaStream_t stream) {
  auto kern = k_pcg_panel<EK, NODEWISE>;
  const size_t smem = kPanelStaticSmem + (size_t)smem_vec * 4;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<nctas, kPT, smem, stream>>>(ds, vk, ek, job, prm, out, queue, scratch, slab, smem_vec);
  return cudaGetLastError();
}

int panel_ctas_per_sm(int smem_vec) {
  int per_sm = 0;
  const size_t smem = kPanelStaticSmem + (size_t)smem_vec * 4;
  cudaFuncSetAttribute(k_pcg_panel<KK_SE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_panel<KK_SE, false>, kPT, smem) != cudaSuccess)
    return 1;
  return per_sm < 1 ? 1 : per_sm;
}

template <bool NODEWISE>
static cudaError_t launch_panel_nw(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek,
                                   const PairJob& job, const SolveParams& prm, const SolveOut& out,
                                   unsigned long long* queue, float* scratch, int64_t slab, int nctas, int smem_vec,
                                   cudaStream_t stream) {
  int kind = prm.labeled ? ek.kind : KK_NONE;
  if (kind == KK_CONST1) kind = KK_NONE;
  switch (kind) {
    case KK_SE:
      return launch_panel_ek<KK_SE, NODEWISE>(ds, vk, ek, job, prm, out, queue, scratch, slab, nctas, smem_vec, stream);
    case KK_DELTA:
      return launch_panel_ek<KK_DELTA, NODEWISE>(ds, vk, ek, job, prm, out, queue, scratch, slab, nctas, smem_vec,
                                                 stream);
    case KK_POLY:
      return launch_panel_ek<KK_POLY, NODEWISE>(ds, vk, ek, job, prm, out, queue, scratch, slab, nctas, smem_vec,
                                                stream);
    default:
      return launch_panel_ek<KK_NONE, NODEWISE>(ds, vk, ek, job, prm, out, queue, scratch, slab, nctas, smem_vec,
                                                stream);
  }
}

cudaError_t launch_pcg_panel(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                             const SolveParams& prm, const SolveOut& out, unsigned long long* queue, float* scratch,
                             int64_t slab, int nctas, int smem_vec, cudaStream_t stream) {
  if ((int64_t)nctas > job.npairs) nctas = (int)job.npairs;
  if (nctas < 1) return cudaSuccess;
  if (out.nodewise)
    return launch_panel_nw<true>(ds, vk, ek, job, prm, out, queue, scratch, slab, nctas, smem_vec, stream);
  return launch_panel_nw<false>(ds, vk, ek, job, prm, out, queue, scratch, slab, nctas, smem_vec, stream);
}

// ---------------------------------------------------------------------------
// Grid class: one pair at a time on the whole GPU (cooperative launch), for
// product systems too large for one SM (config 4: n up to 5000, n m up to
// 2.5e7).  Same XMV items, strided over every warp of the grid; the PCG dot
// products are grid reductions (per-block partials summed in block order by
// every block after a grid barrier, so all blocks agree bit for bit).
// ---------------------------------------------------------------------------
__device__ double2 grid_sum2(double2 v, double2* gbuf, double2* wred, double2* sres, cg::grid_group& grid) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  if (lane == 0) wred[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 b = make_double2(0.0, 0.0);
    for (int k = 0; k < kPW; ++k) {
      b.x += wred[k].x;
      b.y += wred[k].y;
    }
    gbuf[blockIdx.x] = b;
  }
  grid.sync();
  if (w == 0) {
    double2 t = make_double2(0.0, 0.0);
    for (int b = lane; b < (int)gridDim.x; b += 32) {
      const double2 x = gbuf[b];
      t.x += x.x;
      t.y += x.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
      t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
    }
    if (lane == 0) *sres = t;
  }
  __syncthreads();
  return *sres;
}

template <int EK, bool NODEWISE>
__global__ void __launch_bounds__(kPT, 512 / kPT)
k_pcg_grid(DatasetDev ds, KernelDesc vk, KernelDesc ek, PairJob job, SolveParams prm, SolveOut out, float* vec,
           int64_t vstride, double2* gbuf) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) float psm[];
  __shared__ double2 wred[kPW];
  __shared__ double2 sres;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* SEG = psm + warp * kSegFloats;
  const bool vlab = (vk.kind != KK_CONST1 && vk.kind != KK_NONE && ds.nl_kind != LK_NONE);
  const int64_t gtid = (int64_t)blockIdx.x * kPT + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * kPT;
  const int64_t gw = gtid >> 5, GW = gthreads >> 5;
  float* R = vec;
  float* DG = vec + vstride;
  float* X = vec + 2 * vstride;
  float* P = vec + 3 * vstride;
  float* AP = vec + 4 * vstride;
  float* T = vec + 5 * vstride;  // unlabeled: P B^T
  float* SD = vec + 6 * vstride;  // Laplacian splitting: s = diag - rowsum(L)
  int flip = 0;
  auto gsum = [&](double2 v) {
    double2 r = grid_sum2(v, gbuf + flip * gridDim.x, wred, &sres, grid);
    flip ^= 1;
    return r;
  };

  for (int64_t pid = 0; pid < job.npairs; ++pid) {
    int32_t ga, gb;
    decode_pair(job, pid, ga, gb);
    const GraphDesc A = ds.graphs[ga], B = ds.graphs[gb];
    const int64_t costAB = (int64_t)(2 * A.ne) * lane_cost(B) + A.n;
    const int64_t costBA = (int64_t)(2 * B.ne) * lane_cost(A) + B.n;
    const bool swap = costBA < costAB;
    const GraphDesc U = swap ? B : A;
    const GraphDesc L = swap ? A : B;
    const int n = U.n, m = L.n, nm = n * m;
    const int SL = 2 * L.ne;
    const int ns = SL <= 64 ? 2 : (SL <= 128 ? 4 : kPanelSlots);
    const bool lap = EK == KK_NONE && laplacian_pair(prm, U, L);
    PairView v;
    v.urp = ds.rowptr + U.rowptr_off;
    v.ue = ds.rowent + U.nz_off;
    v.lrp = ds.rowptr + L.rowptr_off;
    v.le = ds.rowent + L.nz_off;
    v.prow = SL > 128 ? ds.panel_row + L.panel_off : nullptr;
    v.lsym = ds.symk + L.edge_off;
    v.nund = L.ne;
    v.n = n;
    v.m = m;
    v.np = SL > 128 ? L.npanels : 1;
    v.rpc = prm.panel_rpc > 0 ? ((prm.panel_rpc + 1) & ~1) : 8;
    const int64_t di = gthreads / m, dl = gthreads % m;

    double2 acc = make_double2(0.0, 0.0);
    for (int64_t i = gtid; i < n; i += gthreads) {
      const double dq = ds.deg[U.node_off + i] * ds.q64[U.node_off + i];
      acc.x += dq * dq;
    }
    for (int64_t i = gtid; i < m; i += gthreads) {
      const double dq = ds.deg[L.node_off + i] * ds.q64[L.node_off + i];
      acc.y += dq * dq;
    }
    double2 s = gsum(acc);
    const double eps = prm.tol2 * s.x * s.y;
    acc = make_double2(0.0, 0.0);
    {
      int64_t i = gtid / m, l = gtid % m;
      for (int64_t e = gtid; e < nm; e += gthreads) {
        const int64_t vu = U.node_off + i, vl = L.node_off + l;
        float kv = 1.0f;
        if (vlab)
          kv = floor_kv(kernel_vec(vk, ds.vlabel + vu * ds.nl_dim, ds.vlabel + vl * ds.nl_dim, ds.nl_dim,
                                   ds.nl_kind == LK_CAT), prm, out);
        const double dg64 = ds.deg[vu] * ds.deg[vl] / (double)kv;
        const float dg = (float)dg64;
        const float b = (float)((ds.deg[vu] * ds.q64[vu]) * (ds.deg[vl] * ds.q64[vl]));
        const float z = b * rcp_approx(dg);
        if (lap) SD[e] = (float)(dg64 - (ds.deg[vu] - ds.q64[vu]) * (ds.deg[vl] - ds.q64[vl]));
        DG[e] = dg;
        R[e] = b;
        P[e] = z;
        if constexpr (NODEWISE) X[e] = 0.0f;
        acc.x += (double)b * (double)z;
        acc.y += (double)b * (double)b;
        l += dl;
        i += di;
        if (l >= m) {
          l -= m;
          ++i;
        }
      }
    }
    s = gsum(acc);
    double rho = s.x, rr = s.y;
    bool conv = rr < eps;
    const int64_t max_iter = prm.max_iter > 0 ? prm.max_iter : 10ll * nm;
    int64_t it = 0;
    double value = 0.0;
    const bool self_pair = (ga == gb);
    const bool factor = (int64_t)(2 * U.ne) * SL * 4 > prm.factor_ratio4 * ((int64_t)n * SL + (int64_t)(2 * U.ne) * m);

    while (!conv && it < max_iter) {
      double2 part = make_double2(0.0, 0.0);
      if (EK == KK_NONE && factor) {
        factored_T_dispatch(ns, v, P, T, SEG, lane, gw, GW, lap);
        grid.sync();
        factored_AP(v, P, T, AP, lap ? SD : DG, gtid, gthreads, ds.p + U.node_off, ds.p + L.node_off,
                    self_pair ? nullptr : &part, lap ? ds.dm + L.node_off : nullptr);
      } else {
        xmv_dispatch<EK>(ns, ek, v, P, AP, lap ? SD : DG, SEG, lane, gw, GW, ds.p + U.node_off,
                         ds.p + L.node_off, self_pair ? nullptr : &part, lap);
      }
      if (self_pair) {
        grid.sync();
        for (int64_t e = gtid; e < nm; e += gthreads) {
          const int i = (int)(e / m), l = (int)(e - (int64_t)i * m);
          if (i < l) {
            const int f = l * m + i;
            const float a = AP[e], b = AP[f];
            const float sym = 0.5f * (a + b);
            AP[e] = sym;
            AP[f] = sym;
          }
        }
        grid.sync();
        int64_t i = gtid / m, l = gtid % m;
        for (int64_t e = gtid; e < nm; e += gthreads) {
          const float p = P[e];
          part.x += (double)p * (double)AP[e];
          part.y += (double)(ds.p[U.node_off + i] * ds.p[L.node_off + l]) * (double)p;
          l += dl;
          i += di;
          if (l >= m) {
            l -= m;
            ++i;
          }
        }
      }
      ++it;
      s = gsum(part);
      const double alpha = rho / s.x;
      value += alpha * s.y;
      const float af = (float)alpha;
      acc = pcg_pass2<NODEWISE, int64_t>(gtid, gthreads, (int64_t)nm, af, P, AP, R, DG, X);
      s = gsum(acc);
      rr = s.x;
      const double rho_next = s.y;
      if (rr < eps) {
        conv = true;
        break;
      }
      const float beta = (float)(rho_next / rho);
      pcg_update_p<int64_t>(gtid, gthreads, (int64_t)nm, beta, P, AP);
      rho = rho_next;
      grid.sync();
    }

    if constexpr (NODEWISE) {
      if (out.nodewise) {
        float* nw = out.nodewise + out.nodewise_off[pid];
        int64_t i = gtid / m, l = gtid % m;
        for (int64_t e = gtid; e < nm; e += gthreads) {
          nw[swap ? l * n + i : e] = X[e];
          l += dl;
          i += di;
          if (l >= m) {
            l -= m;
            ++i;
          }
        }
      }
    }
    if (gtid == 0) {
      if (out.value) out.value[pid] = value;
      if (out.iters) out.iters[pid] = (int32_t)it;
      if (out.conv) out.conv[pid] = conv ? 1 : 0;
      if (out.residual) out.residual[pid] = (float)sqrt(rr);
      if (out.pair_a) out.pair_a[pid] = ga;
      if (out.pair_b) out.pair_b[pid] = gb;
      const double kval = conv ? value : __longlong_as_double(0x7ff8000000000000ll);
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
    grid.sync();
  }
}

template <int EK, bool NODEWISE>
static cudaError_t launch_grid_ek(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek,
                                  const PairJob& job, const SolveParams& prm, const SolveOut& out, float* vec,
                                  int64_t vstride, double2* gbuf, int nblocks, cudaStream_t stream) {
  auto kern = k_pcg_grid<EK, NODEWISE>;
  const size_t smem = kPanelStaticSmem;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  DatasetDev a0 = ds;
  KernelDesc a1 = vk, a2 = ek;
  PairJob a3 = job;
  SolveParams a4 = prm;
  SolveOut a5 = out;
  void* args[] = {&a0, &a1, &a2, &a3, &a4, &a5, &vec, &vstride, &gbuf};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(nblocks), dim3(kPT), args, smem, stream);
}

int grid_blocks(int num_sms) {
  int per_sm = 0;
  cudaFuncSetAttribute(k_pcg_grid<KK_SE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPanelStaticSmem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pcg_grid<KK_SE, false>, kPT, kPanelStaticSmem) !=
      cudaSuccess)
    per_sm = 1;
  int nw = 0;
  cudaFuncSetAttribute(k_pcg_grid<KK_SE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPanelStaticSmem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nw, k_pcg_grid<KK_SE, true>, kPT, kPanelStaticSmem) ==
          cudaSuccess &&
      nw < per_sm)
    per_sm = nw;
  return (per_sm < 1 ? 1 : per_sm) * num_sms;
}

template <bool NODEWISE>
static cudaError_t launch_grid_nw(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek,
                                  const PairJob& job, const SolveParams& prm, const SolveOut& out, float* vec,
                                  int64_t vstride, double2* gbuf, int nblocks, cudaStream_t stream) {
  int kind = prm.labeled ? ek.kind : KK_NONE;
  if (kind == KK_CONST1) kind = KK_NONE;
  switch (kind) {
    case KK_SE: return launch_grid_ek<KK_SE, NODEWISE>(ds, vk, ek, job, prm, out, vec, vstride, gbuf, nblocks, stream);
    case KK_DELTA:
      return launch_grid_ek<KK_DELTA, NODEWISE>(ds, vk, ek, job, prm, out, vec, vstride, gbuf, nblocks, stream);
    case KK_POLY:
      return launch_grid_ek<KK_POLY, NODEWISE>(ds, vk, ek, job, prm, out, vec, vstride, gbuf, nblocks, stream);
    default:
      return launch_grid_ek<KK_NONE, NODEWISE>(ds, vk, ek, job, prm, out, vec, vstride, gbuf, nblocks, stream);
  }
}

cudaError_t launch_pcg_grid(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                            const SolveParams& prm, const SolveOut& out, float* vec, int64_t vstride, double2* gbuf,
                            int nblocks, cudaStream_t stream) {
  if (job.npairs < 1) return cudaSuccess;
  if (out.nodewise)
    return launch_grid_nw<true>(ds, vk, ek, job, prm, out, vec, vstride, gbuf, nblocks, stream);
  return launch_grid_nw<false>(ds, vk, ek, job, prm, out, vec, vstride, gbuf, nblocks, stream);
}

}  // namespace MGK_PANEL_NS
}  // namespace mgk
