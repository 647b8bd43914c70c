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
// L-nonzeros k' = l + 32 t (t < SLOTS, held in registers for the whole solve)
// and the L-node i' = l for the vector operations.  The PCG vectors live in
// shared memory as [i][32] (i = U node, column = lane), so the XMV gather
// P[j][col_L(k')] is bank-conflict free (bank = column) and every vector op is
// lane-local.  For U-row i:
//
//   acc[t] = sum_{k in U(i)} kappa(e_k, e'_t) * w_k * P[j_k][col_L(t)]   (registers)
//   SEG[k'] = acc[t] * w'_t;  AP[i][i'] = diag * P[i][i'] - sum_{k' in L(i')} SEG[k']
//
// i.e. exactly sum_{j, j'} w_ij w'_i'j' ke(e_ij, e'_i'j') p[j, j'] (product.py:454-478).
// Unlabeled pairs use the factorised form AP = D.P - A (P B^T) (the paper's
// dense x dense unlabeled primitive, product.py:94), which costs
// n*S_L + S_U*m instead of S_U*S_L.
//
// The octile format is what the warp reads from HBM: the prologue expands the
// two graphs' octiles (16-byte records, one 64-bit bitmap each) into per-row
// neighbour lists with popc/bit-scan, which is also how rows are ordered
// (ascending column, as the reference's tile order implies).
#include <cstdio>

#include "mgk_internal.h"

namespace mgk {

constexpr int kWarpsPerBlock = 2;

template <int NU, int SLOTS, bool UNLAB>
struct WarpSmem {
  float P[NU][32];
  float AP[NU][32];      // + DG: staging area for the L nonzeros during the prologue
  float DG[NU][32];
  float T[UNLAB ? NU : 1][32];
  float4 UE[32 * SLOTS]; // U nonzeros in row order: {col (int bits), w, label, 0}
  float SEG[32 * SLOTS];
  int urow[NU + 8];
  float upq[NU];         // p_i (start probability) of U nodes
  float udq[NU];         // d_i q_i of U nodes
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int EK>
__device__ __forceinline__ float edge_kappa(const KernelDesc& k, float a, float b) {
  if constexpr (EK == KK_SE) {
    float d = a - b;
    return ex2_approx(-d * d);
  } else if constexpr (EK == KK_DELTA) {
    return (__float_as_int(a) == __float_as_int(b)) ? 1.0f : k.h;
  } else if constexpr (EK == KK_POLY) {
    float d = fabsf(a - b);
    float acc = 0.0f;
    for (int c = k.ncoef - 1; c >= 0; --c) acc = fmaf(acc, d, k.coef[c]);
    return fminf(fmaxf(acc, 0.0f), 1.0f);
  } else {
    return 1.0f;
  }
}

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

// Expand a graph's octiles into row-ordered nonzeros {col, w, label} at dst and
// row pointers at rowptr[0..n] (lane i handles row i; n <= 32).
__device__ void octiles_to_rows(const DatasetDev& ds, const GraphDesc& g, int lane, float4* dst, int* rowptr,
                                int el_dim) {
  int cnt = 0;
  const int32_t* tr = ds.trow + g.trow_off;
  const Octile* tiles = ds.tiles + g.tile_off;
  int I = lane >> 3, r = lane & 7;
  int t0 = 0, t1 = 0;
  if (lane < g.n) {
    t0 = tr[I];
    t1 = tr[I + 1];
    for (int t = t0; t < t1; ++t) cnt += __popc((uint32_t)(tiles[t].bitmap >> (8 * r)) & 0xffu);
  }
  int incl = warp_incl_scan(cnt, lane);
  int start = incl - cnt;
  if (lane < g.n) rowptr[lane] = start;
  if (lane == g.n - 1) rowptr[g.n] = incl;
  if (lane < g.n) {
    const float* w = ds.nz_w + g.nz_off;
    const float* lab = ds.nz_label + g.nz_off * el_dim;
    for (int t = t0; t < t1; ++t) {
      Octile o = tiles[t];
      uint32_t byte = (uint32_t)(o.bitmap >> (8 * r)) & 0xffu;
      int base = o.nz_off + __popcll(o.bitmap & ((1ull << (8 * r)) - 1ull));
      for (int c = 0; byte; ++c, byte &= byte - 1) {
        int lc = __ffs(byte) - 1;
        int k = base + c;
        float l0 = el_dim > 0 ? lab[(int64_t)k * el_dim] : 0.0f;
        dst[start++] = make_float4(__int_as_float(o.col * 8 + lc), w[k], l0, 0.0f);
      }
    }
  }
}

__device__ __forceinline__ void write_pair_outputs(const SolveOut& out, unsigned long long pid, int ga, int gb,
                                                   double val, int64_t it, bool conv, double rr, int lane) {
  if (lane != 0) return;
  if (out.value) out.value[pid] = val;
  if (out.iters) out.iters[pid] = (int32_t)it;
  if (out.conv) out.conv[pid] = conv ? 1 : 0;
  if (out.residual) out.residual[pid] = (float)sqrt(rr);
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

// Tiny product systems (n*m <= kTinyNM, or self pairs whose symmetric subspace
// is that small): CG terminates there by Krylov exhaustion, which FP32
// rounding in the matvec delays by a few iterations.  These pairs run the
// same algorithm with FP64 vectors and FP64 accumulation (coefficients stay
// FP32), which restores the reference's iteration counts; element e of the
// field is owned by lane e % 32.
constexpr int kTinyNM = 128;

template <int EK>
__device__ void solve_tiny(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const SolveParams& prm,
                           const GraphDesc& U, const GraphDesc& L, const float4* ue, const int* urow,
                           const float4* le, const int* lrow, double* P, double* AP, double* DG, int lane,
                           double& value_out, int64_t& it_out, bool& conv_out, double& rr_out, float* nw, bool swap) {
  const int nu = U.n, m = L.n, nm = nu * m;
  const bool vlab = (vk.kind != KK_CONST1 && vk.kind != KK_NONE && ds.nl_kind != LK_NONE);
  double r[4], x[4];
  double bb_u = 0.0, bb_l = 0.0;
  if (lane < nu) {
    double dq = ds.deg[U.node_off + lane] * (double)ds.q[U.node_off + lane];
    bb_u = dq * dq;
  }
  if (lane < m) {
    double dq = ds.deg[L.node_off + lane] * (double)ds.q[L.node_off + lane];
    bb_l = dq * dq;
  }
  double rho = 0.0, rr = 0.0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    int e = lane + 32 * s;
    r[s] = 0.0;
    x[s] = 0.0;
    if (e < nm) {
      int i = e / m, l = e - i * m;
      int64_t vu = U.node_off + i, vl = L.node_off + l;
      float kv = 1.0f;
      if (vlab)
        kv = fmaxf(kernel_vec(vk, ds.vlabel + vu * ds.nl_dim, ds.vlabel + vl * ds.nl_dim, ds.nl_dim,
                              ds.nl_kind == LK_CAT), prm.v_min);
      double dg = ds.deg[vu] * ds.deg[vl] / (double)kv;
      double b = (ds.deg[vu] * (double)ds.q[vu]) * (ds.deg[vl] * (double)ds.q[vl]);
      DG[e] = dg;
      r[s] = b;
      double z = b / dg;
      P[e] = z;
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
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      int e = lane + 32 * s;
      if (e < nm) {
        int i = e / m, l = e - i * m;
        double acc = 0.0;
        for (int k = urow[i]; k < urow[i + 1]; ++k) {
          const float4 a = ue[k];
          const double* prow = P + __float_as_int(a.x) * m;
          for (int q = lrow[l]; q < lrow[l + 1]; ++q) {
            const float4 b = le[q];
            float c = edge_kappa<EK>(ek, a.z, b.z) * a.y * b.y;
            acc = fma((double)c, prow[__float_as_int(b.x)], acc);
          }
        }
        AP[e] = DG[e] * P[e] - acc;
      }
    }
    __syncwarp();
    ++it;
    double pap = 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      int e = lane + 32 * s;
      if (e < nm) pap += P[e] * AP[e];
    }
    const double alpha = rho / warp_sum(pap);
    double rr_l = 0.0, rz_l = 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      int e = lane + 32 * s;
      if (e < nm) {
        x[s] += alpha * P[e];
        r[s] -= alpha * AP[e];
        rr_l += r[s] * r[s];
        rz_l += r[s] * (r[s] / DG[e]);
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
      int e = lane + 32 * s;
      if (e < nm) P[e] = r[s] / DG[e] + beta * P[e];
    }
    rho = rho_next;
    __syncwarp();
  }
  double val = 0.0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    int e = lane + 32 * s;
    if (e < nm) {
      int i = e / m, l = e - i * m;
      val += (double)ds.p[U.node_off + i] * (double)ds.p[L.node_off + l] * x[s];
      if (nw) nw[swap ? (int64_t)l * nu + i : (int64_t)e] = (float)x[s];
    }
  }
  value_out = warp_sum(val);
  it_out = it;
  conv_out = conv;
  rr_out = rr;
}

template <int NU, int SLOTS, int EK>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_pcg_warp(DatasetDev ds, KernelDesc vk, KernelDesc ek, PairJob job, SolveParams prm, SolveOut out,
           unsigned long long* queue) {
  constexpr bool UNLAB = (EK == KK_NONE);
  using Smem = WarpSmem<NU, SLOTS, UNLAB>;
  static_assert(sizeof(float) * 2 * NU * 32 >= sizeof(float4) * 32 * SLOTS, "staging area too small");
  static_assert(sizeof(float) * NU * 32 >= 3 * sizeof(double) * kTinyNM, "tiny-pair area too small");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  Smem& S = reinterpret_cast<Smem*>(smem_raw)[threadIdx.x >> 5];
  float4* stage = reinterpret_cast<float4*>(&S.AP[0][0]);
  const int el_dim = ds.el_dim;

  for (;;) {
    unsigned long long pid = 0;
    if (lane == 0) pid = atomicAdd(queue, 1ull);
    pid = __shfl_sync(0xffffffffu, pid, 0);
    if (pid >= (unsigned long long)job.npairs) break;
    int32_t ga, gb;
    decode_pair(job, (int64_t)pid, ga, gb);
    GraphDesc A = ds.graphs[ga], B = ds.graphs[gb];
    // orientation: L takes the graph that minimises S_U * ceil(S_L / 32)
    int SA = 2 * A.ne, SB = 2 * B.ne;
    long costAB = (long)SA * ((SB + 31) / 32) + A.n;  // U = A, L = B
    long costBA = (long)SB * ((SA + 31) / 32) + B.n;
    bool swap = (costBA < costAB) && SA <= 32 * SLOTS;
    if (SB > 32 * SLOTS) swap = true;
    const GraphDesc U = swap ? B : A;
    const GraphDesc L = swap ? A : B;
    const int nu = U.n, m = L.n;
    const int SL = 2 * L.ne;
    const int nslots = (SL + 31) >> 5;

    // ---- prologue: octiles -> rows
    octiles_to_rows(ds, U, lane, S.UE, S.urow, el_dim);
    int lrow_tmp[1];
    (void)lrow_tmp;
    __shared__ int lrow_sh[kWarpsPerBlock][33];
    int* lrow = lrow_sh[threadIdx.x >> 5];
    octiles_to_rows(ds, L, lane, stage, lrow, el_dim);
    if (nu == 0 || m == 0) { /* unreachable: n >= 1 */ }
    __syncwarp();
    int lcol[SLOTS];
    float lw[SLOTS], llab[SLOTS];
#pragma unroll
    for (int t = 0; t < SLOTS; ++t) {
      int k = lane + 32 * t;
      if (k < SL) {
        float4 e = stage[k];
        lcol[t] = __float_as_int(e.x);
        lw[t] = e.y;
        llab[t] = e.z;
      } else {
        lcol[t] = 0;
        lw[t] = 0.0f;
        llab[t] = 0.0f;
      }
    }
    int lr0 = 0, lr1 = 0;
    if (lane < m) {
      lr0 = lrow[lane];
      lr1 = lrow[lane + 1];
    }
    if (nu * m <= kTinyNM) {
      double val, rrt;
      int64_t itt;
      bool cvt;
      double* P64 = reinterpret_cast<double*>(&S.P[0][0]);
      float* nw = out.nodewise ? out.nodewise + out.nodewise_off[pid] : nullptr;
      solve_tiny<EK>(ds, vk, ek, prm, U, L, S.UE, S.urow, stage, lrow, P64, P64 + kTinyNM, P64 + 2 * kTinyNM, lane,
                     val, itt, cvt, rrt, nw, swap);
      write_pair_outputs(out, pid, ga, gb, val, itt, cvt, rrt, lane);
      __syncwarp();
      continue;
    }
    __syncwarp();  // staging (AP/DG) is free again

    // node data: L on lanes, U in shared memory
    float ld = 1.0f, ldq = 0.0f, lp = 0.0f;
    if (lane < m) {
      int64_t v = L.node_off + lane;
      ld = (float)ds.deg[v];
      ldq = (float)(ds.deg[v] * (double)ds.q[v]);
      lp = ds.p[v];
    }
    if (lane < nu) {
      int64_t v = U.node_off + lane;
      S.udq[lane] = (float)(ds.deg[v] * (double)ds.q[v]);
      S.upq[lane] = ds.p[v];
    }
    // diag = d_i d'_i' / max(kv, v_min)  (product.py:164-178, 210)
    const bool vlab = (vk.kind != KK_CONST1 && vk.kind != KK_NONE && ds.nl_kind != LK_NONE);
    double bb_l = (lane < m) ? (double)ldq * (double)ldq : 0.0;
    double bb_u = (lane < nu) ? (double)S.udq[lane] * (double)S.udq[lane] : 0.0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      if (i < nu) {
        float dg = 1.0f;
        if (lane < m) {
          int64_t vu = U.node_off + i, vl = L.node_off + lane;
          float kv = 1.0f;
          if (vlab) {
            const float* la = ds.vlabel + vu * ds.nl_dim;
            const float* lb = ds.vlabel + vl * ds.nl_dim;
            kv = fmaxf(kernel_vec(vk, la, lb, ds.nl_dim, ds.nl_kind == LK_CAT), prm.v_min);
          }
          dg = (float)(ds.deg[vu] * (double)ld) / kv;
        }
        S.DG[i][lane] = dg;
      }
    }
    // b = (d q) (x) (d' q');  eps = tol^2 b.b  (solver.py:69-74, 88) -- b.b is separable
    const double bb = warp_sum(bb_u) * warp_sum(bb_l);
    const double eps = prm.tol2 * bb;
    const int64_t max_iter = prm.max_iter > 0 ? prm.max_iter : 10ll * nu * m;
    __syncwarp();

    float r[NU], x[NU];
    double rho = 0.0, rr = 0.0;
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      x[i] = 0.0f;
      r[i] = 0.0f;
      if (i < nu && lane < m) {
        r[i] = S.udq[i] * ldq;
        float z = r[i] / S.DG[i][lane];
        S.P[i][lane] = z;
        rho += (double)r[i] * (double)z;
        rr += (double)r[i] * (double)r[i];
      } else if (i < nu) {
        S.P[i][lane] = 0.0f;
      }
    }
    rho = warp_sum(rho);
    rr = warp_sum(rr);
    bool conv = rr < eps;
    int64_t it = 0;
    __syncwarp();

    while (!conv && it < max_iter) {
      // ---------------- XMV: AP = diag * P - offdiag(P)
      if constexpr (UNLAB) {
        // T[j][i'] = sum_{k' in L(i')} w' P[j][col(k')]   (P B^T)
        for (int j = 0; j < nu; ++j) {
          const float* prow = S.P[j];
#pragma unroll
          for (int t = 0; t < SLOTS; ++t)
            if (t < nslots) S.SEG[lane + 32 * t] = lw[t] * prow[lcol[t]];
          __syncwarp();
          if (lane < m) {
            float s = 0.0f;
            for (int k = lr0; k < lr1; ++k) s += S.SEG[k];
            S.T[j][lane] = s;
          }
          __syncwarp();
        }
        for (int i = 0; i < nu; ++i) {
          float s = 0.0f;
          for (int k = S.urow[i]; k < S.urow[i + 1]; ++k) {
            float4 e = S.UE[k];
            s = fmaf(e.y, S.T[__float_as_int(e.x)][lane], s);
          }
          S.AP[i][lane] = S.DG[i][lane] * S.P[i][lane] - s;
        }
      } else {
        for (int i = 0; i < nu; ++i) {
          float acc[SLOTS];
#pragma unroll
          for (int t = 0; t < SLOTS; ++t) acc[t] = 0.0f;
          const int k0 = S.urow[i], k1 = S.urow[i + 1];
          for (int k = k0; k < k1; ++k) {
            float4 e = S.UE[k];
            const float* prow = S.P[__float_as_int(e.x)];
            const float wa = e.y, la = e.z;
#pragma unroll
            for (int t = 0; t < SLOTS; ++t) {
              if (t < nslots) {
                float kap = edge_kappa<EK>(ek, la, llab[t]);
                acc[t] = fmaf(kap, wa * prow[lcol[t]], acc[t]);
              }
            }
          }
#pragma unroll
          for (int t = 0; t < SLOTS; ++t)
            if (t < nslots) S.SEG[lane + 32 * t] = acc[t] * lw[t];
          __syncwarp();
          if (lane < m) {
            float s = 0.0f;
            for (int k = lr0; k < lr1; ++k) s += S.SEG[k];
            S.AP[i][lane] = S.DG[i][lane] * S.P[i][lane] - s;
          }
          __syncwarp();
        }
      }
      __syncwarp();
      if (ga == gb) {
        // self pair: the exact operator maps symmetric fields to symmetric fields;
        // symmetrising AP keeps the FP32 Krylov space in that subspace, as the
        // reference's FP64 iteration does (iteration-count parity on the Gram diagonal)
        float sym[NU];
#pragma unroll
        for (int i = 0; i < NU; ++i)
          if (i < nu && lane < m) sym[i] = 0.5f * (S.AP[i][lane] + S.AP[lane][i]);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < NU; ++i)
          if (i < nu && lane < m) S.AP[i][lane] = sym[i];
        __syncwarp();
      }
      ++it;
      // ---------------- PCG update (solver.py:98-110)
      double pap = 0.0;
#pragma unroll
      for (int i = 0; i < NU; ++i)
        if (i < nu && lane < m) pap += (double)S.P[i][lane] * (double)S.AP[i][lane];
      pap = warp_sum(pap);
      const double alpha = rho / pap;
      const float af = (float)alpha;
      double rr_l = 0.0, rz_l = 0.0;
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        if (i < nu && lane < m) {
          x[i] = fmaf(af, S.P[i][lane], x[i]);
          r[i] = fmaf(-af, S.AP[i][lane], r[i]);
          float z = r[i] / S.DG[i][lane];
          rr_l += (double)r[i] * (double)r[i];
          rz_l += (double)r[i] * (double)z;
        }
      }
      rr = warp_sum(rr_l);
      const double rho_next = warp_sum(rz_l);
      if (rr < eps) {
        conv = true;
        break;
      }
      const float beta = (float)(rho_next / rho);
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        if (i < nu && lane < m) {
          float z = r[i] / S.DG[i][lane];
          S.P[i][lane] = fmaf(beta, S.P[i][lane], z);
        }
      }
      rho = rho_next;
      __syncwarp();
    }

    // ---------------- epilogue: value = px . x (solver.py:114)
    double val = 0.0;
#pragma unroll
    for (int i = 0; i < NU; ++i)
      if (i < nu && lane < m) val += (double)S.upq[i] * (double)lp * (double)x[i];
    val = warp_sum(val);
    if (out.nodewise) {
      float* nw = out.nodewise + out.nodewise_off[pid];
      // field is [n_a][n_b] with a = first graph of the pair
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        if (i < nu && lane < m) {
          int64_t idx = swap ? (int64_t)lane * nu + i : (int64_t)i * m + lane;
          nw[idx] = x[i];
        }
      }
    }
    write_pair_outputs(out, pid, ga, gb, val, it, conv, rr, lane);
    __syncwarp();
  }
}

template <int EK>
static cudaError_t launch_ek(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                             const SolveParams& prm, const SolveOut& out, unsigned long long* queue, int num_sms,
                             cudaStream_t stream) {
  constexpr int NU = SmallClass::NU, SLOTS = SmallClass::SLOTS;
  using Smem = WarpSmem<NU, SLOTS, EK == KK_NONE>;
  auto kern = k_pcg_warp<NU, SLOTS, EK>;
  size_t smem = sizeof(Smem) * kWarpsPerBlock;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarpsPerBlock * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)per_sm * num_sms;
  int64_t need = (job.npairs + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, kWarpsPerBlock * 32, smem, stream>>>(ds, vk, ek, job, prm, out, queue);
  return cudaGetLastError();
}

cudaError_t launch_pcg_warp(const DatasetDev& ds, const KernelDesc& vk, const KernelDesc& ek, const PairJob& job,
                            const SolveParams& prm, const SolveOut& out, unsigned long long* queue, int num_sms,
                            cudaStream_t stream) {
  int kind = prm.labeled ? ek.kind : KK_NONE;
  if (kind == KK_CONST1) kind = KK_NONE;
  switch (kind) {
    case KK_SE: return launch_ek<KK_SE>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
    case KK_DELTA: return launch_ek<KK_DELTA>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
    case KK_POLY: return launch_ek<KK_POLY>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
    default: return launch_ek<KK_NONE>(ds, vk, ek, job, prm, out, queue, num_sms, stream);
  }
}

}  // namespace mgk
