// Device-side data layout shared by the octile builder, the PBR reorder and
// the PCG solvers.  See DESIGN.md "Data layout in HBM".
//
// A dataset of G graphs lives in HBM as structure-of-arrays:
//   node arrays   [sum n]            p, q (f32), degree (f64 + f32), vertex label
//   edge arrays   [sum |E|]          i, j (i32), w (f32), edge label (f32 x ED)
//   octiles       [sum T]            Octile{row, col, nz_off, bitmap}
//   compact nz    [sum 2|E|]         w (f32), edge label (f32 x ED) in (tile, bit) order
//   tile-row ptr  [sum (ceil(n/8)+1)] first octile of every tile row (CSR over tile rows)
// Per-graph offsets (GraphDesc) index into these arrays.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mgk {

constexpr int kTile = 8;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One non-empty 8x8 block (tiles.py:23-48): bit (r%8)*8 + c%8 set per nonzero;
// the block's values sit at nz_off .. nz_off+popc(bitmap) in ascending bit order.
struct __align__(16) Octile {
  uint16_t row;      // tile row    (r / 8)
  uint16_t col;      // tile column (c / 8)
  uint32_t nz_off;   // offset of the first compact value, relative to the graph's nz base
  uint64_t bitmap;   // occupancy, bit = local_row * 8 + local_col
};

struct GraphDesc {
  int32_t n;          // node count
  int32_t ne;         // undirected edge count (S = 2 ne directed nonzeros)
  int64_t node_off;   // into node arrays
  int64_t edge_off;   // into edge arrays
  int64_t nz_off;     // into compact nz arrays (= 2 * edge_off)
  int64_t tile_off;   // into octiles
  int64_t trow_off;   // into tile-row pointer array (ceil(n/8) + 1 entries)
  int32_t ntiles;     // non-empty octiles
  int32_t maxdeg;     // largest row length (nonzeros of one node)
  int64_t rowptr_off; // into the row-pointer array (n + 1 entries, = node_off + graph index)
  int64_t panel_off;  // into the panel row-boundary array (npanels + 1 entries)
  int32_t npanels;    // row panels of <= kPanelCap nonzeros (0 if a row exceeds the cap)
  float dqr;          // max_i d_i / q_i: drives the Laplacian-splitting switch (laplacian_pair)
};

// SURVEY.md §7 H1.  For kappa_e = 1 the operator's diagonal d d'/kv and the row
// sums of the off-diagonal part (d - q)(d' - q') nearly cancel when q << d, so
// FP32 diag * p - XMV(p) loses log10(diag / s) digits, s = diag - rowsum.  With
// the Laplacian splitting the solvers form
//   A p = s * p - sum_{jj'} L_{ii',jj'} (p_jj' - p_ii'),   s in FP64,
// whose FP32 terms are differences of nearby values.  The cancellation factor
// diag / s ~ a b / (a + b) with a, b the graphs' max d/q; pairs above
// kLapFactor (error ~3e-8 x factor without the splitting, i.e. <= 5e-6 below it) switch it on.
// Config-4 random geometric graphs at q = 0.05 peak at 143 and keep the cheaper unsplit form (the
// split factored XMV gathers P twice); datasets past 2 * kPreciseLap run on the FP64 block solver.
constexpr float kLapFactor = 160.0f;

// Row panels (pcg_panel.cu): consecutive rows whose nonzeros fit 32 lanes x kPanelSlots.
#ifndef MGK_PANEL_SLOTS
#define MGK_PANEL_SLOTS 8
#endif
constexpr int kPanelSlots = MGK_PANEL_SLOTS;
constexpr int kPanelCap = 32 * kPanelSlots;

// Base-kernel descriptor (basekernels.py:60-244); kind codes match basekernels.py.
// KK_PROD = ProductComposite (one scalar sub-kernel per label component,
// basekernels.py:175-211), KK_RCONV = RConvolution (sum of a scalar inner
// kernel over all component pairs, basekernels.py:214-244).
enum KernelKind : int32_t { KK_CONST1 = 0, KK_DELTA = 1, KK_SE = 2, KK_POLY = 3, KK_NONE = 4, KK_PROD = 5,
                            KK_RCONV = 6 };
constexpr int kMaxPoly = 8;
constexpr int kMaxSub = 4;
struct KernelDesc {
  int32_t kind;
  int32_t ncoef;
  float h;             // delta baseline
  float alpha;         // SE alpha
  float se_scale;      // sqrt(alpha * log2(e)): labels are pre-scaled so SE = exp2(-|a-b|^2)
  float coef[kMaxPoly];
  int32_t nsub;                 // PROD: components; RCONV: 1 (the inner kernel)
  int32_t sub_kind[kMaxSub];    // scalar kinds (CONST1 / DELTA / SE / POLY; POLY uses coef)
  float sub_h[kMaxSub];         // delta baselines
};


// Edge base kernel on lowered scalar labels, specialised on the kind
// (basekernels.py:73-172): SE labels are pre-scaled so kappa = exp2(-(a-b)^2),
// delta labels are equivalence-class ids compared as integers.
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

// kappa(a, b) * w with the weight carried in the form the kind prefers: for SE
// the U-side weight is stored as log2(w) and folded into the exponent,
// kappa * w = exp2(log2 w - (a - b)^2)  (FADD + FFMA + MUFU.EX2 per contribution);
// the other kinds multiply (wf = w).
template <int EK>
__device__ __forceinline__ float edge_kappa_w(const KernelDesc& k, float a, float b, float wf) {
  if constexpr (EK == KK_SE) {
    const float d = a - b;
    return ex2_approx(fmaf(-d, d, wf));
  } else {
    return edge_kappa<EK>(k, a, b) * wf;
  }
}

// U-side weight in the form edge_kappa_w expects.
template <int EK>
__device__ __forceinline__ float weight_form(float w) {
  if constexpr (EK == KK_SE) return log2f(w);
  return w;
}

// Label storage kinds (graphs.py:126-146).
enum LabelKind : int32_t { LK_NONE = 0, LK_CAT = 1, LK_VEC = 2 };

constexpr int kMaxLabelDim = 4;

struct DatasetDev {
  int32_t G;
  int32_t nl_kind, nl_dim;     // vertex labels
  int32_t el_kind, el_dim;     // edge labels
  const GraphDesc* graphs;
  // node arrays
  const float* p;
  const float* q;
  const double* deg;           // d_i = sum_j w_ij + q_i, accumulated in ascending column order (f64)
  const double* q64;           // q_i (f64)
  const float* dm;             // d_i - q_i (= the FP32 row sum of the weights), Laplacian splitting
  const float* vlabel;         // [sum n * nl_dim]  (categorical tokens stored as int bits)
  // octiles
  const Octile* tiles;
  const int32_t* trow;         // tile-row pointers, relative to the graph's tile_off
  const float* nz_w;           // [sum S]
  const float* nz_label;       // [sum S * el_dim]
  // row-ordered expansion of the octiles (built on the device once per dataset)
  const int32_t* rowptr;       // [sum (n + 1)] relative to the graph's nz base
  const float4* rowent;        // [sum S] {col (int bits), w, label0, 0} ascending column per row
  const int32_t* panel_row;    // [sum (npanels + 1)] first row of every panel
  const int2* symk;            // [sum E] per undirected edge (i, j): positions of i->j and j->i in the row
                               // expansion (relative to the graph's nz base; k_sym_fill)
};

__host__ __device__ inline int ceil8(int n) { return (n + 7) >> 3; }

// kappa(a, b) for scalar labels with the descriptor semantics.
// SE labels are pre-scaled by se_scale, so kappa = exp2(-(a-b)^2).
__device__ __forceinline__ float kernel_scalar(const KernelDesc& k, float a, float b) {
  switch (k.kind) {
    case KK_DELTA:
      return (a == b) ? 1.0f : k.h;
    case KK_SE: {
      float d = a - b;
      return exp2f(-d * d);
    }
    case KK_POLY: {
      float d = fabsf(a - b);
      float acc = 0.0f;
      for (int c = k.ncoef - 1; c >= 0; --c) acc = fmaf(acc, d, k.coef[c]);
      return fminf(fmaxf(acc, 0.0f), 1.0f);
    }
    default:
      return 1.0f;
  }
}

// Scalar sub-kernel c of a composite / convolution descriptor on lowered labels
// (delta components are equivalence-class ids, SE components pre-scaled).
__device__ __forceinline__ float sub_kernel(const KernelDesc& k, int c, float a, float b) {
  switch (k.sub_kind[c]) {
    case KK_DELTA:
      return (__float_as_int(a) == __float_as_int(b)) ? 1.0f : k.sub_h[c];
    case KK_SE: {
      float d = a - b;
      return exp2f(-d * d);
    }
    case KK_POLY: {
      float d = fabsf(a - b);
      float acc = 0.0f;
      for (int i = k.ncoef - 1; i >= 0; --i) acc = fmaf(acc, d, k.coef[i]);
      return fminf(fmaxf(acc, 0.0f), 1.0f);
    }
    default:
      return 1.0f;
  }
}

// Vector-label version (dim <= kMaxLabelDim); categorical labels compare as ints.
__device__ __forceinline__ float kernel_vec(const KernelDesc& k, const float* a, const float* b, int dim,
                                            bool categorical) {
  switch (k.kind) {
    case KK_PROD: {
      float out = 1.0f;
      for (int c = 0; c < k.nsub; ++c) out *= sub_kernel(k, c, a[c], b[c]);
      return out;
    }
    case KK_RCONV: {
      float s = 0.0f;
      for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j) s += sub_kernel(k, 0, a[i], b[j]);
      return s;
    }
    case KK_DELTA: {
      bool eq = true;
      if (categorical) {
        for (int c = 0; c < dim; ++c) eq &= (__float_as_int(a[c]) == __float_as_int(b[c]));
      } else {
        for (int c = 0; c < dim; ++c) eq &= (a[c] == b[c]);
      }
      return eq ? 1.0f : k.h;
    }
    case KK_SE: {
      float s = 0.0f;
      for (int c = 0; c < dim; ++c) {
        float d = a[c] - b[c];
        s = fmaf(d, d, s);
      }
      return exp2f(-s);
    }
    case KK_POLY:
      return kernel_scalar(k, a[0], b[0]);
    default:
      return 1.0f;
  }
}

}  // namespace mgk
