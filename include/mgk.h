/* mgk.h -- C-ABI of the B200 marginalized-graph-kernel solver (libmgk.so).
 *
 * This is the drop-in boundary for the reference's array bindings
 * (pkg/bindings/src/mgkbind) and its core facade (pkg/src/mgksolver):
 * plain pointers and sizes, no torch or numpy types.  Each entry point names
 * the reference interface it replaces.  Return codes: 0 = ok, < 0 = error
 * class (MGK_E_*); mgk_last_error() returns the thread-local message, whose
 * text follows the reference's exceptions (graphs.py:161-199, product.py:
 * 153-178, solver.py:226-231).  The library copies what it needs and never
 * retains caller pointers after a call returns.  A context is bound to one
 * CUDA device; calls on one context are serialised by the caller.
 */
#ifndef MGK_H
#define MGK_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mgk_ctx mgk_ctx;

enum {
  MGK_OK = 0,
  MGK_E_INVALID = -1,   /* ValueError: invalid graph / argument (graphs.py:161-199, solver.py:226-231) */
  MGK_E_SHAPE = -2,     /* KernelShapeError (basekernels.py:14-15, product.py:153-178) */
  MGK_E_CUDA = -3,      /* CUDA runtime failure (no CPU fallback exists) */
  MGK_E_UNSUPPORTED = -4, /* kernel variant without a device lowering */
  MGK_E_STATE = -5      /* call order (e.g. solve before upload) */
};

/* label kinds (graphs.py:126-146) */
enum { MGK_LABEL_NONE = 0, MGK_LABEL_CATEGORICAL = 1, MGK_LABEL_VECTOR = 2 };
/* reorder methods (solver.py:209, 249-259) */
enum { MGK_REORDER_NONE = 0, MGK_REORDER_PBR = 1, MGK_REORDER_RCM = 2, MGK_REORDER_MORTON = 3 };

/* Version string of the library build. */
const char* mgk_version(void);

/* Thread-local message of the last failing call on this thread. */
const char* mgk_last_error(void);

/* Create a context on CUDA device `device` (replaces the per-call
 * `python -m mgksolver` subprocess of marshal.py:150-155). */
int mgk_ctx_create(mgk_ctx** out, int device);
int mgk_ctx_destroy(mgk_ctx* ctx);

/* Upload a dataset of N graphs in packed form (replaces write_graph_json +
 * load_graph, marshal.py:87-115 / graphio.py:115-180, and the LabeledGraph
 * list passed to compute_gram, gram.py:57).
 *   node_off[N+1], edge_off[N+1]: prefix offsets into the node / edge arrays;
 *   ei, ej: endpoints local to their graph (stored once per undirected edge);
 *   w: edge weights; p, q: start / stop probabilities per node;
 *   node_labels: int64[sum n] (categorical) or double[sum n * nl_dim] (vector);
 *   edge_labels: int64[sum E] or double[sum E * el_dim].
 * Validation follows validate_graph (graphs.py:161-199); the first invalid
 * graph fails the call with "graph <g> invalid: <violations>". */
int mgk_upload(mgk_ctx* ctx, int32_t N, const int64_t* node_off, const int64_t* edge_off, const int32_t* ei,
               const int32_t* ej, const double* w, const double* p, const double* q, int nl_kind, int nl_dim,
               const void* node_labels, int el_kind, int el_dim, const void* edge_labels);

/* Base kernels by the reference SPEC grammar `const1 | delta:H | se:A | poly:c0,c1,..`
 * (basekernels.py:247-261); NULL or "" means None (vertex: all-ones
 * similarity, product.py:172; edge: kappa = 1, product.py:74-79). */
int mgk_set_kernels(mgk_ctx* ctx, const char* vertex_spec, const char* edge_spec);

/* Vertex-similarity floor v_min of the solves that follow (SolverConfig.v_min,
 * solver.py:39-52, threaded into vertex_similarity_matrix by solver.py:241-242,
 * product.py:164-178): kv = max(kappa_v, v_min); a floored similarity <= 0
 * fails the solve with MGK_E_INVALID "vertex kernel produced non-positive
 * similarity".  Default 1e-12 (DEFAULT_VERTEX_FLOOR). */
int mgk_set_vertex_floor(mgk_ctx* ctx, double v_min);

/* Per-graph node reordering on the device (solver.py:249-259 _reorder_for),
 * one method for every graph:
 *   MGK_REORDER_PBR     pbr_reorder (reorder.py:361-404), same seed for every
 *                       graph (solver.py:236-237);
 *   MGK_REORDER_RCM     rcm_reorder (reorder.py:412-443), seed unused;
 *   MGK_REORDER_MORTON  morton_reorder of the node coordinates (reorder.py:
 *                       448-478): the dataset's vector node labels of
 *                       dimension 2 or 3, else MGK_E_INVALID "morton
 *                       reordering needs 2D/3D coordinate node labels".
 * Writes forward maps (old -> new) into perms_out[sum n] when non-NULL.  With
 * apply != 0 the dataset is relabelled (apply_permutation, reorder.py:86-109)
 * and its octiles rebuilt. */
int mgk_reorder(mgk_ctx* ctx, int method, uint64_t seed, int apply, int64_t* perms_out);

/* Octiles of graph g as built on the device (build_tiles, tiles.py:85-127).
 * Call with rc_out == NULL to get *ntiles and *nnz; then pass buffers of
 * 2*ntiles int32 (row, col), ntiles uint64 bitmaps, nnz float values. */
int mgk_tiles(mgk_ctx* ctx, int32_t g, int32_t* ntiles, int32_t* nnz, int32_t* rc_out, uint64_t* bitmap_out,
              float* w_out);

/* Degree vector d_i = sum_j w_ij + q_i of graph g (degree_vector, graphs.py:202-214). */
int mgk_degrees(mgk_ctx* ctx, int32_t g, double* d_out);

/* All-pairs Gram matrix (compute_gram, gram.py:57-95): K[N*N] row-major,
 * mirrored, NaN where the pair did not converge; iters[N*N], conv[N*N].
 * Any output may be NULL (the result then stays on the device; used by the
 * device-resident benchmark).  max_iter 0 -> 10*n*m (solver.py:87). */
int mgk_gram(mgk_ctx* ctx, double tol, int64_t max_iter, double* K, int32_t* iters, uint8_t* conv);

/* Iteration counts of the last mgk_gram / mgk_gram_normalized on this context as
 * int64[N*N] (the reference's GramResult.iterations dtype, gram.py:73), widened
 * on the device so the host receives them without a conversion pass. */
int mgk_gram_iterations64(mgk_ctx* ctx, int64_t* iters);

/* mgk_gram followed by normalize_gram (gram.py:98-107) on the device-resident
 * matrix: K[a,b] / sqrt(K[a,a] K[b,b]), unit diagonal, NaN propagates; a
 * non-NaN diagonal entry <= 0 fails with MGK_E_INVALID (the reference's
 * ValueError).  Replaces mgkbind.gram(normalize=True) (__init__.py:70-92). */
int mgk_gram_normalized(mgk_ctx* ctx, double tol, int64_t max_iter, double* K, int32_t* iters, uint8_t* conv);

/* Shard of the Gram pairs for multi-GPU runs (the per-GPU part of the
 * 8-GPU pair scheduling in north_star; the reference's equivalent is the
 * pair queue of gram.py:69-86): this context solves the pairs whose
 * cost-ordered id is congruent to rank modulo world and writes compact
 * per-pair results (graph ids a, b, value, iterations, converged).  Call
 * with all outputs NULL to learn *npairs_out; the results of the last call
 * also stay on the device. */
int mgk_gram_shard(mgk_ctx* ctx, int rank, int world, double tol, int64_t max_iter, int64_t* npairs_out,
                   int32_t* pair_a, int32_t* pair_b, double* value, int32_t* iters, uint8_t* conv);

/* mgk_gram_shard with the per-pair records written to caller-owned DEVICE
 * buffers on this context's device (no host round trip): the input of a
 * device-side gather (NCCL / peer copies) in multi-process runs.  All outputs
 * NULL: only *npairs_out. */
int mgk_gram_shard_device(mgk_ctx* ctx, int rank, int world, double tol, int64_t max_iter, int64_t* npairs_out,
                          int32_t* d_pair_a, int32_t* d_pair_b, double* d_value, int32_t* d_iters,
                          uint8_t* d_conv);

/* Assemble gathered shard records (device buffers on `device`, graph ids < 0
 * mark padding) into device-resident G x G matrices: mirrored writes, NaN
 * where the pair did not converge (gram.py:86-90).  Any matrix may be NULL. */
int mgk_gram_assemble(int device, int64_t npairs, const int32_t* d_pair_a, const int32_t* d_pair_b,
                      const double* d_value, const int32_t* d_iters, const uint8_t* d_conv, int64_t G, double* d_K,
                      int32_t* d_K_iters, uint8_t* d_K_conv);

/* All-pairs Gram over several devices from ONE host process (north_star (4):
 * the N(N+1)/2 pair list load-balanced over the GPUs of a box, no collective
 * beyond the final gather; the reference's pair queue, gram.py:69-86).  Every
 * context holds the same dataset and kernels (one context per device);
 * context k solves the cost-ordered pair ids congruent to k mod nctx on its own
 * host thread and scatters its compact results straight into the caller's
 * K / iters / conv (mirrored, NaN where not converged).  mgk_last_timing of
 * each context then reports the slowest device's solve time. */
int mgk_gram_multi(mgk_ctx* const* ctxs, int nctx, double tol, int64_t max_iter, double* K, int32_t* iters,
                   uint8_t* conv);

/* Batch of explicit pairs (the per-pair `kernel` of solver.py:212-246 without
 * reordering): value[k], iters[k], residual[k], conv[k]; nodewise (nullable)
 * receives the n_a x m_b float64 field of every pair back to back. */
int mgk_pairs(mgk_ctx* ctx, int64_t npairs, const int32_t* a, const int32_t* b, double tol, int64_t max_iter,
              double* value, int32_t* iters, double* residual, uint8_t* conv, double* nodewise);

/* Consumer of streamed nodewise results: one call per chunk of solved pairs.
 * offsets[k] .. offsets[k+1] index pair k's n_a x n_b float32 field inside
 * `nodewise` (row-major, first graph's nodes as rows).  Buffers are valid only
 * during the call.  Return 0 to continue, nonzero to abort the stream. */
typedef int (*mgk_nodewise_sink)(void* user, int64_t npairs, const int32_t* a, const int32_t* b, const double* value,
                                 const int32_t* iters, const uint8_t* conv, const int64_t* offsets,
                                 const float* nodewise);

/* Nodal similarity of every Gram pair (a <= b) of this rank's shard (pair ids
 * congruent to rank modulo world, as mgk_gram_shard), streamed to `sink` in
 * chunks of at most chunk_bytes of float32 field (the per-pair KernelResult.
 * nodewise of solver.py:212-246 for all N(N+1)/2 pairs of gram.py:57-95; the
 * full field of a 10k-graph dataset exceeds device memory, so it is produced
 * and handed off chunk by chunk through pinned host buffers).  Reports the
 * pairs and floats streamed. */
int mgk_gram_nodewise(mgk_ctx* ctx, int rank, int world, double tol, int64_t max_iter, int64_t chunk_bytes,
                      mgk_nodewise_sink sink, void* user, int64_t* npairs_out, int64_t* nfloats_out);

/* Single pair convenience wrapper of mgk_pairs (mgkbind.kernel, __init__.py:41-67). */
int mgk_kernel(mgk_ctx* ctx, int32_t a, int32_t b, double tol, int64_t max_iter, double* value, double* nodewise,
               int32_t* iters, double* residual, uint8_t* conv);

/* Device graph ingestion: spatial_graph (graphio.py:211-240)
 * for N point clouds at once on CUDA device `device`.  node_off[N+1] offsets
 * into points[sum n * dim] (dim 2 or 3, float64, row-major).  Every pair i < j
 * with distance d < cutoff becomes an edge (i, j lexicographic, local ids),
 * w = (1 - (d/cutoff)^2)^2, label d -- edges and d bit-identical to the
 * reference's float64 numpy evaluation, w within 1e-13 relative (numpy squares with libm pow).  Writes edge_off[N+1]; call with the four edge arrays NULL
 * to size them, then again with buffers of edge_off[N] entries. */
int mgk_spatial_edges(int device, int32_t N, const int64_t* node_off, int dim, const double* points, double cutoff,
                      int64_t* edge_off, int32_t* ei, int32_t* ej, double* w, double* d);

/* Cost counters of the pair (a, b) after `applies` operator applications
 * (ProductOperator.counter_report, product.py:212-272, 423-436; the solver
 * applies the operator once per iteration, solver.py:98-99):
 * model = {E, F, X, r} (CostModel, costs.py:27-43; tile size 8),
 * thresholds = {sparse_min_max, sparse_max_max, dense_min}
 * (SelectionThresholds, product.py:38-53), force_dense = the reference's
 * force_dense_stream.  out = {flops, t1_load, t1_store, t2_load, t2_store,
 * tile_pairs}, summed from the device octiles' per-graph density histograms
 * (nonzeros per tile, non-empty tile rows). */
int mgk_counters(mgk_ctx* ctx, int32_t a, int32_t b, int64_t applies, const double* model,
                 const int32_t* thresholds, int force_dense, double* out);

/* Device time (ms, CUDA events on the solver stream) and the number of
 * kernel launches of the last solve call. */
int mgk_last_timing(mgk_ctx* ctx, double* solve_ms, int32_t* launches);

/* Benchmark support (not part of the reference interface): measured FP32
 * FFMA throughput (TFLOP/s) and MUFU ex2 throughput (T ops/s) of `device`,
 * the denominators of the roofline fractions bench.py reports. */
int mgk_bench_peaks(int device, double* fp32_tflops, double* ex2_tops);

/* Benchmark support: cumulative host->device and device->host payload bytes
 * moved by this process's libmgk calls (for end-to-end accounting). */
int mgk_transfer_bytes(int64_t* h2d, int64_t* d2h);

#ifdef __cplusplus
}
#endif
#endif /* MGK_H */
