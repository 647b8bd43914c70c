"""B200-native marginalized graph kernel solver (arXiv:1910.06310).

Drop-in for the reference ``mgksolver`` / ``mgkbind`` hot path: graph list
in, N x N kernel matrix or nodal similarity out, pluggable base kernels and
stopping probability q.  All numerics run in hand-written sm_100a CUDA behind
the C-ABI library ``libmgk.so`` (include/mgk.h); this package is the
host-side mirror of the reference interface.
"""

from .basekernels import (BaseKernel, CompactPolynomial, ConstantOne, KernelRangeError, KernelShapeError,
                          KroneckerDelta, ProductComposite, RConvolution, SquareExponential, kernel_from_spec)
from .costs import CostModel, CounterReport, PRIMITIVES, SelectionThresholds, predict_costs, select_tile_kernel
from .graphs import DEFAULT_STOP_PROB, LabeledGraph, ValidationReport, validate_graph
from .graphio import GraphFileError, PointCloud, load_edge_list, load_graph, save_graph, spatial_graph, spatial_graphs
from .gram import (GramResult, compute_gram, load_gram_binary, load_gram_csv, nodewise_gram, normalize_gram,
                   save_gram_binary, save_gram_csv, save_nodewise_csv, load_nodewise_csv, schedule_pairs,
                   stream_nodewise)
from .reorder import (Permutation, apply_permutation, morton_reorder, objective, partition_objective, pbr_reorder,
                      pbr_reorder_many, rcm_reorder, rcm_reorder_many)
from .solver import KernelResult, SolverConfig, kernel
from .tiles import TILE_SIZE, Tile, TiledMatrix, TileHistogram, build_tiles, dump_tiles, expand_tile, tile_histogram

__version__ = "0.1.0"


def degree_vector(g, device: int = 0):
    """graphs.py:202-214, computed by the device tile pipeline."""
    from . import native
    from .solver import _ctx_lock, context

    ctx = context(device)
    with _ctx_lock:
        ctx.upload(native.PackedDataset([g], with_labels=False))
        ctx.set_kernels(None, None)
        return ctx.degrees(0, g.node_count)
