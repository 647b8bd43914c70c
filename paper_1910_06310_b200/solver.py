"""Kernel evaluation facade mirroring ``mgksolver.solver`` (solver.py:39-259).

``kernel(g_a, g_b, ...)`` validates, optionally reorders both graphs with the
same seed, and solves the pair on the GPU through libmgk (octiles built on
the device, persistent PCG with the on-the-fly product matvec).  There is no
host numerical path.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import native
from .basekernels import (as_kernel, BaseKernel, CompactPolynomial, ConstantOne, KroneckerDelta, ProductComposite,
                          RConvolution, SquareExponential)
from .costs import CounterReport, SelectionThresholds, default_model
from .graphs import LabeledGraph, validate_graph

DEFAULT_VERTEX_FLOOR = 1e-12


@dataclass
class SolverConfig:
    """solver.py:39-52."""

    tolerance: float = 1e-10
    max_iterations: Optional[int] = None
    oracle_guard: int = 4096
    deterministic: bool = True
    v_min: float = DEFAULT_VERTEX_FLOOR

    def __post_init__(self):
        if self.tolerance <= 0:
            raise ValueError("tolerance must be positive")
        if self.max_iterations is not None and self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")


@dataclass
class KernelResult:
    """solver.py:54-62."""

    value: float
    nodewise: np.ndarray
    iterations: int
    final_residual: float
    converged: bool
    wall_time: float = 0.0
    counters: Optional[object] = field(default=None, repr=False)


def kernel_spec(k: BaseKernel | None) -> str | None:
    """Lower a kernel object to the device SPEC string (None stays None)."""
    if k is None:
        return None
    if isinstance(k, ConstantOne):
        return "const1"
    if isinstance(k, KroneckerDelta):
        return f"delta:{k.h!r}"
    if isinstance(k, SquareExponential):
        return f"se:{k.alpha!r}"
    if isinstance(k, CompactPolynomial):
        k.device_descriptor()  # raises for unsupported variants
        return "poly:" + ",".join(repr(c) for c in k.coeffs)
    if isinstance(k, (ProductComposite, RConvolution)):
        return k.spec()
    k.device_descriptor()
    raise NotImplementedError(f"{type(k).__name__} has no device lowering yet")


_ctx_lock = threading.Lock()
_contexts: dict[int, native.Context] = {}


def context(device: int = 0) -> native.Context:
    """Process-wide libmgk context per CUDA device."""
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = native.Context(device)
            _contexts[device] = ctx
        return ctx


_REORDER_METHODS = ("pbr", "rcm", "morton", "none", None)
# ProductOperator keywords (product.py:184-194).  Tiles, thresholds and cache limits only steer the
# reference's plan (value-transparent, tests/test_product.py:297-316); cost_model, thresholds and
# force_dense_stream shape the counters.
_OPERATOR_OPTIONS = ("tiles_a", "tiles_b", "cost_model", "thresholds", "force_dense_stream", "cache_limit_bytes")


def _edge_mode(g_a: LabeledGraph, g_b: LabeledGraph) -> str:
    """product.py:153-161 (label-presence mismatch raises at upload, native.PackedDataset)."""
    la = g_a.edge_labels is not None and g_a.edge_count > 0
    lb = g_b.edge_labels is not None and g_b.edge_count > 0
    return "labeled" if (la or lb) else "unlabeled"


def kernel(g_a: LabeledGraph, g_b: LabeledGraph, vertex_kernel=None, edge_kernel=None,
           cfg: SolverConfig | None = None, *, reorder: str | None = None, seed: int = 0,
           operator_options: dict | None = None, device: int = 0) -> KernelResult:
    """solver.py:212-246: validate -> [reorder] -> device solve -> un-permute nodewise."""
    cfg = cfg or SolverConfig()
    for name, g in (("first", g_a), ("second", g_b)):
        rep = validate_graph(g)
        if not rep.ok:
            raise ValueError(f"{name} graph invalid: " + "; ".join(rep.violations))
    if reorder not in _REORDER_METHODS:
        raise ValueError(f"unknown reorder method {reorder!r}")
    opts = dict(operator_options or {})
    for key in opts:
        if key not in _OPERATOR_OPTIONS:
            raise TypeError(f"ProductOperator.__init__() got an unexpected keyword argument {key!r}")
    vk = as_kernel(vertex_kernel, "vertex")
    ek = as_kernel(edge_kernel, "edge")
    mode = _edge_mode(g_a, g_b)
    model = opts.get("cost_model") or default_model(g_a, g_b, mode, ek)
    thresholds = opts.get("thresholds") or SelectionThresholds.for_mode(mode)
    start = time.perf_counter()
    ctx = context(device)
    with _ctx_lock:
        ctx.upload(native.PackedDataset([g_a, g_b]))
        ctx.set_kernels(kernel_spec(vk), kernel_spec(ek))
        ctx.set_vertex_floor(cfg.v_min)
        perm = None
        if reorder and reorder != "none":  # same method and seed for both graphs (solver.py:236-237)
            perm = ctx.reorder(reorder, seed, apply=True)
        val, it, res, cv, nw = ctx.pairs([0], [1], cfg.tolerance, cfg.max_iterations or 0, nodewise=True,
                                         sizes=[g_a.node_count, g_b.node_count])
        # one operator apply per iteration (solver.py:98-99); counters of the (reordered) device octiles
        cnt = ctx.counters(0, 1, int(it[0]), model, thresholds, bool(opts.get("force_dense_stream", False)))
    nodewise = nw.reshape(g_a.node_count, g_b.node_count)
    if perm is not None:
        fa, fb = perm[: g_a.node_count], perm[g_a.node_count:]
        nodewise = nodewise[fa[:, None], fb[None, :]]
    counters = CounterReport(flops=float(cnt[0]), t1_load=float(cnt[1]), t1_store=float(cnt[2]),
                             t2_load=float(cnt[3]), t2_store=float(cnt[4]), tile_pairs=int(cnt[5])).finalize()
    return KernelResult(value=float(val[0]), nodewise=nodewise, iterations=int(it[0]),
                        final_residual=float(res[0]), converged=bool(cv[0]),
                        wall_time=time.perf_counter() - start, counters=counters)
