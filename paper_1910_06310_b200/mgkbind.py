"""Array bindings mirroring the reference ``mgkbind`` package
(pkg/bindings/src/mgkbind/__init__.py:41-117, marshal.py:30-72).

Where the reference marshals graphs to JSON files and runs the solver CLI in
a subprocess (marshal.py:150-155), these bindings hand plain arrays to
libmgk through its C-ABI (include/mgk.h) in-process; the signatures, option
names and return shapes are the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .gram import compute_gram, normalize_gram, load_gram_binary as read_gram_binary
from .graphs import LabeledGraph
from .solver import SolverConfig, kernel as _kernel

__all__ = ["BoundGraph", "SolverError", "kernel", "gram", "read_gram_binary"]


class SolverError(RuntimeError):
    """The solver rejected the input; carries the core's message (marshal.py:26-28)."""


@dataclass
class BoundGraph:
    """Graph as plain arrays: dense symmetric matrix or (i, j, w) triplets (marshal.py:30-72)."""

    adjacency: object
    node_labels: Optional[np.ndarray] = None
    edge_labels: Optional[np.ndarray] = None
    start_prob: Optional[np.ndarray] = None
    stop_prob: Optional[np.ndarray] = None
    name: str = ""

    def edge_arrays(self):
        adj = self.adjacency
        if isinstance(adj, tuple) and len(adj) == 3:
            i, j, w = (np.asarray(x) for x in adj)
            labels = None if self.edge_labels is None else np.asarray(self.edge_labels)
            n = int(max(i.max(initial=-1), j.max(initial=-1))) + 1
            if self.node_labels is not None:
                n = max(n, len(self.node_labels))
            if self.stop_prob is not None:
                n = max(n, len(self.stop_prob))
            return n, i, j, w, labels
        dense = np.asarray(adj, dtype=np.float64)
        if dense.ndim != 2 or dense.shape[0] != dense.shape[1]:
            raise ValueError("dense adjacency must be square")
        if not np.array_equal(dense, dense.T):
            raise ValueError("dense adjacency must be symmetric")
        i, j = np.nonzero(np.triu(dense, k=1))
        labels = None
        if self.edge_labels is not None:
            lm = np.asarray(self.edge_labels)
            if lm.shape[:2] != dense.shape:
                raise ValueError("dense edge labels must mirror the adjacency shape")
            labels = lm[i, j]
        return dense.shape[0], i, j, dense[i, j], labels


def _to_graph(g: BoundGraph, q: float | None, unlabeled: bool) -> LabeledGraph:
    n, i, j, w, el = g.edge_arrays()
    kw = {}
    if q is not None and g.stop_prob is None:
        kw["default_q"] = float(q)
    return LabeledGraph.from_arrays(
        n, i, j, w,
        node_labels=None if unlabeled else g.node_labels,
        edge_labels=None if unlabeled else el,
        start_prob=g.start_prob, stop_prob=g.stop_prob, name=g.name, **kw)


def _opts(options: dict):
    known = {"vkernel", "ekernel", "q", "tol", "reorder", "unlabeled"}
    bad = set(options) - known
    if bad:
        raise TypeError(f"unknown option(s) {sorted(bad)}")
    unl = bool(options.get("unlabeled"))
    vk = None if unl else options.get("vkernel")
    ek = None if unl else options.get("ekernel")
    cfg = SolverConfig(tolerance=float(options["tol"])) if options.get("tol") is not None else SolverConfig()
    return vk, ek, cfg, options.get("q"), unl, options.get("reorder")


def kernel(g_a: BoundGraph, g_b: BoundGraph, **options):
    """``(value, nodewise, {"iterations", "residual", "converged"})`` (__init__.py:41-67)."""
    vk, ek, cfg, q, unl, reo = _opts(options)
    try:
        ga, gb = _to_graph(g_a, q, unl), _to_graph(g_b, q, unl)
        res = _kernel(ga, gb, vk, ek, cfg, reorder=reo)
    except ValueError as exc:
        if "dense adjacency" in str(exc):
            raise
        raise SolverError(str(exc)) from exc
    diag = {"iterations": res.iterations, "residual": res.final_residual, "converged": res.converged}
    return res.value, res.nodewise, diag


def gram(graphs: list[BoundGraph], *, normalize: bool = False, workers: int = 1, deterministic: bool = True,
         **options):
    """``(matrix, converged)``; non-converged pairs are NaN (__init__.py:70-92)."""
    vk, ek, cfg, q, unl, _ = _opts(options)
    try:
        ds = [_to_graph(g, q, unl) for g in graphs]
        res = compute_gram(ds, vk, ek, cfg, workers=workers, deterministic=deterministic, normalize=normalize)
    except ValueError as exc:
        if "dense adjacency" in str(exc):
            raise
        raise SolverError(str(exc)) from exc
    m = res.matrix
    return m, ~np.isnan(m)
