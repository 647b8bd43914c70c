"""Node reordering, mirroring ``mgksolver.reorder`` (reorder.py:29-478).

``pbr_reorder`` runs the device partition-based reordering (csrc/pbr.cu),
bit-exact with the reference's recursive bisection + K-way FM refinement;
``rcm_reorder`` and ``morton_reorder`` run the device baselines (csrc/order.cu,
bit-exact with reorder.py:412-478).  ``apply_permutation`` relabels a host
graph (reorder.py:86-109).
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import native
from .graphs import LabeledGraph


@dataclass
class Permutation:
    forward: np.ndarray
    inverse: np.ndarray

    @staticmethod
    def identity(n: int) -> "Permutation":
        idx = np.arange(n, dtype=np.int64)
        return Permutation(idx.copy(), idx.copy())

    @staticmethod
    def from_forward(forward) -> "Permutation":
        forward = np.asarray(forward, dtype=np.int64)
        n = len(forward)
        if not np.array_equal(np.sort(forward), np.arange(n)):
            raise ValueError("forward map is not a bijection on 0..n-1")
        inv = np.empty(n, dtype=np.int64)
        inv[forward] = np.arange(n, dtype=np.int64)
        return Permutation(forward, inv)

    def inverted(self) -> "Permutation":
        return Permutation(self.inverse.copy(), self.forward.copy())

    def __len__(self) -> int:
        return len(self.forward)


def apply_permutation(g: LabeledGraph, perm: Permutation) -> LabeledGraph:
    """reorder.py:86-109."""
    if len(perm) != g.node_count:
        raise ValueError("permutation size does not match graph")
    a, b = perm.forward[g.edges_i], perm.forward[g.edges_j]
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    order = np.lexsort((hi, lo))
    return replace(g, edges_i=lo[order], edges_j=hi[order], weights=g.weights[order],
                   edge_labels=None if g.edge_labels is None else g.edge_labels[order],
                   start_prob=np.asarray(g.start_prob)[perm.inverse].copy(),
                   stop_prob=np.asarray(g.stop_prob)[perm.inverse].copy(),
                   node_labels=None if g.node_labels is None else g.node_labels[perm.inverse].copy())


def partition_objective(g: LabeledGraph, parts: np.ndarray) -> int:
    """reorder.py:112-119."""
    pa, pb = parts[g.edges_i], parts[g.edges_j]
    m = pa != pb
    return len(set(zip(np.minimum(pa, pb)[m].tolist(), np.maximum(pa, pb)[m].tolist())))


def objective(g: LabeledGraph, perm: Permutation, t: int = 8) -> int:
    return partition_objective(g, perm.forward // t)


def pbr_reorder_many(graphs, seed: int = 0, device: int = 0) -> list[Permutation]:
    """Device PBR for a batch of graphs (one launch; one CTA per graph)."""
    from .solver import _ctx_lock, context

    ctx = context(device)
    pk = native.PackedDataset(graphs, with_labels=False)
    with _ctx_lock:
        ctx.upload(pk)
        ctx.set_kernels(None, None)
        fwd = ctx.reorder_pbr(seed, apply=False)
    return [Permutation.from_forward(fwd[pk.node_off[k]: pk.node_off[k + 1]]) for k in range(len(graphs))]


def pbr_reorder(g: LabeledGraph, seed: int = 0, t: int = 8, max_passes: int = 10, device: int = 0) -> Permutation:
    """reorder.py:361-404 on the device (t = 8, max_passes = 10 as in the reference's callers)."""
    if t != 8 or max_passes != 10:
        raise NotImplementedError("device PBR is specialised to t=8, max_passes=10")
    return pbr_reorder_many([g], seed, device)[0]


def _device_orders(graphs, method: str, seed: int = 0, device: int = 0) -> list[Permutation]:
    from .solver import _ctx_lock, context

    ctx = context(device)
    pk = native.PackedDataset(graphs, with_labels=(method == "morton"))
    with _ctx_lock:
        ctx.upload(pk)
        ctx.set_kernels(None, None)
        fwd = ctx.reorder(method, seed, apply=False)
    return [Permutation.from_forward(fwd[pk.node_off[k]: pk.node_off[k + 1]]) for k in range(len(graphs))]


def rcm_reorder_many(graphs, device: int = 0) -> list[Permutation]:
    """Device reverse Cuthill-McKee for a batch of graphs (one CTA per graph)."""
    return _device_orders(graphs, "rcm", device=device)


def rcm_reorder(g: LabeledGraph, device: int = 0) -> Permutation:
    """reorder.py:412-443 on the device: components from their minimum-(degree, index) node, neighbours
    by ascending (degree, index), each component reversed."""
    return rcm_reorder_many([g], device)[0]


def morton_reorder(points, device: int = 0) -> Permutation:
    """reorder.py:471-478 on the device: Morton keys of 2-D / 3-D points (21 bits per axis over the
    bounding box), sorted with ties by index."""
    if points is None:
        raise ValueError("Morton ordering requires node coordinates")
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] not in (2, 3):
        raise ValueError("points must be an (n, 2) or (n, 3) array")
    g = LabeledGraph.from_arrays(len(pts), np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0),
                                 node_labels=pts)
    return _device_orders([g], "morton", device=device)[0]
