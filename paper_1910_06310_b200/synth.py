"""Seeded synthetic datasets for the five BASELINE.json configurations.

Shapes follow SURVEY.md §8(d).  There is no network in this build, so every
dataset is generated from a fixed seed; the GPU path, the CPU oracle and the
reference (in the build container) all read the same graphs.

* ``config1`` -- 16 ER graphs (n 18..22, density 0.3), categorical node
  labels, scalar edge labels, q = 0.05 (reference test fixture shape,
  ``tests/conftest.py:7-25``).
* ``config2`` -- QM7-shaped molecules: n 4..23, 3-D self-avoiding chains of
  1.4 A steps, elements drawn {H .50, C .35, N .06, O .08, S .01}, edges by
  a 3 A cutoff with the reference's spatial weighting
  ``w = (1-(d/rc)^2)^2`` and distance labels (``graphio.py:211-240``).
* ``config3`` -- protein-sized C-alpha chains (n 200..600, 3.8 A steps,
  8 A contacts), node order shuffled so PBR has work.
* ``config4`` -- 3-D random geometric graphs, n 2000..5000, cutoff tuned
  to mean degree 4/8/16/32, shuffled.
* ``config5`` -- 10k mixed-size molecules (60% 4..23, 30% 24..64,
  10% 65..128).
"""

from __future__ import annotations

import numpy as np

from .graphs import LabeledGraph

ELEMENTS = np.array([1, 6, 7, 8, 16], dtype=np.int64)
ELEMENT_P = np.array([0.50, 0.35, 0.06, 0.08, 0.01])
PROTEIN_ELEMENTS = np.array([6, 7, 8, 16], dtype=np.int64)


def er_graph(rng, n, density=0.3, labeled=True, q=0.05):
    """Erdos-Renyi graph with the reference fixture's label/weight draws."""
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(len(iu)) < density
    ei, ej = iu[keep], ju[keep]
    w = rng.uniform(0.2, 2.0, size=len(ei))
    el = rng.uniform(0.0, 2.0, size=len(ei))
    nl = rng.integers(0, 3, size=n)
    return LabeledGraph.from_arrays(n, ei, ej, w, node_labels=nl if labeled else None,
                                    edge_labels=el if labeled else None, default_q=q)


def spatial_edges(points, cutoff):
    """Pairs closer than ``cutoff``; weight (1-(d/rc)^2)^2, label d."""
    diff = points[:, None, :] - points[None, :, :]
    dist = np.sqrt(np.sum(diff * diff, axis=-1))
    iu, ju = np.triu_indices(len(points), 1)
    d = dist[iu, ju]
    keep = d < cutoff
    d = d[keep]
    return iu[keep], ju[keep], (1.0 - (d / cutoff) ** 2) ** 2, d


def chain(rng, n, step, min_sep):
    """3-D self-avoiding random chain: unit steps scaled by ``step``; every
    new point keeps ``min_sep`` from all earlier non-adjacent points."""
    pts = np.zeros((n, 3))
    for k in range(1, n):
        for _ in range(64):
            v = rng.normal(size=3)
            cand = pts[k - 1] + step * v / np.linalg.norm(v)
            if k < 2 or np.min(np.linalg.norm(pts[: k - 1] - cand, axis=1)) >= min_sep:
                break
        pts[k] = cand
    return pts


def molecule(rng, n, cutoff=3.0, q=0.05):
    pts = chain(rng, n, 1.4, 0.8 * 1.4)
    ei, ej, w, d = spatial_edges(pts, cutoff)
    labels = rng.choice(ELEMENTS, size=n, p=ELEMENT_P)
    return LabeledGraph.from_arrays(n, ei, ej, w, node_labels=labels, edge_labels=d, default_q=q)


def protein(rng, n, q=0.05):
    pts = chain(rng, n, 3.8, 0.8 * 3.8)
    ei, ej, w, d = spatial_edges(pts, 8.0)
    labels = rng.choice(PROTEIN_ELEMENTS, size=n)
    g = LabeledGraph.from_arrays(n, ei, ej, w, node_labels=labels, edge_labels=d, default_q=q)
    return shuffle_nodes(rng, g)


def shuffle_nodes(rng, g: LabeledGraph) -> LabeledGraph:
    """Relabel nodes by a seeded permutation (input order for PBR to fix)."""
    n = g.node_count
    fwd = rng.permutation(n)
    inv = np.empty(n, dtype=np.int64)
    inv[fwd] = np.arange(n)
    a, b = fwd[g.edges_i], fwd[g.edges_j]
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    order = np.lexsort((hi, lo))
    return LabeledGraph(n, lo[order], hi[order], g.weights[order], g.start_prob[inv].copy(),
                        g.stop_prob[inv].copy(),
                        None if g.node_labels is None else g.node_labels[inv].copy(),
                        None if g.edge_labels is None else g.edge_labels[order].copy(), g.name)


def rgg(rng, n, mean_degree, q=0.05):
    """Random geometric graph in the unit cube with E[degree] = mean_degree."""
    from scipy.spatial import cKDTree

    r = (3.0 * mean_degree / (4.0 * np.pi * n)) ** (1.0 / 3.0)
    pts = rng.random((n, 3))
    pairs = cKDTree(pts).query_pairs(r, output_type="ndarray")
    ei, ej = pairs[:, 0], pairs[:, 1]
    d = np.linalg.norm(pts[ei] - pts[ej], axis=1)
    w = (1.0 - (d / r) ** 2) ** 2 + 1e-3
    g = LabeledGraph.from_arrays(n, ei, ej, w, edge_labels=d / r, default_q=q)
    return shuffle_nodes(rng, g)


def config1(seed=0):
    rng = np.random.default_rng(seed)
    return [er_graph(rng, int(rng.integers(18, 23))) for _ in range(16)]


def config2(count=7165, seed=7165):
    rng = np.random.default_rng(seed)
    return [molecule(rng, int(rng.integers(4, 24))) for _ in range(count)]


def config3(count=1000, seed=1000, n_lo=200, n_hi=600):
    rng = np.random.default_rng(seed)
    return [protein(rng, int(rng.integers(n_lo, n_hi + 1))) for _ in range(count)]


def config4(count=100, seed=100, n_lo=2000, n_hi=5000, degrees=(4, 8, 16, 32)):
    rng = np.random.default_rng(seed)
    per = max(count // len(degrees), 1)
    out = []
    for k in range(count):
        out.append(rgg(rng, int(rng.integers(n_lo, n_hi + 1)), degrees[min(k // per, len(degrees) - 1)]))
    return out


def config5(count=10000, seed=10000):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        u = rng.random()
        if u < 0.6:
            n = int(rng.integers(4, 24))
        elif u < 0.9:
            n = int(rng.integers(24, 65))
        else:
            n = int(rng.integers(65, 129))
        out.append(molecule(rng, n))
    return out


CONFIG_KERNELS = {
    1: ("delta:0.5", "se:1.0"),
    2: ("delta:0.5", "se:1.0"),
    3: ("delta:0.5", "se:1.0"),
    4: (None, None),
    5: ("delta:0.5", "se:1.0"),
}
