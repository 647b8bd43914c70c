"""Golden vectors that need the REAL reference at sizes where it is slow
(build container only; minutes on 8 cores):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_large.py [pbr|smallq]

* ``pbr_large.json``: reference ``pbr_reorder`` forward maps (seed 0, the seed
  ``bench.py`` uses) and post-reorder octile counts for shuffled config-3
  protein graphs of 300-600 nodes and config-4-shaped random geometric graphs
  scaled to <= 600 nodes (``reorder.py:361-404``; the
  reference recomputes an O(n k^2) gain matrix per move, 7-35 s per graph).
* ``smallq.json``: reference ``kernel()`` values / iterations / nodewise
  fields for unlabeled and kappa_e = 1 pairs at q in {5e-4, 5e-3} across the
  solver size classes (tiny n m <= 128, warp n <= 24, mid 25-200) -- the
  cases SURVEY.md §7 H1's Laplacian splitting exists for.

Inputs come from the repo's seeded synthesis (``synth.py``); outputs are
serialised with ``repr`` floats (exact round trip).
"""

from __future__ import annotations

import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, os.environ.get("MGK_REFERENCE_SRC", "/root/reference/pkg/src"))

import mgksolver as ref  # noqa: E402  (the reference)

from make_golden import gjson, random_graph, to_ref  # noqa: E402
from paper_1910_06310_b200 import synth  # noqa: E402  (input synthesis only)


def pbr_inputs():
    """(name, graph) pairs: shuffled proteins spread over 300..600 nodes, scaled RGG density buckets."""
    out = []
    rng = np.random.default_rng(1000)
    for n in (300, 360, 420, 480, 540, 600):
        out.append((f"protein{n}", synth.protein(rng, n)))
    rng = np.random.default_rng(100)
    for n, deg in ((400, 4), (500, 8), (550, 16), (600, 32)):
        out.append((f"rgg{n}_d{deg}", synth.rgg(rng, n, deg)))
    return out


def _pbr_one(args):
    name, g = args
    rg = to_ref(g)
    perm = ref.pbr_reorder(rg, seed=0)
    return {
        "name": name,
        "graph": gjson(rg),
        "seed": 0,
        "forward": perm.forward.tolist(),
        "tiles_before": ref.build_tiles(rg).tile_count,
        "tiles_after": ref.build_tiles(ref.apply_permutation(rg, perm)).tile_count,
        "objective": int(ref.objective(rg, perm)),
        "rcm": ref.rcm_reorder(rg).forward.tolist(),
    }


def make_pbr():
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        recs = list(ex.map(_pbr_one, pbr_inputs()))
    for r in recs:
        print("pbr", r["name"], r["graph"]["n"], r["tiles_before"], "->", r["tiles_after"], flush=True)
    return recs


def order_cases():
    """RCM (reorder.py:412-442) on small / disconnected / edgeless graphs and Morton (reorder.py:445-478)
    on 2-D and 3-D point sets, including duplicate points and a degenerate (flat) axis."""
    out = {"rcm": [], "morton": []}
    rng = np.random.default_rng(412)
    graphs = [("edgeless5", ref.LabeledGraph.from_edges(5, [])),
              ("path_rev", ref.LabeledGraph.from_edges(6, [(4, 5, 1.0), (0, 5, 1.0), (1, 2, 1.0), (2, 3, 1.0)])),
              ("two_comp", ref.LabeledGraph.from_edges(9, [(0, 3, 1.0), (3, 6, 1.0), (1, 4, 1.0), (4, 7, 1.0),
                                                          (7, 8, 1.0), (2, 8, 1.0)])),
              ("star", ref.LabeledGraph.from_edges(7, [(3, k, 1.0) for k in range(7) if k != 3]))]
    for k in range(8):
        graphs.append((f"er{k}", random_graph(rng, int(rng.integers(2, 80)), density=float(rng.uniform(0.02, 0.3)))))
    graphs.append(("nws96", ref.gen_nws(96, 3, 0.1, 7)))
    graphs.append(("ba64", ref.gen_ba(64, 3, 5)))
    for name, g in graphs:
        out["rcm"].append({"name": name, "graph": gjson(g), "forward": ref.rcm_reorder(g).forward.tolist()})
    for k, (n, dim) in enumerate(((1, 3), (7, 2), (50, 3), (200, 3), (333, 2))):
        pts = rng.normal(size=(n, dim)) * rng.uniform(0.1, 10.0)
        if n > 10:
            pts[5] = pts[3]  # duplicate point: ties broken by index
        if k == 3:
            pts[:, 1] = 2.5  # flat axis (span 0 -> 1)
        out["morton"].append({"name": f"pts{k}", "points": pts.tolist(),
                              "keys": __import__("mgksolver.reorder", fromlist=["x"]).morton_keys(pts).tolist(),
                              "forward": ref.morton_reorder(pts).forward.tolist()})
    return out


def unlabeled(g):
    """Strip the labels (unlabeled mode, product.py:153-161)."""
    return ref.LabeledGraph.from_edges(g.node_count,
                                       list(zip(g.edges_i.tolist(), g.edges_j.tolist(), g.weights.tolist())),
                                       start_prob=g.start_prob, stop_prob=g.stop_prob)


def with_q(g, q):
    return ref.LabeledGraph.from_edges(g.node_count,
                                       list(zip(g.edges_i.tolist(), g.edges_j.tolist(), g.weights.tolist())),
                                       node_labels=g.node_labels, edge_labels=g.edge_labels,
                                       start_prob=g.start_prob, stop_prob=np.full(g.node_count, q))


def smallq_cases():
    cases = []
    mrng = np.random.default_rng(77)
    rng = np.random.default_rng(78)
    for q in (5e-4, 5e-3):
        # tiny (n m <= 128), warp (n, m <= 24), mid (25-200 nodes, panel / block classes)
        for k, (na, nb) in enumerate(((4, 9), (11, 11), (6, 20), (15, 23), (23, 23), (40, 12), (60, 30),
                                      (120, 90))):
            if na <= 24 and nb <= 24:
                ga = to_ref(synth.molecule(mrng, na, q=q))
                gb = to_ref(synth.molecule(mrng, nb, q=q))
            else:
                ga = random_graph(rng, na, density=min(0.3, 6.0 / na), labeled=True, q_range=(q, q))
                gb = random_graph(rng, nb, density=min(0.3, 6.0 / nb), labeled=True, q_range=(q, q))
            # unlabeled (no edge labels, delta vertex kernel on the element labels where present)
            cases.append((f"u_q{q:g}_{k}", unlabeled(ga), unlabeled(gb), None, None))
            # labeled graphs with kappa_e = const1 (kappa_e = 1 on every edge pair) and a delta vertex kernel
            cases.append((f"k1_q{q:g}_{k}", with_q(ga, q), with_q(gb, q), "delta:0.5", "const1"))
        # a self pair (Gram diagonal) and a complete graph (dense octiles) at each q
        gs = to_ref(synth.molecule(mrng, 19, q=q))
        cases.append((f"u_q{q:g}_self", unlabeled(gs), unlabeled(gs), None, None))
        kn = ref.LabeledGraph.from_edges(20, [(i, j, 0.5 + 0.01 * (i + j)) for i in range(20)
                                              for j in range(i + 1, 20)], stop_prob=np.full(20, q))
        cases.append((f"u_q{q:g}_k20x{9}", kn, unlabeled(to_ref(synth.molecule(mrng, 9, q=q))), None, None))
    return cases


def _kernel_one(args):
    name, ga, gb, vs, es = args
    vk = None if vs is None else ref.kernel_from_spec(vs).with_role("vertex")
    ek = None if es is None else ref.kernel_from_spec(es).with_role("edge")
    out = []
    for tol in (1e-6, 1e-8):
        res = ref.kernel(ga, gb, vk, ek, ref.SolverConfig(tolerance=tol))
        out.append({"name": name, "a": gjson(ga), "b": gjson(gb), "vkernel": vs, "ekernel": es, "reorder": None,
                    "tol": tol, "value": res.value, "iterations": res.iterations, "residual": res.final_residual,
                    "converged": res.converged, "nodewise": res.nodewise.tolist()})
    return out


def make_smallq():
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        recs = [r for rs in ex.map(_kernel_one, smallq_cases()) for r in rs]
    for r in recs:
        print("smallq", r["name"], r["tol"], r["iterations"], flush=True)
    return recs


if __name__ == "__main__":
    what = sys.argv[1:] or ["pbr", "smallq", "order"]
    if "order" in what:
        (HERE / "order.json").write_text(json.dumps(order_cases()))
    if "pbr" in what:
        (HERE / "pbr_large.json").write_text(json.dumps(make_pbr()))
    if "smallq" in what:
        (HERE / "smallq.json").write_text(json.dumps(make_smallq()))
