"""Device node orderings against the REAL reference's permutations (bit-exact):

* PBR at config-3 sizes (300-600-node shuffled proteins, RGG density buckets; tests/golden/pbr_large.json,
  make_golden_large.py) -- forward maps and post-reorder octile counts (BASELINE.md
  "bit-exact up to n <= 600");
* RCM (reorder.py:412-443) and Morton (reorder.py:448-478) on the device (csrc/order.cu), on
  edgeless / disconnected / star / random / small-world / scale-free graphs, duplicate points and a
  flat axis (order.json), and on the ten large graphs;
* kernel(reorder=...) for every method leaves values within 1e-5 and maps the nodewise field back to
  the input order (solver.py:236-246).
"""
import numpy as np
import pytest

from conftest import graph_from_json, load_golden
from oracle import mgk_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mgk():
    import paper_1910_06310_b200 as m
    from paper_1910_06310_b200 import native

    native.load()
    return m


def test_pbr_large_bit_exact(mgk):
    recs = load_golden("pbr_large.json")
    graphs = [graph_from_json(r["graph"]) for r in recs]
    perms = mgk.pbr_reorder_many(graphs, seed=0)
    for rec, g, perm in zip(recs, graphs, perms):
        assert perm.forward.tolist() == rec["forward"], rec["name"]
        assert mgk.build_tiles(mgk.apply_permutation(g, perm)).tile_count == rec["tiles_after"], rec["name"]
        assert mgk.build_tiles(g).tile_count == rec["tiles_before"], rec["name"]


def test_rcm_bit_exact(mgk):
    recs = load_golden("order.json")["rcm"]
    graphs = [graph_from_json(r["graph"]) for r in recs]
    for rec, perm in zip(recs, mgk.rcm_reorder_many(graphs)):  # one launch, one CTA per graph
        assert perm.forward.tolist() == rec["forward"], rec["name"]
    for rec in recs[:3]:
        assert mgk.rcm_reorder(graph_from_json(rec["graph"])).forward.tolist() == rec["forward"]
    big = load_golden("pbr_large.json")
    for rec, perm in zip(big, mgk.rcm_reorder_many([graph_from_json(r["graph"]) for r in big])):
        assert perm.forward.tolist() == rec["rcm"], rec["name"]


def test_rcm_random_graphs_vs_oracle(mgk):
    """Seeded random graphs of 1-3000 nodes (isolated nodes, many components, hubs) against the pinned
    oracle restatement."""
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(443)
    graphs = []
    for n in (1, 2, 9, 40, 130, 700, 3000):
        graphs.append(synth.er_graph(rng, n, density=min(0.3, 4.0 / n), labeled=False))
        graphs.append(synth.rgg(rng, n, 6) if n >= 40 else synth.er_graph(rng, n, 0.5, labeled=False))
    perms = mgk.rcm_reorder_many(graphs)
    for g, perm in zip(graphs, perms):
        assert perm.forward.tolist() == O.rcm_order(g).tolist(), g.node_count


def test_morton_bit_exact(mgk):
    for rec in load_golden("order.json")["morton"]:
        pts = np.asarray(rec["points"], dtype=np.float64)
        assert mgk.morton_reorder(pts).forward.tolist() == rec["forward"], rec["name"]
    rng = np.random.default_rng(471)
    for n, dim in ((1000, 3), (4000, 2), (2500, 3)):
        pts = rng.normal(size=(n, dim)) * 10.0 ** rng.uniform(-3, 3)
        pts[n // 2] = pts[n // 3]
        assert mgk.morton_reorder(pts).forward.tolist() == O.morton_order(pts).tolist()


def test_kernel_reorder_methods(mgk):
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(9)
    pts_a, pts_b = rng.normal(size=(30, 3)), rng.normal(size=(27, 3))
    ga, gb = synth.protein(rng, 30), synth.protein(rng, 27)
    # Morton needs coordinate node labels: the point clouds serve as vector node labels
    ca = mgk.LabeledGraph.from_arrays(30, ga.edges_i, ga.edges_j, ga.weights, node_labels=pts_a,
                                      edge_labels=ga.edge_labels)
    cb = mgk.LabeledGraph.from_arrays(27, gb.edges_i, gb.edges_j, gb.weights, node_labels=pts_b,
                                      edge_labels=gb.edge_labels)
    o = O.solve_pcg(ca, cb, None, ("se", 1.0))
    for method in ("none", "pbr", "rcm", "morton"):
        r = mgk.kernel(ca, cb, None, "se:1.0", reorder=method)
        assert abs(r.value - o.value) <= 1e-5 * abs(o.value), method
        assert abs(r.iterations - o.iterations) <= 1, method
        assert np.max(np.abs(r.nodewise - o.nodewise)) <= 1e-5 * np.max(np.abs(o.nodewise)), method
    with pytest.raises(ValueError, match="2D/3D coordinate"):
        mgk.kernel(ga, gb, None, "se:1.0", reorder="morton")
    with pytest.raises(ValueError, match="unknown reorder"):
        mgk.kernel(ga, gb, None, "se:1.0", reorder="spectral")


def test_kernel_counters_reference_golden(mgk):
    """KernelResult.counters (product.py:212-272, 423-436) from the device octile density histograms
    (mgk_counters) equal the reference's per-apply totals exactly: default labeled / unlabeled models,
    a custom CostModel + SelectionThresholds, force_dense_stream and a PBR-reordered pair."""
    for rec in load_golden("counters.json")["kernels"]:
        ga, gb = graph_from_json(rec["a"]), graph_from_json(rec["b"])
        opt = dict(rec["options"])
        ops = {}
        if "cost_model" in opt:
            ops["cost_model"] = mgk.CostModel(**opt["cost_model"])
        if "thresholds" in opt:
            ops["thresholds"] = mgk.SelectionThresholds(**opt["thresholds"])
        if opt.get("force_dense_stream"):
            ops["force_dense_stream"] = True
        r = mgk.kernel(ga, gb, rec["vkernel"], rec["ekernel"], mgk.SolverConfig(tolerance=rec["tol"]),
                       reorder=rec["reorder"], operator_options=ops or None)
        ref = rec["counters"]
        assert abs(r.iterations - rec["iterations"]) <= 1, rec["name"]
        for k in ("flops", "t1_load", "t1_store", "t2_load", "t2_store", "tile_pairs"):
            assert getattr(r.counters, k) / r.iterations == ref[k] / rec["iterations"], (rec["name"], k)
        if r.iterations == rec["iterations"]:
            assert r.counters.ai1 == ref["ai1"] and r.counters.ai2 == ref["ai2"], rec["name"]
    with pytest.raises(TypeError, match="unexpected keyword"):
        mgk.kernel(ga, gb, None, None, operator_options={"bogus": 1})


def test_reference_graph_files_kernel(mgk):
    """Graphs loaded from files the reference wrote give the reference's kernel value and nodewise CSV."""
    import json

    from conftest import GOLDEN

    files = GOLDEN / "files"
    index = json.loads((files / "index.json").read_text())
    ga, gb = mgk.load_graph(files / "cat.json"), mgk.load_graph(files / "cat.json")
    r = mgk.kernel(ga, gb, mgk.KroneckerDelta(0.5), mgk.SquareExponential(1.0))
    assert abs(r.value - index["nodewise_value"]) <= 1e-5 * abs(index["nodewise_value"])
    ref = mgk.load_nodewise_csv(files / "nodewise.csv")
    assert np.max(np.abs(r.nodewise - ref)) <= 1e-5 * np.max(np.abs(ref))
