"""The CPU oracle (oracle/mgk_oracle.py) against the reference's own outputs.

Golden vectors were produced by the real reference (tests/golden/make_golden.py);
these tests pin the oracle before it is trusted as the checker of the CUDA path.
"""
import numpy as np
import pytest

from conftest import graph_from_json, load_golden
from oracle import mgk_oracle as O


def test_splitmix_known_answers(golden_rng):
    # reference tests/test_generators.py:11-18
    r = O.SplitMix64(0)
    assert [r.next_u64() for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    for seed, rec in golden_rng.items():
        r = O.SplitMix64(int(seed))
        assert [hex(r.next_u64()) for _ in range(8)] == rec["u64"]
        assert [O.SplitMix64(int(seed)).randint(k) for k in (1, 2, 3, 7, 1000, 2**40 + 3)] == rec["randint"]
        assert [O.SplitMix64(int(seed)).random()] == rec["random"]
        xs = list(range(20))
        O.SplitMix64(int(seed)).shuffle(xs)
        assert xs == rec["shuffle20"]


def test_degree_and_tiles_bit_exact(golden_structure):
    for rec in golden_structure:
        g = graph_from_json(rec["graph"])
        assert O.degree_vector(g).tolist() == rec["degree"], rec["name"]
        t = O.build_octiles(g)
        assert t.rows.tolist() == rec["tiles"]["rows"], rec["name"]
        assert t.cols.tolist() == rec["tiles"]["cols"], rec["name"]
        assert [hex(b) for b in t.bitmaps] == rec["tiles"]["bitmaps"], rec["name"]
        assert t.values.tolist() == rec["tiles"]["values"], rec["name"]
        assert t.dump() == rec["tiles"]["dump"], rec["name"]


def test_known_tile_answers():
    # reference tests/test_tiles.py:33-47, 151-156
    from paper_1910_06310_b200.graphs import LabeledGraph

    k8 = LabeledGraph.from_edges(8, [(i, j, 1.0) for i in range(8) for j in range(i + 1, 8)])
    t = O.build_octiles(k8)
    assert t.count == 1 and t.bitmaps[0] == (2**64 - 1) - sum(1 << (9 * k) for k in range(8))
    t = O.build_octiles(LabeledGraph.from_edges(16, [(0, 9, 1.0)]))
    assert list(zip(t.rows.tolist(), t.cols.tolist())) == [(0, 1), (1, 0)]
    assert t.bitmaps == [1 << 1, 1 << 8]
    assert t.dump().splitlines()[0] == "0 1 0x0000000000000002 1"


def test_pbr_bit_exact(golden_structure):
    for rec in golden_structure:
        g = graph_from_json(rec["graph"])
        if g.node_count > 130:
            continue  # the python restatement is O(n k^2) per move; large cases run in the slow test
        for seed, fwd in rec["pbr"].items():
            assert O.pbr_reorder(g, int(seed)).tolist() == fwd, (rec["name"], seed)
        if "pbr_t2" in rec:
            assert O.pbr_reorder(g, 0, t=2).tolist() == rec["pbr_t2"]


@pytest.mark.slow
def test_pbr_bit_exact_large(golden_structure):
    for rec in golden_structure:
        g = graph_from_json(rec["graph"])
        if g.node_count <= 130:
            continue
        for seed, fwd in rec["pbr"].items():
            assert O.pbr_reorder(g, int(seed)).tolist() == fwd, (rec["name"], seed)


def test_kernel_values_iterations(golden_kernels):
    for rec in golden_kernels:
        ga, gb = graph_from_json(rec["a"]), graph_from_json(rec["b"])
        res = O.kernel(ga, gb, rec["vkernel"], rec["ekernel"], tol=rec["tol"], reorder=rec["reorder"])
        assert res.iterations == rec["iterations"], rec["name"]
        assert res.converged == rec["converged"]
        assert abs(res.value - rec["value"]) <= 1e-12 * abs(rec["value"]), rec["name"]
        assert np.allclose(res.nodewise, np.asarray(rec["nodewise"]), rtol=1e-10, atol=1e-14), rec["name"]


def test_composite_kernels_golden():
    """ProductComposite / RConvolution (basekernels.py:175-244) restated in the oracle, pinned
    against the reference kernel() on vector-labelled pairs (tests/golden/composite.json)."""
    from conftest import load_golden

    for rec in load_golden("composite.json"):
        ga, gb = graph_from_json(rec["a"]), graph_from_json(rec["b"])
        res = O.kernel(ga, gb, rec["vkernel"], rec["ekernel"], tol=rec["tol"])
        assert res.iterations == rec["iterations"], rec["name"]
        assert abs(res.value - rec["value"]) <= 1e-11 * abs(rec["value"]), rec["name"]
        assert np.allclose(res.nodewise, np.asarray(rec["nodewise"]), rtol=1e-9, atol=1e-14), rec["name"]


def test_closed_forms():
    # reference tests/test_solver.py:38-69
    from paper_1910_06310_b200.graphs import LabeledGraph

    a = LabeledGraph.from_edges(1, [], node_labels=np.array([0]), stop_prob=[0.3], start_prob=[1.0])
    b = LabeledGraph.from_edges(1, [], node_labels=np.array([1]), stop_prob=[0.3], start_prob=[1.0])
    r = O.kernel(a, b, "delta:0.8")
    assert r.value == pytest.approx(0.072, rel=1e-14) and r.iterations == 1
    p2 = LabeledGraph.from_edges(2, [(0, 1, 1.0)], stop_prob=[0.5, 0.5])
    assert O.kernel(p2, p2).value == pytest.approx(0.45, rel=1e-10)


def test_operator_known_answers():
    # reference tests/test_product.py:50-58 (diagonal cache) and :88-94 (apply)
    from paper_1910_06310_b200.graphs import LabeledGraph

    a = LabeledGraph.from_edges(1, [], node_labels=np.array([0]), stop_prob=[0.3], start_prob=[1.0])
    b = LabeledGraph.from_edges(1, [], node_labels=np.array([1]), stop_prob=[0.3], start_prob=[1.0])
    sn = O.ProductSystem(a, b, ("delta", 0.8))
    assert np.allclose(sn.diag, [0.3 * 0.3 / 0.8], rtol=0, atol=1e-16)
    assert np.allclose(sn.diag * np.array([2.0]), [0.225])
    p2 = LabeledGraph.from_edges(2, [(0, 1, 1.0)], stop_prob=[0.5, 0.5])
    op = O.ProductSystem(p2, p2)
    assert np.array_equal(op.diag, np.full(4, 2.25))
    assert np.allclose(op.offdiag(np.ones(4)), np.ones(4), rtol=0, atol=0)
    assert np.allclose(op.apply(np.ones(4)), np.full(4, 1.25), rtol=1e-15)


def test_pbr_known_answers():
    # reference tests/test_reorder.py:38-65: objective examples, 4-node optimum, block-diagonal 0
    from paper_1910_06310_b200.graphs import LabeledGraph

    assert O.pair_objective(LabeledGraph.from_edges(6, []), np.arange(6) // 2) == 0
    four = LabeledGraph.from_edges(4, [(0, 2, 1.0), (1, 3, 1.0)])
    assert O.pair_objective(four, np.arange(4) // 2) == 1
    assert O.pair_objective(four, O.pbr_reorder(four, 0, t=2) // 2) == 0
    k24 = LabeledGraph.from_edges(24, [(i, j, 1.0) for i in range(24) for j in range(i + 1, 24)])
    assert O.pair_objective(k24, np.arange(24) // 8) == 3
    cl = [(i, j, 1.0) for i in range(8) for j in range(i + 1, 8)]
    cl += [(i, j, 1.0) for i in range(8, 16) for j in range(i + 1, 16)]
    blocks = LabeledGraph.from_edges(16, cl)
    assert O.pair_objective(blocks, O.pbr_reorder(blocks, 1) // 8) == 0


def test_direct_solve_agrees():
    # the oracle's COO product against a dense solve (reference test_solver.py:75-88 triad)
    rng = np.random.default_rng(5)
    from paper_1910_06310_b200 import synth

    for _ in range(5):
        ga, gb = synth.er_graph(rng, 9), synth.er_graph(rng, 7)
        sysm = O.ProductSystem(ga, gb, ("delta", 0.5), ("se", 1.0))
        qa, qb = ga.stop_prob, gb.stop_prob
        b = np.outer(sysm.d_a * qa, sysm.d_b * qb).ravel()
        x = np.linalg.solve(sysm.dense(), b)
        val = float(np.outer(ga.start_prob, gb.start_prob).ravel() @ x)
        assert O.solve_pcg(ga, gb, ("delta", 0.5), ("se", 1.0)).value == pytest.approx(val, rel=1e-9)


def test_gram_config1(golden_gram):
    rec = golden_gram["config1"]
    graphs = [graph_from_json(g) for g in rec["graphs"]]
    K, it, conv = O.gram(graphs, rec["vkernel"], rec["ekernel"])
    assert np.allclose(K, np.asarray(rec["matrix"]), rtol=1e-12, atol=0)
    assert it.tolist() == rec["iterations"]
    assert np.allclose(O.normalize_gram(K), np.asarray(rec["normalized"]), rtol=1e-12)
    order = O.schedule_pairs([g.node_count for g in graphs], [2 * g.edge_count for g in graphs])
    assert [list(p) for p in order] == rec["order"]


def test_schedule_golden(golden_gram):
    s = golden_gram["schedule"]
    assert [list(p) for p in O.schedule_pairs([4, 4, 4], [6, 6, 6])] == s["uniform"]
    assert [list(p) for p in O.schedule_pairs([4, 100, 4, 4], [6, 2000, 6, 6])] == s["giant"]
    assert [list(p) for p in O.schedule_pairs([10, 20, 10, 7, 3], [30, 120, 20, 14, 2])] == s["mixed"]


def test_spatial_edges_golden():
    """graphio.spatial_graph (graphio.py:211-240) restated, bit-exact vs the reference on seeded clouds."""
    from conftest import load_golden

    for rec in load_golden("spatial.json"):
        ei, ej, w, d = O.spatial_edges(rec["points"], rec["cutoff"])
        assert ei.tolist() == rec["ei"] and ej.tolist() == rec["ej"]
        assert w.tolist() == rec["w"] and d.tolist() == rec["d"]


def test_rcm_morton_oracle_golden():
    """Oracle RCM / Morton restatements against the reference (order.json; the pbr_large.json graphs
    carry the reference's rcm_reorder forward maps of 300-600-node proteins and RGGs)."""
    order = load_golden("order.json")
    for rec in order["rcm"]:
        g = graph_from_json(rec["graph"])
        assert O.rcm_order(g).tolist() == rec["forward"], rec["name"]
    for rec in load_golden("pbr_large.json"):
        assert O.rcm_order(graph_from_json(rec["graph"])).tolist() == rec["rcm"], rec["name"]
    for rec in order["morton"]:
        pts = np.asarray(rec["points"], dtype=np.float64)
        assert O.morton_keys(pts).tolist() == rec["keys"], rec["name"]
        assert O.morton_order(pts).tolist() == rec["forward"], rec["name"]


def test_pbr_large_oracle_golden():
    """Oracle PBR at config-3 sizes (300-600 nodes) against the reference's forward maps -- the two
    smallest graphs (the oracle is pure Python; the GPU test covers all ten on the device)."""
    recs = sorted(load_golden("pbr_large.json"), key=lambda r: r["graph"]["n"])[:2]
    for rec in recs:
        g = graph_from_json(rec["graph"])
        assert O.pbr_reorder(g, seed=rec["seed"]).tolist() == rec["forward"], rec["name"]
