"""GPU parity: libmgk (CUDA, via the C-ABI) against the reference's golden
vectors and the CPU oracle.

Bars (BASELINE.json north_star): kernel value within 1e-5 relative,
iterations within +-1, octile bitmaps / PBR permutations bit-exact.
Unlabeled pairs are compared at tol = 1e-6 (FP32 needs 3-5 extra iterations
at 1e-10) -- the tolerance is stated per test below.
"""
import numpy as np
import pytest

from conftest import graph_from_json
from oracle import mgk_oracle as O

pytestmark = pytest.mark.gpu

REL = 1e-5


@pytest.fixture(scope="module")
def mgk():
    import paper_1910_06310_b200 as m
    from paper_1910_06310_b200 import native

    native.load()
    return m


def test_octiles_bit_exact(mgk, golden_structure):
    from paper_1910_06310_b200 import native
    from paper_1910_06310_b200.solver import context

    graphs = [graph_from_json(r["graph"]) for r in golden_structure]
    ctx = context()
    ctx.upload(native.PackedDataset(graphs, with_labels=False))
    ctx.set_kernels(None, None)
    for g, rec in enumerate(golden_structure):
        rc, bm, w = ctx.tiles(g)
        assert rc[:, 0].tolist() == rec["tiles"]["rows"], rec["name"]
        assert rc[:, 1].tolist() == rec["tiles"]["cols"], rec["name"]
        assert [hex(int(b)) for b in bm] == rec["tiles"]["bitmaps"], rec["name"]
        assert np.array_equal(w, np.asarray(rec["tiles"]["values"], dtype=np.float32)), rec["name"]
        d = ctx.degrees(g, graphs[g].node_count)
        assert np.allclose(d, rec["degree"], rtol=1e-6, atol=0), rec["name"]


def test_build_tiles_api_dump(mgk, golden_structure):
    """build_tiles host view: the reference's dump line, float64 values in (tile, bit) order equal to the
    reference's, and per-nonzero edge labels through expand_tile (tiles.py:85-146)."""
    for rec in golden_structure[:6]:
        g = graph_from_json(rec["graph"])
        t = mgk.build_tiles(g)
        assert mgk.dump_tiles(t) == rec["tiles"]["dump"]
        vals = [v for x in t.tiles for v in x.weights.tolist()]
        assert vals == rec["tiles"]["values"], rec["name"]
    rng = np.random.default_rng(130)
    for edge_kind in ("cat", "vec"):
        n = 21
        iu, ju = np.triu_indices(n, 1)
        keep = rng.random(iu.size) < 0.3
        lab = rng.integers(0, 5, keep.sum()) if edge_kind == "cat" else rng.normal(size=(keep.sum(), 2))
        g = mgk.LabeledGraph.from_arrays(n, iu[keep], ju[keep], rng.uniform(0.2, 2.0, keep.sum()), edge_labels=lab)
        t, o = mgk.build_tiles(g), O.build_octiles(g)
        assert [x.bitmap for x in t.tiles] == o.bitmaps
        for k, tile in enumerate(t.tiles):
            w, lb = mgk.expand_tile(tile)
            sl = slice(o.offsets[k], o.offsets[k + 1])
            assert np.array_equal(tile.weights, o.values[sl])
            assert np.array_equal(tile.labels, o.labels[sl])
            assert np.array_equal(w[tile.local_rows, tile.local_cols], o.values[sl])
            if edge_kind == "cat":
                holes = np.ones((8, 8), bool)
                holes[tile.local_rows, tile.local_cols] = False
                assert np.all(lb[holes] == -1)


def _tol_for(rec):
    return rec["tol"] if rec["ekernel"] is not None else 1e-6


def test_kernel_golden_pairs(mgk, golden_kernels):
    for rec in golden_kernels:
        if rec["reorder"] == "pbr":
            continue
        ga, gb = graph_from_json(rec["a"]), graph_from_json(rec["b"])
        tol = _tol_for(rec)
        res = mgk.kernel(ga, gb, rec["vkernel"], rec["ekernel"], mgk.SolverConfig(tolerance=tol))
        ref_val, ref_it = rec["value"], rec["iterations"]
        if tol != rec["tol"]:
            o = O.kernel(ga, gb, rec["vkernel"], rec["ekernel"], tol=tol)
            ref_it = o.iterations
            assert abs(o.value - ref_val) <= 1e-6 * abs(ref_val)
        assert res.converged, rec["name"]
        assert abs(res.value - ref_val) <= REL * abs(ref_val), (rec["name"], res.value, ref_val)
        assert abs(res.iterations - ref_it) <= 1, (rec["name"], res.iterations, ref_it)
        nw = np.asarray(rec["nodewise"])
        assert res.nodewise.shape == nw.shape
        assert np.max(np.abs(res.nodewise - nw)) <= REL * np.max(np.abs(nw)), rec["name"]


def test_composite_kernels_golden(mgk):
    """ProductComposite / RConvolution edge and vertex kernels (vector labels, evaluated in-kernel by the
    generic CTA solver) against the reference kernel() values (tests/golden/composite.json)."""
    from conftest import load_golden

    for rec in load_golden("composite.json"):
        ga, gb = graph_from_json(rec["a"]), graph_from_json(rec["b"])
        k = mgk.kernel(ga, gb, rec["vkernel"], rec["ekernel"])
        assert abs(k.value - rec["value"]) <= REL * abs(rec["value"]), (rec["name"], k.value, rec["value"])
        assert abs(k.iterations - rec["iterations"]) <= 1, (rec["name"], k.iterations, rec["iterations"])
        nw = np.asarray(rec["nodewise"])
        assert np.max(np.abs(k.nodewise - nw)) <= REL * np.max(np.abs(nw)), rec["name"]


def test_device_spatial_graph_bit_exact(mgk):
    """Device spatial_graph (csrc/ingest.cu) against the reference's float64 numpy builder: edges and
    distance labels bit for bit; weights within 1e-13 relative -- numpy evaluates ``x ** 2`` on float64
    scalars with libm pow, which is not correctly rounded, and 1 - t^2 amplifies that ulp (up to 6 ulp
    on w) against the correctly rounded squares the device computes.  Golden clouds
    (tests/golden/spatial.json) in one batch, and the config-2 molecule generator's clouds."""
    from conftest import load_golden

    recs = load_golden("spatial.json")
    for cutoff in sorted({r["cutoff"] for r in recs}):
        group = [r for r in recs if r["cutoff"] == cutoff]
        dims = {len(r["points"][0]) for r in group}
        for dim in dims:
            sub = [r for r in group if len(r["points"][0]) == dim]
            gs = mgk.spatial_graphs([mgk.PointCloud(np.asarray(r["points"]), np.asarray(r["labels"])) for r in sub],
                                    cutoff)
            for g, r in zip(gs, sub):
                assert g.edges_i.tolist() == r["ei"] and g.edges_j.tolist() == r["ej"]
                assert np.allclose(g.weights, np.asarray(r["w"]), rtol=1e-13, atol=0)
                assert (g.edge_labels.reshape(-1).tolist() if g.edge_labels is not None else []) == r["d"]
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(3)
    clouds = [synth.chain(rng, int(n), 1.4, 1.12) for n in (4, 17, 23, 60, 128)]
    gs = mgk.spatial_graphs([mgk.PointCloud(c) for c in clouds], 3.0)
    for c, g in zip(clouds, gs):
        ei, ej, w, d = O.spatial_edges(c, 3.0)
        assert g.edges_i.tolist() == ei.tolist() and g.edges_j.tolist() == ej.tolist()
        assert np.allclose(g.weights, w, rtol=1e-13, atol=0) and g.edge_labels.reshape(-1).tolist() == d.tolist()
    with pytest.raises(ValueError, match="cutoff must be positive"):
        mgk.spatial_graph(mgk.PointCloud(clouds[0]), 0.0)


def test_closed_forms(mgk):
    a = mgk.LabeledGraph.from_edges(1, [], node_labels=np.array([0]), stop_prob=[0.3], start_prob=[1.0])
    b = mgk.LabeledGraph.from_edges(1, [], node_labels=np.array([1]), stop_prob=[0.3], start_prob=[1.0])
    r = mgk.kernel(a, b, mgk.KroneckerDelta(0.8))
    assert r.value == pytest.approx(0.072, rel=1e-6)
    assert r.iterations in (1, 2) and r.converged
    p2 = mgk.LabeledGraph.from_edges(2, [(0, 1, 1.0)], stop_prob=[0.5, 0.5])
    assert mgk.kernel(p2, p2).value == pytest.approx(0.45, rel=1e-6)


def test_gram_config1_golden(mgk, golden_gram):
    rec = golden_gram["config1"]
    graphs = [graph_from_json(g) for g in rec["graphs"]]
    res = mgk.compute_gram(graphs, mgk.KroneckerDelta(0.5), mgk.SquareExponential(1.0))
    ref = np.asarray(rec["matrix"])
    assert res.converged.all()
    assert np.all(np.abs(res.matrix - ref) <= REL * np.abs(ref))
    assert np.array_equal(res.matrix, res.matrix.T)
    assert np.max(np.abs(res.iterations - np.asarray(rec["iterations"]))) <= 1
    assert np.allclose(mgk.normalize_gram(res.matrix), np.asarray(rec["normalized"]), rtol=2 * REL)


def test_gram_normalized_on_device(mgk, golden_gram):
    """normalize_gram (gram.py:98-107) applied on the device == the host restatement == the golden matrix."""
    rec = golden_gram["config1"]
    graphs = [graph_from_json(g) for g in rec["graphs"]]
    res = mgk.compute_gram(graphs, rec["vkernel"], rec["ekernel"], normalize=True)
    raw = mgk.compute_gram(graphs, rec["vkernel"], rec["ekernel"])
    assert np.array_equal(np.diagonal(res.matrix), np.ones(len(graphs)))
    assert np.allclose(res.matrix, mgk.normalize_gram(raw.matrix), rtol=1e-15, atol=0)
    gold = np.asarray(rec["normalized"])
    assert np.max(np.abs(res.matrix - gold) / np.abs(gold)) <= 2 * REL


def test_gram_unlabeled_golden(mgk, golden_gram):
    rec = golden_gram["unlabeled5"]
    graphs = [graph_from_json(g) for g in rec["graphs"]]
    res = mgk.compute_gram(graphs, cfg=mgk.SolverConfig(tolerance=1e-6))
    ref = np.asarray(rec["matrix"])
    assert np.all(np.abs(res.matrix - ref) <= REL * np.abs(ref))


def test_gram_equals_pairs(mgk):
    # reference tests/test_gram.py:55-61: Gram entries == individual kernel() calls
    from paper_1910_06310_b200 import synth

    ds = synth.config2(count=12, seed=3)
    res = mgk.compute_gram(ds, "delta:0.5", "se:1.0")
    for a in range(0, 12, 3):
        for b in range(a, 12, 4):
            k = mgk.kernel(ds[a], ds[b], "delta:0.5", "se:1.0")
            assert res.matrix[a, b] == pytest.approx(k.value, rel=1e-6)
    # mid graphs (25-40 nodes) against 1-5-node graphs: n m <= 128 pairs take the FP64 block solver in
    # both entry points (one routing predicate), so the Gram and kernel() agree on values and iterations
    rng = np.random.default_rng(4)
    mix = [synth.molecule(rng, n) for n in (25, 31, 40)] + [synth.molecule(rng, n) for n in (1, 2, 4, 5)]
    res = mgk.compute_gram(mix, "delta:0.5", "se:1.0")
    for a in range(3):
        for b in range(3, len(mix)):
            k = mgk.kernel(mix[a], mix[b], "delta:0.5", "se:1.0")
            assert res.matrix[a, b] == pytest.approx(k.value, rel=1e-12), (a, b)
            assert res.iterations[a, b] == k.iterations


def test_config2_sample_vs_oracle(mgk):
    from paper_1910_06310_b200 import synth

    ds = synth.config2(count=40, seed=11)
    res = mgk.compute_gram(ds, "delta:0.5", "se:1.0")
    rng = np.random.default_rng(0)
    for _ in range(40):
        a, b = sorted(rng.integers(0, 40, size=2))
        o = O.solve_pcg(ds[a], ds[b], ("delta", 0.5), ("se", 1.0))
        assert abs(res.matrix[a, b] - o.value) <= REL * abs(o.value)
        assert abs(int(res.iterations[a, b]) - o.iterations) <= 1


def _medium_molecules():
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(5)
    return [synth.molecule(rng, int(n)) for n in (30, 45, 12, 60, 100)]


def _check_gram_vs_oracle(mgk, ds, vspec=("delta", 0.5), espec=("se", 1.0), tol=1e-10):
    res = mgk.compute_gram(ds, "delta:0.5" if vspec else None, "se:1.0" if espec else None,
                           mgk.SolverConfig(tolerance=tol))
    for a in range(len(ds)):
        for b in range(a, len(ds)):
            o = O.solve_pcg(ds[a], ds[b], vspec, espec, tol=tol)
            assert abs(res.matrix[a, b] - o.value) <= REL * abs(o.value), (a, b, res.matrix[a, b], o.value)
            assert abs(int(res.iterations[a, b]) - o.iterations) <= 1, (a, b)


def test_edge_case_graphs_vs_oracle(mgk):
    """Single-node and edgeless graphs, an isolated node beside edges, and the size-class
    boundaries (24 nodes = largest warp-class graph, 25 = smallest panel-class graph, 33)."""
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(11)
    iso = mgk.LabeledGraph.from_edges(4, [(0, 1, 1.0), (1, 2, 0.5)], node_labels=np.array([0, 1, 2, 0]),
                                      edge_labels=np.array([0.25, 1.5]))
    ds = [mgk.LabeledGraph.from_edges(1, [], node_labels=np.array([2])),
          mgk.LabeledGraph.from_edges(5, [], node_labels=np.arange(5) % 3), iso,
          synth.molecule(rng, 2), synth.molecule(rng, 24), synth.molecule(rng, 25), synth.molecule(rng, 33)]
    _check_gram_vs_oracle(mgk, ds)
    one = mgk.compute_gram(ds[4:5], "delta:0.5", "se:1.0")
    o = O.solve_pcg(ds[4], ds[4], ("delta", 0.5), ("se", 1.0))
    assert one.matrix.shape == (1, 1) and abs(one.matrix[0, 0] - o.value) <= REL * o.value
    empty = mgk.compute_gram([], "delta:0.5", "se:1.0")
    assert empty.matrix.shape == (0, 0) and empty.converged.shape == (0, 0)
    # gram.py:87: a pair that hits max_iterations is NaN and flagged unconverged (no pair here
    # converges within +-1 iteration of the cap of 8, so the FP32 vectors cannot flip a flag)
    capped = mgk.compute_gram(ds, "delta:0.5", "se:1.0", mgk.SolverConfig(tolerance=1e-10, max_iterations=8))
    for a in range(len(ds)):
        for b in range(a, len(ds)):
            o = O.solve_pcg(ds[a], ds[b], ("delta", 0.5), ("se", 1.0), tol=1e-10, max_iter=8)
            assert bool(capped.converged[a, b]) == o.converged, (a, b)
            if o.converged:
                assert abs(capped.matrix[a, b] - o.value) <= REL * abs(o.value)
            else:
                assert np.isnan(capped.matrix[a, b]) and capped.iterations[a, b] == 8, (a, b)
    # solver.py:77-121: a single kernel() call reports the best iterate, not NaN
    cap = mgk.SolverConfig(tolerance=1e-10, max_iterations=8)
    r = mgk.kernel(ds[4], ds[6], mgk.KroneckerDelta(0.5), mgk.SquareExponential(1.0), cap)
    o = O.solve_pcg(ds[4], ds[6], ("delta", 0.5), ("se", 1.0), tol=1e-10, max_iter=8)
    assert not r.converged and r.iterations == 8 and abs(r.value - o.value) <= 1e-4 * abs(o.value)


def _random_graph(mgk, rng, n):
    """Erdos-Renyi-like graph with random weights, integer node labels and scalar edge labels."""
    p = min(1.0, rng.uniform(1.5, 4.0 if rng.random() < 0.7 else 12.0) / max(n - 1, 1))
    ii, jj = np.triu_indices(n, 1)
    keep = rng.random(ii.size) < p
    ii, jj = ii[keep], jj[keep]
    return mgk.LabeledGraph.from_arrays(n, ii, jj, rng.uniform(0.2, 2.0, ii.size),
                                        node_labels=rng.integers(0, 4, n), edge_labels=rng.uniform(0, 2, ii.size),
                                        stop_prob=rng.uniform(0.05, 0.5, n))


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_random_datasets_vs_oracle(mgk, seed):
    """Seeded random mixes across every size class (1..200 nodes: tiny, warp, wide, panel), random
    densities, weights, stopping probabilities and labels; labeled and unlabeled kernels."""
    rng = np.random.default_rng(100 + seed)
    sizes = [1, 3] + rng.integers(2, 25, 8).tolist() + rng.integers(25, 121, 4).tolist() + [int(rng.integers(121, 201))]
    ds = [_random_graph(mgk, rng, int(n)) for n in sizes]
    # a complete graph on 20 + seed nodes: few nodes but more nonzeros than a warp's slots (380+)
    k = 20 + seed
    ii, jj = np.triu_indices(k, 1)
    ds.append(mgk.LabeledGraph.from_arrays(k, ii, jj, rng.uniform(0.2, 2.0, ii.size), node_labels=rng.integers(0, 4, k),
                                           edge_labels=rng.uniform(0, 2, ii.size)))
    _check_gram_vs_oracle(mgk, ds)
    _check_gram_vs_oracle(mgk, ds[:10] + ds[-1:], None, None, tol=1e-6)  # unlabeled protocol


@pytest.mark.parametrize("vs,es,edge_kind", [
    ("poly:0.5,0.25", "se:0.7", "scalar"),        # polynomial vertex kernel
    ("delta:0.3", "delta:0.4", "int"),            # categorical-delta edges
    ("const1", "se:1.5", "vec3"),                 # 3-D vector edge labels (CTA kernel)
    ("delta:0.5", "prod:se:1.0|delta:0.5", "vec2"),  # composite edge kernel
    ("se:0.5", "delta:0.4", "int"),               # SE vertex kernel on integer node labels
    # (RConvolution sums up to dim^2 sub-kernel values, so on random weights the product system is
    # indefinite; it is covered on the reference's own pairs by test_composite_kernels_golden)
])
def test_random_kernel_families_vs_oracle(mgk, vs, es, edge_kind):
    """Seeded random graphs (1-60 nodes) under each base-kernel family and edge-label kind."""
    rng = np.random.default_rng(300)
    ds = []
    for n in [1, 2] + rng.integers(3, 61, 8).tolist():
        g = _random_graph(mgk, rng, int(n))
        e = g.edge_count
        lab = {"scalar": rng.uniform(0, 2, e), "int": rng.integers(0, 3, e),
               "vec3": rng.uniform(0, 1, (e, 3)), "vec2": np.stack([rng.uniform(0, 1, e), rng.integers(0, 2, e)], 1)}
        ds.append(mgk.LabeledGraph.from_arrays(g.node_count, g.edges_i, g.edges_j, g.weights,
                                               node_labels=g.node_labels, edge_labels=lab[edge_kind],
                                               stop_prob=g.stop_prob))
    res = mgk.compute_gram(ds, vs, es, mgk.SolverConfig(tolerance=1e-10))
    for a in range(len(ds)):
        for b in range(a, len(ds)):
            o = O.solve_pcg(ds[a], ds[b], O.parse_spec(vs), O.parse_spec(es), tol=1e-10)
            assert abs(res.matrix[a, b] - o.value) <= REL * abs(o.value), (a, b, res.matrix[a, b], o.value)
            assert abs(int(res.iterations[a, b]) - o.iterations) <= 1, (a, b, int(res.iterations[a, b]), o.iterations)


def test_random_pairs_nodewise_pbr_vs_oracle(mgk):
    """kernel() with PBR reordering on random pairs across the size classes: value, iterations and
    the un-permuted nodewise field against the oracle on the original node order."""
    rng = np.random.default_rng(400)
    for n1, n2 in [(5, 9), (20, 22), (24, 60), (70, 110), (150, 3)]:
        ga, gb = _random_graph(mgk, rng, n1), _random_graph(mgk, rng, n2)
        r = mgk.kernel(ga, gb, mgk.KroneckerDelta(0.5), mgk.SquareExponential(1.0), reorder="pbr")
        o = O.solve_pcg(ga, gb, ("delta", 0.5), ("se", 1.0), tol=1e-10)
        assert abs(r.value - o.value) <= REL * abs(o.value), (n1, n2)
        assert abs(r.iterations - o.iterations) <= 1, (n1, n2, r.iterations, o.iterations)
        assert np.max(np.abs(r.nodewise - o.nodewise)) <= 1e-5 * np.max(np.abs(o.nodewise)), (n1, n2)


def test_dense_small_graph_tiny_pairs(mgk):
    """A complete K20 (20 nodes, 380 nonzeros: outside the warp class) against a triangle: n m = 60
    is tiny, so kernel() and the Gram run it with FP64 vectors (block solver) and the unlabeled pair
    matches the oracle's iteration count at the reference default 1e-10, where FP32 vectors stall."""
    rng = np.random.default_rng(100)
    sizes = [1, 3] + rng.integers(2, 25, 8).tolist() + rng.integers(25, 121, 4).tolist() + [int(rng.integers(121, 201))]
    ds = [_random_graph(mgk, rng, int(n)) for n in sizes]
    ii, jj = np.triu_indices(20, 1)
    k20 = mgk.LabeledGraph.from_arrays(20, ii, jj, rng.uniform(0.2, 2.0, ii.size), node_labels=rng.integers(0, 4, 20),
                                       edge_labels=rng.uniform(0, 2, ii.size))
    for vs, es in [(None, None), ("delta:0.5", "se:1.0")]:
        for ga, gb in [(ds[1], k20), (k20, ds[1]), (ds[4], k20), (ds[0], k20)]:  # 3, 3, 4, 1 nodes
            r = mgk.kernel(ga, gb, vs and mgk.KroneckerDelta(0.5), es and mgk.SquareExponential(1.0))
            o = O.solve_pcg(ga, gb, O.parse_spec(vs), O.parse_spec(es), tol=1e-10)
            assert abs(r.value - o.value) <= REL * abs(o.value)
            assert abs(r.iterations - o.iterations) <= 1, (vs, ga.node_count, gb.node_count, r.iterations, o.iterations)
    # the Gram routes the same pairs to the FP64 block solver (the mid x small tiny job of gram_jobs);
    # unlabeled at 1e-10 every pair runs there (kPreciseTol)
    gs = [ds[0], ds[1], ds[4], k20, ds[2]]
    for vs, es in [(None, None), (("delta", 0.5), ("se", 1.0))]:
        _check_gram_vs_oracle(mgk, gs, vs, es, tol=1e-10)


def test_medium_pairs_panel_kernel(mgk):
    # graphs above the warp class (n > 24) go through the CTA-per-pair panel kernel
    # (pcg_panel.cu): self pairs, small x medium (orientation swap), medium x medium
    _check_gram_vs_oracle(mgk, _medium_molecules())


def test_medium_pairs_block_kernel(mgk, monkeypatch):
    # the generic CTA kernel (pcg_block.cu) stays the path for vector edge labels
    monkeypatch.setenv("MGK_NO_PANEL", "1")
    _check_gram_vs_oracle(mgk, _medium_molecules()[:4])


def test_panel_protein_pairs_vs_oracle(mgk):
    """Config-3 shapes (shuffled C-alpha chains, several 256-nonzero row panels per graph)."""
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(31)
    ds = [synth.protein(rng, int(n)) for n in (120, 200, 240)]
    ds = [mgk.apply_permutation(g, mgk.pbr_reorder(g, seed=0)) for g in ds]
    _check_gram_vs_oracle(mgk, ds)


def test_panel_nodewise_vs_oracle(mgk):
    """Nodewise field through the panel kernel, both orientations (U/L swap transposes on write)."""
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(8)
    big = synth.protein(rng, 90)
    small = synth.molecule(rng, 9)
    mid = synth.molecule(rng, 40)
    for ga, gb in ((big, small), (small, big), (mid, big), (big, big)):
        k = mgk.kernel(ga, gb, "delta:0.5", "se:1.0")
        o = O.solve_pcg(ga, gb, ("delta", 0.5), ("se", 1.0))
        assert abs(k.value - o.value) <= REL * abs(o.value)
        assert abs(k.iterations - o.iterations) <= 1
        assert k.nodewise.shape == o.nodewise.shape
        assert np.max(np.abs(k.nodewise - o.nodewise)) <= REL * np.max(np.abs(o.nodewise))


def test_grid_class_vs_oracle(mgk, monkeypatch):
    """The whole-device cooperative solver (k_pcg_grid), driven at oracle-sized graphs by
    lowering its size threshold: Gram (self pairs included) and nodewise pair lists."""
    from paper_1910_06310_b200 import synth

    monkeypatch.setenv("MGK_GRID_N", "60")
    rng = np.random.default_rng(12)
    ds = [synth.protein(rng, int(n)) for n in (70, 130, 180)]
    _check_gram_vs_oracle(mgk, ds)
    k = mgk.kernel(ds[0], ds[2], "delta:0.5", "se:1.0")
    o = O.solve_pcg(ds[0], ds[2], ("delta", 0.5), ("se", 1.0))
    assert abs(k.value - o.value) <= REL * abs(o.value)
    assert abs(k.iterations - o.iterations) <= 1
    assert np.max(np.abs(k.nodewise - o.nodewise)) <= REL * np.max(np.abs(o.nodewise))
    ul = [mgk.LabeledGraph.from_arrays(g.node_count, g.edges_i, g.edges_j, g.weights, default_q=0.05) for g in ds]
    _check_gram_vs_oracle(mgk, ul[:2], None, None, tol=1e-6)


def test_gram_shards_cover_all_pairs(mgk):
    """mgk_gram_shard: world = 3 shards of a mixed dataset (tiny, narrow, wide, panel classes) are
    disjoint, cover every pair a <= b once and reproduce the single-device Gram bit for bit."""
    from paper_1910_06310_b200 import native, synth

    rng = np.random.default_rng(41)
    ii, jj = np.triu_indices(20, 1)
    k20 = mgk.LabeledGraph.from_arrays(20, ii, jj, rng.uniform(0.2, 2.0, ii.size), node_labels=rng.integers(0, 4, 20),
                                       edge_labels=rng.uniform(0, 2, ii.size))
    ds = [synth.molecule(rng, int(n)) for n in rng.integers(4, 24, size=24)] + \
         [synth.molecule(rng, int(n)) for n in (30, 45, 60, 2, 3)] + [k20]
    ctx = native.Context(0)
    ctx.upload(native.PackedDataset(ds))
    ctx.set_kernels("delta:0.5", "se:1.0")
    K, it, cv = ctx.gram(1e-10)
    seen = {}
    for rank in range(3):
        pa, pb, v, its, c = ctx.gram_shard(rank, 3, 1e-10)
        for a, b, x, i in zip(pa.tolist(), pb.tolist(), v.tolist(), its.tolist()):
            assert a <= b and (a, b) not in seen
            seen[(a, b)] = (x, i)
    G = len(ds)
    assert len(seen) == G * (G + 1) // 2
    for (a, b), (x, i) in seen.items():
        assert x == K[a, b] and i == it[a, b]


def test_stream_nodewise_vs_oracle(mgk):
    """mgk_gram_nodewise: every pair a <= b of a mixed-size set (warp, tiny, panel classes), streamed in
    several chunks and sharded over two ranks; fields and values against the oracle."""
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(21)
    ii, jj = np.triu_indices(20, 1)
    k20 = mgk.LabeledGraph.from_arrays(20, ii, jj, rng.uniform(0.2, 2.0, ii.size), node_labels=rng.integers(0, 4, 20),
                                       edge_labels=rng.uniform(0, 2, ii.size))
    ds = [synth.molecule(rng, int(n)) for n in (5, 9, 14, 23, 30, 47, 3)] + [k20]
    sizes = [g.node_count for g in ds]
    seen = {}
    chunks = []

    def take(a, b, v, it, cv, off, f):
        chunks.append(len(a))
        for k in range(len(a)):
            key = (int(a[k]), int(b[k]))
            assert key not in seen
            seen[key] = (float(v[k]), int(it[k]), bool(cv[k]),
                         f[off[k]:off[k + 1]].reshape(sizes[a[k]], sizes[b[k]]).copy())

    for rank in range(2):
        mgk.stream_nodewise(ds, take, "delta:0.5", "se:1.0", chunk_bytes=4 * 1500, rank=rank, world=2)
    assert sorted(seen) == [(a, b) for a in range(8) for b in range(a, 8)]
    assert len(chunks) > 4
    for (a, b), (v, it, cv, field) in seen.items():
        o = O.solve_pcg(ds[a], ds[b], ("delta", 0.5), ("se", 1.0))
        assert cv and abs(v - o.value) <= REL * abs(o.value) and abs(it - o.iterations) <= 1
        assert np.max(np.abs(field - o.nodewise)) <= REL * np.max(np.abs(o.nodewise)), (a, b)


def test_stream_nodewise_consumer_error(mgk):
    """A consumer exception stops the stream, surfaces in Python, and leaves the context usable."""
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(22)
    ds = [synth.molecule(rng, int(n)) for n in (6, 9, 12, 15, 20)]
    calls = []

    def boom(a, b, v, it, cv, off, f):
        calls.append(len(a))
        if len(calls) == 2:
            raise RuntimeError("consumer stop")

    with pytest.raises(RuntimeError, match="consumer stop"):
        mgk.stream_nodewise(ds, boom, "delta:0.5", "se:1.0", chunk_bytes=4 * 200)
    assert len(calls) == 2
    res = mgk.compute_gram(ds, "delta:0.5", "se:1.0")
    assert np.all(res.converged)


def test_panel_unlabeled_rgg_vs_oracle(mgk):
    """Config-4 shape (random geometric graphs, unlabeled, tol 1e-6 per SURVEY H1) at reduced n."""
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(4)
    ds = [synth.rgg(rng, int(n), d) for n, d in ((150, 8), (220, 16), (180, 4))]
    ds = [mgk.LabeledGraph.from_arrays(g.node_count, g.edges_i, g.edges_j, g.weights, default_q=0.05)
          for g in ds]
    _check_gram_vs_oracle(mgk, ds, None, None, tol=1e-6)


def test_validation_errors(mgk):
    g = mgk.LabeledGraph.from_edges(3, [(0, 0, 1.0), (1, 2, 1.0)])
    with pytest.raises(ValueError, match="self-loop at node 0"):
        mgk.kernel(g, g)
    bad_q = mgk.LabeledGraph.from_edges(2, [(0, 1, 1.0)], stop_prob=[0.0, 0.5])
    with pytest.raises(ValueError, match="stopping probability must be > 0 at node 0"):
        mgk.compute_gram([bad_q])


def test_bindings_roundtrip(mgk):
    from paper_1910_06310_b200 import mgkbind

    p2 = mgkbind.BoundGraph(adjacency=np.array([[0.0, 1.0], [1.0, 0.0]]), stop_prob=np.array([0.5, 0.5]))
    v, nw, diag = mgkbind.kernel(p2, p2)
    assert v == pytest.approx(0.45, rel=1e-6) and diag["converged"] and nw.shape == (2, 2)
    loop = mgkbind.BoundGraph(adjacency=(np.array([0]), np.array([0]), np.array([1.0])),
                              stop_prob=np.array([0.5, 0.5]))
    with pytest.raises(mgkbind.SolverError, match="self-loop"):
        mgkbind.kernel(loop, loop)
    m, flags = mgkbind.gram([p2, p2], normalize=True)
    assert flags.all() and np.allclose(np.diagonal(m), 1.0)


def test_pbr_permutations_bit_exact(mgk, golden_structure):
    """Device PBR (csrc/pbr.cu) == reference pbr_reorder on every golden graph, seeds 0 and 3."""
    graphs = [graph_from_json(r["graph"]) for r in golden_structure]
    for seed in ("0", "3"):
        perms = mgk.pbr_reorder_many(graphs, seed=int(seed))
        for rec, perm in zip(golden_structure, perms):
            assert perm.forward.tolist() == rec["pbr"][seed], (rec["name"], seed)


def test_pbr_known_answers_on_device(mgk):
    """Reference tests/test_reorder.py:61-65: two 8-cliques are already optimal (objective 0), and the
    device permutation equals the oracle's on them and on K24."""
    cl = [(i, j, 1.0) for i in range(8) for j in range(i + 1, 8)]
    cl += [(i, j, 1.0) for i in range(8, 16) for j in range(i + 1, 16)]
    blocks = mgk.LabeledGraph.from_edges(16, cl)
    k24 = mgk.LabeledGraph.from_edges(24, [(i, j, 1.0) for i in range(24) for j in range(i + 1, 24)])
    perms = mgk.pbr_reorder_many([blocks, k24], seed=1)
    assert O.pair_objective(blocks, perms[0].forward // 8) == 0
    assert perms[0].forward.tolist() == O.pbr_reorder(blocks, 1).tolist()
    assert perms[1].forward.tolist() == O.pbr_reorder(k24, 1).tolist()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_pbr_random_graphs_bit_exact(mgk, seed):
    """Device PBR == oracle pbr_reorder on seeded random graphs (9-220 nodes, often disconnected,
    mixed densities), with the PBR seed varied alongside."""
    rng = np.random.default_rng(200 + seed)
    graphs = [_random_graph(mgk, rng, int(n)) for n in rng.integers(9, 221, 8)]
    perms = mgk.pbr_reorder_many(graphs, seed=seed)
    for i, (g, perm) in enumerate(zip(graphs, perms)):
        assert perm.forward.tolist() == O.pbr_reorder(g, seed).tolist(), (i, g.node_count)


def test_pbr_tiles_after_reorder(mgk, golden_structure):
    for rec in golden_structure:
        g = graph_from_json(rec["graph"])
        perm = mgk.pbr_reorder(g, seed=0)
        t = mgk.build_tiles(mgk.apply_permutation(g, perm))
        assert t.tile_count == rec["pbr_tiles_0"], rec["name"]


def test_kernel_with_pbr_reorder_golden(mgk, golden_kernels):
    for rec in golden_kernels:
        if rec["reorder"] != "pbr":
            continue
        ga, gb = graph_from_json(rec["a"]), graph_from_json(rec["b"])
        res = mgk.kernel(ga, gb, rec["vkernel"], rec["ekernel"], reorder="pbr", seed=0)
        assert abs(res.value - rec["value"]) <= REL * abs(rec["value"])
        assert abs(res.iterations - rec["iterations"]) <= 1
        nw = np.asarray(rec["nodewise"])
        assert np.max(np.abs(res.nodewise - nw)) <= REL * np.max(np.abs(nw))


def test_pbr_protein_shaped_vs_oracle(mgk):
    """Shuffled C-alpha chains (config 3 shape) at n up to 200 against the oracle restatement."""
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(77)
    graphs = [synth.protein(rng, int(n)) for n in (40, 90, 150)]
    perms = mgk.pbr_reorder_many(graphs, seed=5)
    for g, p in zip(graphs, perms):
        assert p.forward.tolist() == O.pbr_reorder(g, 5).tolist()


def _mixed_dataset(mgk, seed):
    from paper_1910_06310_b200 import synth

    rng = np.random.default_rng(seed)
    ii, jj = np.triu_indices(20, 1)
    k20 = mgk.LabeledGraph.from_arrays(20, ii, jj, rng.uniform(0.2, 2.0, ii.size), node_labels=rng.integers(0, 4, 20),
                                       edge_labels=rng.uniform(0, 2, ii.size))
    return [synth.molecule(rng, int(n)) for n in rng.integers(2, 24, size=30)] + \
           [synth.molecule(rng, int(n)) for n in (30, 45, 60)] + [k20]


def test_gram_multi_device_bit_identical(mgk):
    """compute_gram(devices=[...]) (mgk_gram_multi: one process, one context + host thread per device,
    round-robin cost-ordered shards scattered into the host matrix) reproduces the single-device Gram
    bit for bit -- here with 2 and 3 contexts on the one GPU of the test box."""
    ds = _mixed_dataset(mgk, 51)
    ref = mgk.compute_gram(ds, "delta:0.5", "se:1.0")
    for devs in ([0, 0], [0, 0, 0]):
        res = mgk.compute_gram(ds, "delta:0.5", "se:1.0", devices=devs)
        assert np.array_equal(res.matrix, ref.matrix), devs
        assert np.array_equal(res.iterations, ref.iterations) and np.array_equal(res.converged, ref.converged)
    res = mgk.compute_gram(ds, "delta:0.5", "se:1.0", devices=[0, 0], normalize=True)
    assert np.allclose(res.matrix, mgk.normalize_gram(ref.matrix), rtol=1e-15, atol=0)


def test_gram_shard_device_records_assemble(mgk):
    """mgk_gram_shard_device writes each shard's records to caller-owned device tensors (the input of the
    NCCL gather in bench.py), mgk_gram_assemble scatters the concatenated records into a device Gram:
    identical to the single-device matrix, padding records (id -1) ignored."""
    import torch

    from paper_1910_06310_b200 import native
    from paper_1910_06310_b200.solver import context

    ds = _mixed_dataset(mgk, 52)
    ref = mgk.compute_gram(ds, "delta:0.5", "se:1.0")
    ctx = context(0)
    ctx.upload(native.PackedDataset(ds))
    ctx.set_kernels("delta:0.5", "se:1.0")
    dev = torch.device("cuda", 0)
    parts = []
    for rank in range(3):
        n = ctx.gram_shard_device(rank, 3, 1e-10)
        rec = (torch.empty(n + 2, dtype=torch.int32, device=dev), torch.empty(n + 2, dtype=torch.int32, device=dev),
               torch.empty(n + 2, dtype=torch.float64, device=dev), torch.empty(n + 2, dtype=torch.int32, device=dev),
               torch.zeros(n + 2, dtype=torch.uint8, device=dev))
        rec[0][n:] = -1  # padding
        rec[1][n:] = -1
        assert ctx.gram_shard_device(rank, 3, 1e-10, out=rec) == n
        parts.append(rec)
    recs = [torch.cat([p[k] for p in parts]) for k in range(5)]
    G = len(ds)
    K = torch.empty((G, G), dtype=torch.float64, device=dev)
    it = torch.empty((G, G), dtype=torch.int32, device=dev)
    cv = torch.empty((G, G), dtype=torch.uint8, device=dev)
    native.gram_assemble(0, recs, G, K, it, cv)
    assert np.array_equal(K.cpu().numpy(), ref.matrix)
    assert np.array_equal(it.cpu().numpy(), ref.iterations) and np.array_equal(cv.cpu().numpy().astype(bool),
                                                                               ref.converged)


def test_large_gram_staged_transfer(mgk):
    """A 4100-graph Gram (0.13 GB of values, 67 MB of int32 iteration counts) leaves the device through
    the pinned double-buffered staging path with host-side int64 widening (capi.cu d2h_staged): the
    matrix is symmetric, every pair converged, and sampled entries equal the oracle and kernel()."""
    from paper_1910_06310_b200 import synth

    ds = synth.config2(count=4100, seed=21)
    res = mgk.compute_gram(ds, "delta:0.5", "se:1.0")
    K, it = res.matrix, res.iterations
    assert K.shape == (4100, 4100) and it.dtype == np.int64
    assert np.array_equal(K, K.T) and np.array_equal(it, it.T)
    assert res.converged.all() and (it > 0).all()
    rng = np.random.default_rng(5)
    pairs = list(zip(rng.integers(0, 4100, 6), rng.integers(0, 4100, 6)))
    pairs += [(4099, 4099), (0, 4099), (4098, 17)]  # entries of the last staged chunks
    for a, b in pairs:
        o = O.solve_pcg(ds[a], ds[b], ("delta", 0.5), ("se", 1.0))
        assert abs(K[a, b] - o.value) <= 1e-5 * abs(o.value), (a, b)
        assert abs(int(it[a, b]) - o.iterations) <= 1, (a, b)
        k = mgk.kernel(ds[a], ds[b], "delta:0.5", "se:1.0")  # the pair API (plain small transfers)
        assert K[a, b] == pytest.approx(k.value, rel=1e-6), (a, b)
