"""Host-side logic of the drop-in (no GPU): graph container and validation
texts, schedule order, kernel SPEC lowering, dataset packing, bindings'
array marshalling, Gram post-processing and persistence formats."""
import numpy as np
import pytest

from conftest import graph_from_json
from oracle import mgk_oracle as O


def test_validation_messages_match_reference_texts():
    from paper_1910_06310_b200 import LabeledGraph, validate_graph

    g = LabeledGraph(3, np.array([0, 1, 1, 0]), np.array([0, 2, 2, 5]), np.array([1.0, -1.0, 1.0, 1.0]),
                     np.array([0.5, -0.1, 0.2]), np.array([0.0, 0.5, 1.5]))
    got = validate_graph(g).violations
    assert got == O.validate(g)
    assert "self-loop at node 0" in got and "duplicate edge (1,2)" in got
    assert "stopping probability must be > 0 at node 0" in got
    assert "stopping probability must be <= 1 at node 2" in got
    assert "edge (0,5) references unknown node" in got


def test_from_edges_defaults():
    from paper_1910_06310_b200 import LabeledGraph

    g = LabeledGraph.from_edges(4, [(2, 1, 0.5)])
    assert g.edges_i.tolist() == [1] and g.edges_j.tolist() == [2]
    assert np.allclose(g.start_prob, 0.25) and np.allclose(g.stop_prob, 0.05)
    with pytest.raises(ValueError):
        LabeledGraph.from_edges(2, [], default_q=1e-5)


def test_schedule_pairs_matches_reference(golden_gram):
    from paper_1910_06310_b200 import schedule_pairs

    s = golden_gram["schedule"]
    assert [list(p) for p in schedule_pairs([4, 4, 4], [6, 6, 6])] == s["uniform"]
    assert [list(p) for p in schedule_pairs([4, 100, 4, 4], [6, 2000, 6, 6])] == s["giant"]
    assert [list(p) for p in schedule_pairs([10, 20, 10, 7, 3], [30, 120, 20, 14, 2])] == s["mixed"]
    rec = golden_gram["config1"]
    graphs = [graph_from_json(g) for g in rec["graphs"]]
    got = schedule_pairs([g.node_count for g in graphs], [2 * g.edge_count for g in graphs])
    assert [list(p) for p in got] == rec["order"]


def test_kernel_spec_lowering():
    from paper_1910_06310_b200 import (CompactPolynomial, ConstantOne, KroneckerDelta, ProductComposite,
                                       RConvolution, SquareExponential, kernel_from_spec)
    from paper_1910_06310_b200.solver import kernel_spec

    assert kernel_spec(None) is None
    assert kernel_spec(ConstantOne()) == "const1"
    assert kernel_spec(KroneckerDelta(0.5)) == "delta:0.5"
    assert kernel_spec(SquareExponential(1.25)) == "se:1.25"
    assert kernel_spec(CompactPolynomial([1.0, -0.5])) == "poly:1.0,-0.5"
    assert kernel_spec(kernel_from_spec("se:2.0")) == "se:2.0"
    # composites lower to the extended grammar; nesting and >4 components have no device lowering
    assert kernel_spec(ProductComposite([ConstantOne(), SquareExponential(0.5)])) == "prod:const1|se:0.5"
    assert kernel_spec(RConvolution(KroneckerDelta(0.25))) == "rconv:delta:0.25"
    assert kernel_spec(kernel_from_spec("prod:delta:0.5|poly:1.0,-0.2")) == "prod:delta:0.5|poly:1.0,-0.2"
    with pytest.raises(NotImplementedError):
        kernel_spec(ProductComposite([RConvolution(ConstantOne())]))
    with pytest.raises(NotImplementedError):
        kernel_spec(ProductComposite([ConstantOne()] * 5))
    with pytest.raises(ValueError):
        KroneckerDelta(0.0)
    assert KroneckerDelta(0.5).flop_count == 1 and SquareExponential(1.0).flop_count == 4


def test_packed_dataset_layout():
    from paper_1910_06310_b200 import native, synth
    from paper_1910_06310_b200.basekernels import KernelShapeError

    ds = synth.config1()
    pk = native.PackedDataset(ds)
    assert pk.G == 16 and pk.node_off[-1] == sum(g.node_count for g in ds)
    assert pk.edge_off[-1] == len(pk.ei) == len(pk.w)
    assert pk.nl_kind == native.LABEL_CAT and pk.el_kind == native.LABEL_VEC and pk.el_dim == 1
    k = 5
    lo, hi = pk.edge_off[k], pk.edge_off[k + 1]
    assert np.array_equal(pk.ei[lo:hi], ds[k].edges_i) and np.array_equal(pk.w[lo:hi], ds[k].weights)
    mixed = [ds[0], ds[1].with_probabilities()]
    mixed[1] = type(ds[1])(**{**ds[1].__dict__, "edge_labels": None})
    with pytest.raises(KernelShapeError, match="presence"):
        native.PackedDataset(mixed)


def test_boundgraph_marshalling():
    from paper_1910_06310_b200.mgkbind import BoundGraph, _to_graph

    dense = np.array([[0, 1.5, 0], [1.5, 0, 2.0], [0, 2.0, 0]])
    g = _to_graph(BoundGraph(adjacency=dense), q=0.3, unlabeled=False)
    assert g.edges_i.tolist() == [0, 1] and g.edges_j.tolist() == [1, 2]
    assert np.allclose(g.stop_prob, 0.3)
    with pytest.raises(ValueError, match="symmetric"):
        BoundGraph(adjacency=np.array([[0, 1.0], [0.5, 0]])).edge_arrays()
    trip = BoundGraph(adjacency=(np.array([0]), np.array([3]), np.array([1.0])))
    assert trip.edge_arrays()[0] == 4


def test_gram_persistence_roundtrip(tmp_path):
    from paper_1910_06310_b200 import load_gram_binary, load_gram_csv, normalize_gram, save_gram_binary, save_gram_csv

    K = np.array([[2.0, 1.0, np.nan], [1.0, 4.0, 0.5], [np.nan, 0.5, 1.0]])
    save_gram_binary(K, tmp_path / "k.bin")
    raw = (tmp_path / "k.bin").read_bytes()
    assert raw[:5] == b"GRAM\x01" and int.from_bytes(raw[5:13], "little") == 3
    assert np.array_equal(load_gram_binary(tmp_path / "k.bin"), K, equal_nan=True)
    save_gram_csv(K, ["a", "b", "c"], tmp_path / "k.csv")
    ids, K2 = load_gram_csv(tmp_path / "k.csv")
    assert ids == ["a", "b", "c"] and np.array_equal(K2, K, equal_nan=True)
    N = normalize_gram(K)
    assert N[0, 1] == pytest.approx(1.0 / np.sqrt(8.0)) and N[2, 2] == 1.0 and np.isnan(N[0, 2])
    assert np.allclose(N, O.normalize_gram(K), equal_nan=True)


def test_synth_configs_shapes():
    from paper_1910_06310_b200 import synth

    c2 = synth.config2(count=50)
    assert all(4 <= g.node_count <= 23 for g in c2)
    assert all(g.edge_labels is not None and g.node_labels is not None for g in c2)
    c3 = synth.config3(count=2, n_lo=200, n_hi=210)
    assert all(200 <= g.node_count <= 210 for g in c3)
    assert synth.config2(count=5, seed=1)[3].edges_i.tolist() == synth.config2(count=5, seed=1)[3].edges_i.tolist()


def test_predict_costs_golden():
    """predict_costs (costs.py:74-128) against the reference's cells, exactly (counters.json)."""
    from conftest import load_golden
    from paper_1910_06310_b200 import CostModel, predict_costs

    for rec in load_golden("counters.json")["predict"]:
        got = predict_costs(CostModel(**rec["model"]), rec["n"], rec["m"], rec["primitive"])
        for k, v in rec["report"].items():
            assert getattr(got, k) == v, (rec["primitive"], rec["n"], rec["m"], k)


def test_cost_model_validation_and_selection():
    """costs.py:35-43 validation; product.py:56-66 selection with the reference's per-mode thresholds."""
    from paper_1910_06310_b200 import CostModel, CounterReport, select_tile_kernel

    for bad in ({"E": -1}, {"F": 0}, {"X": 0}, {"t": 8, "r": 3}):
        with pytest.raises(ValueError):
            CostModel(**bad)
    assert select_tile_kernel(10, 16, "unlabeled") == "sparse-sparse"
    assert select_tile_kernel(11, 16, "unlabeled") == "dense-sparse"
    assert select_tile_kernel(16, 24, "labeled") == "sparse-sparse"
    assert select_tile_kernel(32, 40, "labeled") == "dense-dense"
    assert select_tile_kernel(5, 40, "labeled") == "dense-sparse"
    rep = CounterReport(flops=100.0, t1_load=40.0, t1_store=10.0, t2_load=0.0, t2_store=0.0).finalize()
    assert rep.ai1 == 2.0 and rep.ai2 is None


def _same_graph(g, rec):
    ref = graph_from_json(rec)
    assert g.node_count == ref.node_count
    for f in ("edges_i", "edges_j", "weights", "start_prob", "stop_prob"):
        assert np.array_equal(np.asarray(getattr(g, f)), np.asarray(getattr(ref, f))), f
    for f in ("node_labels", "edge_labels"):
        a, b = getattr(g, f), getattr(ref, f)
        assert (a is None) == (b is None), f
        if a is not None:
            assert np.array_equal(np.asarray(a).reshape(len(a), -1), np.asarray(b).reshape(len(b), -1)), f


def test_graph_files_reference_fixtures(tmp_path):
    """load_graph / load_edge_list on files the reference wrote (graphio.py:61-208), save -> load round
    trip, and the reference's GraphFileError texts."""
    import json

    from conftest import GOLDEN
    from paper_1910_06310_b200 import GraphFileError, load_edge_list, load_graph, save_graph

    files = GOLDEN / "files"
    index = json.loads((files / "index.json").read_text())
    for name in ("cat", "vec", "plain"):
        g = load_graph(files / f"{name}.json")
        _same_graph(g, index[name])
        save_graph(g, tmp_path / f"{name}.json")
        assert json.loads((tmp_path / f"{name}.json").read_text()) == json.loads((files / f"{name}.json").read_text())
    _same_graph(load_edge_list(files / "edges.txt"), index["edges"])
    bad = {"missing": ({"node_count": 2, "nodes": []}, "missing field 'edges'"),
           "count": ({"node_count": 2, "nodes": [{"id": 0}], "edges": []}, "nodes: expected 2 entries, got 1"),
           "ids": ({"node_count": 2, "nodes": [{"id": 0}, {"id": 2}], "edges": []}, "ids must be dense 0..1"),
           "kind": ({"node_count": 1, "nodes": [{"id": 0}], "edges": [], "node_label_kind": "x"}, "unknown label kind"),
           "edge": ({"node_count": 2, "nodes": [{"id": 0}, {"id": 1}], "edges": [{"i": 0, "j": 5, "w": 1.0}]},
                    "edge 0: unknown node id 5"),
           "label": ({"node_count": 2, "nodes": [{"id": 0}, {"id": 1}], "edges": [{"i": 0, "j": 1, "w": 1, "label": 2}]},
                     "edge 0: label present but kind is none")}
    for key, (doc, msg) in bad.items():
        (tmp_path / f"{key}.json").write_text(json.dumps(doc))
        with pytest.raises(GraphFileError, match=msg):
            load_graph(tmp_path / f"{key}.json")
    (tmp_path / "e.txt").write_text("0 1 2 3\n")
    with pytest.raises(GraphFileError, match="line 1: expected 'i j \\[w\\]'"):
        load_edge_list(tmp_path / "e.txt")


def test_nodewise_csv_roundtrip(tmp_path):
    """save_nodewise_csv writes the CLI's nodewise format (cli.py:65-69): reading the reference's file
    back and writing it again reproduces it byte for byte."""
    from conftest import GOLDEN
    from paper_1910_06310_b200 import load_nodewise_csv, save_nodewise_csv

    src = GOLDEN / "files" / "nodewise.csv"
    field = load_nodewise_csv(src)
    save_nodewise_csv(field, tmp_path / "nw.csv")
    assert (tmp_path / "nw.csv").read_text() == src.read_text()
