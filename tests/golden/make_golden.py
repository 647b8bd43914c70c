"""Generate golden vectors by running the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [composite|spatial]

The reference (``mgksolver``, /root/reference/pkg/src) is imported read-only
and evaluated on seeded inputs; inputs and outputs are written to
``tests/golden/*.json`` so the GPU box (which has no /root/reference) can
check both the oracle and the CUDA path against the reference's own numbers.
Floats are serialised with ``repr`` (json default), which round-trips exactly.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, os.environ.get("MGK_REFERENCE_SRC", "/root/reference/pkg/src"))

import mgksolver as ref  # noqa: E402  (the reference)

from paper_1910_06310_b200 import synth  # noqa: E402  (input synthesis only)


def gjson(g) -> dict:
    def lab(x):
        if x is None:
            return None
        return {"kind": "categorical" if x.dtype.kind in "iu" else "vector", "data": x.tolist()}

    return {
        "n": int(g.node_count),
        "ei": np.asarray(g.edges_i).tolist(),
        "ej": np.asarray(g.edges_j).tolist(),
        "w": np.asarray(g.weights, float).tolist(),
        "p": np.asarray(g.start_prob, float).tolist(),
        "q": np.asarray(g.stop_prob, float).tolist(),
        "node_labels": lab(g.node_labels),
        "edge_labels": lab(g.edge_labels),
    }


def to_ref(g) -> "ref.LabeledGraph":
    return ref.LabeledGraph.from_edges(
        g.node_count, list(zip(g.edges_i.tolist(), g.edges_j.tolist(), g.weights.tolist())),
        node_labels=g.node_labels, edge_labels=g.edge_labels,
        start_prob=g.start_prob, stop_prob=g.stop_prob)


def random_graph(rng, n, density=0.3, labeled=False, q_range=(0.2, 0.9), cat_edges=False,
                 edge_dim=1, vec_nodes=False):
    """Same draws as the reference fixture (tests/conftest.py:7-25) plus variants."""
    edges, el = [], []
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < density:
                edges.append((i, j, float(rng.uniform(0.2, 2.0))))
                el.append(float(rng.uniform(0.0, 2.0)))
    nl = rng.integers(0, 3, size=n) if labeled else None
    if labeled and vec_nodes:
        nl = rng.integers(0, 2, size=(n, 2)).astype(float)
    elab = None
    if labeled:
        if cat_edges:
            elab = (np.array(el) * 1.5).astype(np.int64)
        elif edge_dim > 1:
            elab = np.array([[v * (c + 1) / edge_dim for c in range(edge_dim)] for v in el])
        else:
            elab = np.array(el)
        if not edges:
            elab = None
    return ref.LabeledGraph.from_edges(n, edges, node_labels=nl, edge_labels=elab,
                                       start_prob=rng.uniform(0.1, 1.0, size=n),
                                       stop_prob=rng.uniform(*q_range, size=n))


def make_rng_vectors():
    out = {}
    for seed in (0, 1, 42, 2**63 + 5):
        r = ref.SplitMix64(seed)
        out[str(seed)] = {
            "u64": [hex(r.next_u64()) for _ in range(8)],
            "randint": [ref.SplitMix64(seed).randint(k) for k in (1, 2, 3, 7, 1000, 2**40 + 3)],
            "random": [ref.SplitMix64(seed).random()],
        }
        xs = list(range(20))
        ref.SplitMix64(seed).shuffle(xs)
        out[str(seed)]["shuffle20"] = xs
    return out


def structure_graphs():
    rng = np.random.default_rng(11)
    gs = []
    gs.append(("edgeless8", ref.LabeledGraph.from_edges(8, [])))
    gs.append(("k8", ref.LabeledGraph.from_edges(8, [(i, j, 1.0) for i in range(8) for j in range(i + 1, 8)])))
    gs.append(("edge_0_9", ref.LabeledGraph.from_edges(16, [(0, 9, 1.0)])))
    gs.append(("four_node", ref.LabeledGraph.from_edges(4, [(0, 2, 1.0), (1, 3, 1.0)])))
    blocks = [(i, j, 1.0) for i in range(8) for j in range(i + 1, 8)]
    blocks += [(i, j, 1.0) for i in range(8, 16) for j in range(i + 1, 16)]
    gs.append(("two_cliques", ref.LabeledGraph.from_edges(16, blocks)))
    for k in range(12):
        n = int(rng.integers(2, 60))
        gs.append((f"er{k}", random_graph(rng, n, density=float(rng.uniform(0.05, 0.4)), labeled=True)))
    gs.append(("nws96", ref.gen_nws(96, 3, 0.1, 7)))
    gs.append(("ba64", ref.gen_ba(64, 3, 5)))
    srng = np.random.default_rng(1000)
    for k, n in enumerate((120, 200)):
        gs.append((f"protein{n}", to_ref(synth.protein(srng, n))))
    mrng = np.random.default_rng(7165)
    for k in range(6):
        gs.append((f"mol{k}", to_ref(synth.molecule(mrng, int(mrng.integers(4, 24))))))
    return gs


def make_structure():
    out = []
    for name, g in structure_graphs():
        tiles = ref.build_tiles(g)
        rec = {
            "name": name,
            "graph": gjson(g),
            "degree": ref.degree_vector(g).tolist(),
            "tiles": {
                "rows": [t.tile_row for t in tiles.tiles],
                "cols": [t.tile_col for t in tiles.tiles],
                "bitmaps": [hex(t.bitmap) for t in tiles.tiles],
                "values": np.concatenate([t.weights for t in tiles.tiles]).tolist() if tiles.tiles else [],
                "dump": ref.dump_tiles(tiles),
            },
            "pbr": {},
        }
        for seed in (0, 3):
            perm = ref.pbr_reorder(g, seed=seed)
            rec["pbr"][str(seed)] = perm.forward.tolist()
            rec["pbr_tiles_" + str(seed)] = ref.build_tiles(ref.apply_permutation(g, perm)).tile_count
        if name == "four_node":
            rec["pbr_t2"] = ref.pbr_reorder(g, seed=0, t=2).forward.tolist()
        out.append(rec)
        print("structure", name, g.node_count, flush=True)
    return out


def kernel_cases():
    rng = np.random.default_rng(200)
    cases = []
    for trial in range(24):
        labeled = trial % 2 == 0
        ga = random_graph(rng, int(rng.integers(1, 25)), labeled=labeled)
        gb = random_graph(rng, int(rng.integers(1, 25)), labeled=labeled)
        cases.append((f"rand{trial}", ga, gb, "delta:0.5" if labeled else None,
                      "se:1.0" if labeled else None, None))
    for trial in range(4):
        ga = random_graph(rng, int(rng.integers(5, 30)), labeled=True, q_range=(0.0005, 0.001))
        gb = random_graph(rng, int(rng.integers(5, 30)), labeled=True, q_range=(0.0005, 0.001))
        cases.append((f"smallq{trial}", ga, gb, "delta:0.5", "se:1.0", None))
    for trial in range(3):
        ga = random_graph(rng, int(rng.integers(5, 20)), labeled=True, cat_edges=True)
        gb = random_graph(rng, int(rng.integers(5, 20)), labeled=True, cat_edges=True)
        cases.append((f"catedge{trial}", ga, gb, "delta:0.7", "delta:0.3", None))
    for trial in range(3):
        ga = random_graph(rng, int(rng.integers(5, 20)), labeled=True, edge_dim=3, vec_nodes=True)
        gb = random_graph(rng, int(rng.integers(5, 20)), labeled=True, edge_dim=3, vec_nodes=True)
        cases.append((f"vec{trial}", ga, gb, "delta:0.6", "se:0.5", None))
    for trial in range(3):
        ga = random_graph(rng, int(rng.integers(5, 20)), labeled=True)
        gb = random_graph(rng, int(rng.integers(5, 20)), labeled=True)
        cases.append((f"poly{trial}", ga, gb, "const1", "poly:1.0,-0.3,0.02", None))
    for trial in range(2):
        ga = random_graph(rng, int(rng.integers(10, 30)), labeled=True, density=0.15)
        gb = random_graph(rng, int(rng.integers(10, 30)), labeled=True, density=0.15)
        cases.append((f"pbr{trial}", ga, gb, "delta:0.5", "se:1.0", "pbr"))
    mrng = np.random.default_rng(7165)
    for trial in range(6):
        ga = to_ref(synth.molecule(mrng, int(mrng.integers(4, 24))))
        gb = to_ref(synth.molecule(mrng, int(mrng.integers(4, 24))))
        cases.append((f"mol{trial}", ga, gb, "delta:0.5", "se:1.0", None))
    single_a = ref.LabeledGraph.from_edges(1, [], node_labels=np.array([0]), stop_prob=[0.3], start_prob=[1.0])
    single_b = ref.LabeledGraph.from_edges(1, [], node_labels=np.array([1]), stop_prob=[0.3], start_prob=[1.0])
    cases.append(("single_node", single_a, single_b, "delta:0.8", None, None))
    p2 = ref.LabeledGraph.from_edges(2, [(0, 1, 1.0)], stop_prob=[0.5, 0.5])
    cases.append(("p2", p2, p2, None, None, None))
    return cases


def make_kernels():
    out = []
    for name, ga, gb, vs, es, reo in kernel_cases():
        vk = None if vs is None else ref.kernel_from_spec(vs).with_role("vertex")
        ek = None if es is None else ref.kernel_from_spec(es).with_role("edge")
        res = ref.kernel(ga, gb, vk, ek, reorder=reo, seed=0)
        out.append({
            "name": name, "a": gjson(ga), "b": gjson(gb), "vkernel": vs, "ekernel": es,
            "reorder": reo, "tol": 1e-10,
            "value": res.value, "iterations": res.iterations, "residual": res.final_residual,
            "converged": res.converged, "nodewise": res.nodewise.tolist(),
        })
        print("kernel", name, res.iterations, flush=True)
    return out


def make_gram():
    ds = [to_ref(g) for g in synth.config1()]
    vk = ref.KroneckerDelta(0.5).with_role("vertex")
    ek = ref.SquareExponential(1.0).with_role("edge")
    res = ref.compute_gram(ds, vk, ek)
    small = [random_graph(np.random.default_rng(31 + k), 10) for k in range(5)]
    res_u = ref.compute_gram(small)
    return {
        "config1": {"graphs": [gjson(g) for g in ds], "vkernel": "delta:0.5", "ekernel": "se:1.0",
                    "matrix": res.matrix.tolist(), "iterations": res.iterations.tolist(),
                    "converged": res.converged.tolist(), "order": [list(p) for p in res.order],
                    "normalized": ref.normalize_gram(res.matrix).tolist()},
        "unlabeled5": {"graphs": [gjson(g) for g in small], "matrix": res_u.matrix.tolist(),
                       "iterations": res_u.iterations.tolist()},
        "schedule": {
            "uniform": ref.schedule_pairs([4, 4, 4], [6, 6, 6]),
            "giant": ref.schedule_pairs([4, 100, 4, 4], [6, 2000, 6, 6]),
            "mixed": ref.schedule_pairs([10, 20, 10, 7, 3], [30, 120, 20, 14, 2]),
        },
    }


def ref_kernel(spec, role):
    """Extended spec (prod:K1|K2, rconv:K) -> the reference's ProductComposite / RConvolution objects."""
    if spec is None:
        return None
    head, _, rest = spec.partition(":")
    if head == "prod":
        k = ref.ProductComposite([ref.kernel_from_spec(p) for p in rest.split("|")])
    elif head == "rconv":
        k = ref.RConvolution(ref.kernel_from_spec(rest))
    else:
        k = ref.kernel_from_spec(spec)
    return k.with_role(role)


def composite_graph(rng, n, edge_dim, node_dim, density=0.3, w_range=(0.2, 2.0), q_range=(0.2, 0.9)):
    """Vector-labelled graph: node labels small ints (element, charge); edge labels
    (length, bond order) for edge_dim 2, three lengths for edge_dim 3."""
    edges, el = [], []
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < density:
                edges.append((i, j, float(rng.uniform(*w_range))))
                d = float(rng.uniform(0.5, 2.0))
                el.append([d, float(rng.integers(1, 4))] if edge_dim == 2 else
                          [d, d * float(rng.uniform(0.5, 1.5)), float(rng.uniform(0.0, 2.0))])
    nl = rng.integers(0, 3, size=(n, node_dim)).astype(float)
    return ref.LabeledGraph.from_edges(n, edges, node_labels=nl, edge_labels=np.array(el) if edges else None,
                                       start_prob=rng.uniform(0.1, 1.0, size=n),
                                       stop_prob=rng.uniform(*q_range, size=n))


def make_composite():
    """ProductComposite / RConvolution pairs through the reference kernel() (composite.json)."""
    rng = np.random.default_rng(175)
    cases = []
    for trial in range(4):
        ga = composite_graph(rng, int(rng.integers(5, 22)), 2, 2)
        gb = composite_graph(rng, int(rng.integers(5, 22)), 2, 2)
        cases.append((f"prod{trial}", ga, gb, "prod:delta:0.5|delta:0.8", "prod:se:1.0|delta:0.5"))
    # RConvolution values reach dim^2 (the kernel's range exceeds 1, basekernels.py:217-219): light
    # weights and large q keep these product systems positive definite
    for trial in range(3):
        kw = dict(w_range=(0.05, 0.2), q_range=(0.5, 0.9))
        ga = composite_graph(rng, int(rng.integers(5, 18)), 3, 2, **kw)
        gb = composite_graph(rng, int(rng.integers(5, 18)), 3, 2, **kw)
        cases.append((f"rconv{trial}", ga, gb, "delta:0.5", "rconv:se:0.7"))
    kw = dict(w_range=(0.05, 0.2), q_range=(0.5, 0.9))
    ga = composite_graph(rng, 12, 3, 1, **kw)
    gb = composite_graph(rng, 15, 3, 1, **kw)
    cases.append(("rconv_vertex", ga, gb, "rconv:delta:0.5", "rconv:se:0.7"))
    ga = composite_graph(rng, 30, 2, 2, density=0.2)
    gb = composite_graph(rng, 26, 2, 2, density=0.2)
    cases.append(("prod_poly", ga, gb, "prod:const1|delta:0.5", "prod:poly:1.0,-0.3,0.02|se:0.5"))
    out = []
    for name, ga, gb, vs, es in cases:
        res = ref.kernel(ga, gb, ref_kernel(vs, "vertex"), ref_kernel(es, "edge"))
        out.append({"name": name, "a": gjson(ga), "b": gjson(gb), "vkernel": vs, "ekernel": es, "tol": 1e-10,
                    "value": res.value, "iterations": res.iterations, "nodewise": res.nodewise.tolist()})
        print("composite", name, res.iterations, flush=True)
    return out


def make_spatial():
    """Reference spatial_graph (graphio.py:211-240) on seeded point clouds (spatial.json)."""
    from mgksolver.graphio import PointCloud, spatial_graph

    rng = np.random.default_rng(211)
    out = []
    for n, dim, cutoff in ((1, 3, 2.0), (5, 2, 0.7), (40, 3, 0.45), (150, 3, 0.3), (90, 2, 0.2)):
        pts = rng.random((n, dim)) * (1.0 + 0.3 * rng.random())
        labels = rng.integers(0, 4, size=n)
        g = spatial_graph(PointCloud(pts, labels), cutoff)
        out.append({"points": pts.tolist(), "labels": labels.tolist(), "cutoff": cutoff,
                    "ei": np.asarray(g.edges_i).tolist(), "ej": np.asarray(g.edges_j).tolist(),
                    "w": np.asarray(g.weights).tolist(),
                    "d": [] if g.edge_labels is None else np.asarray(g.edge_labels).reshape(-1).tolist()})
    return out


def main():
    if sys.argv[1:] == ["spatial"]:
        (HERE / "spatial.json").write_text(json.dumps(make_spatial()))
        print("done")
        return
    if sys.argv[1:] == ["composite"]:
        (HERE / "composite.json").write_text(json.dumps(make_composite()))
        print("done")
        return
    (HERE / "rng.json").write_text(json.dumps(make_rng_vectors(), indent=0))
    (HERE / "structure.json").write_text(json.dumps(make_structure()))
    (HERE / "kernels.json").write_text(json.dumps(make_kernels()))
    (HERE / "gram.json").write_text(json.dumps(make_gram()))
    print("done")


if __name__ == "__main__":
    main()
