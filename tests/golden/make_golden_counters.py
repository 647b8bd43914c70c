"""Golden cost counters from the REAL reference (build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_counters.py

Writes ``counters.json``: ``KernelResult.counters`` of reference ``kernel()`` calls
(ProductOperator counters, product.py:212-272, 423-436: default models in labeled and
unlabeled mode, a custom CostModel / SelectionThresholds, force_dense_stream, a PBR-reordered
pair) and ``predict_costs`` cells (costs.py:74-128) for the four primitives.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from make_golden import gjson, random_graph, ref, to_ref  # noqa: F401  (ref: the reference package)
from paper_1910_06310_b200 import synth

HERE = Path(__file__).resolve().parent


def rep(c):
    return {k: getattr(c, k) for k in ("flops", "t1_load", "t1_store", "t2_load", "t2_store", "tile_pairs", "ai1",
                                       "ai2")}


def main():
    rng = np.random.default_rng(2701)
    cases = []
    mol = [synth.molecule(rng, n) for n in (9, 17, 23)]
    prot = [synth.protein(rng, n) for n in (40, 64)]
    er = [random_graph(rng, n, density=d) for n, d in ((20, 0.3), (33, 0.6), (12, 0.9))]
    pairs = [("mol_l", mol[0], mol[1], "delta:0.5", "se:1.0", {}), ("mol_l2", mol[2], mol[1], None, "se:1.0", {}),
             ("prot_l", prot[0], prot[1], "delta:0.5", "se:1.0", {}), ("er_u", er[0], er[1], None, None, {}),
             ("er_u_dense", er[1], er[2], None, None, {}),
             ("er_force", er[0], er[2], None, None, {"force_dense_stream": True}),
             ("prot_model", prot[0], mol[2], "delta:0.5", "se:1.0",
              {"cost_model": {"E": 8, "F": 8, "X": 10, "t": 8, "r": 4},
               "thresholds": {"sparse_min_max": 6, "sparse_max_max": 30, "dense_min": 20}}),
             ("prot_pbr", prot[1], prot[0], "delta:0.5", "se:1.0", {"reorder": "pbr"})]
    for name, ga, gb, vs, es, opt in pairs:
        opt = dict(opt)
        reorder = opt.pop("reorder", None)
        ops = {}
        if "cost_model" in opt:
            ops["cost_model"] = ref.CostModel(**opt["cost_model"])
        if "thresholds" in opt:
            ops["thresholds"] = ref.SelectionThresholds(**opt["thresholds"])
        if "force_dense_stream" in opt:
            ops["force_dense_stream"] = True
        r = ref.kernel(to_ref(ga), to_ref(gb), ref.kernel_from_spec(vs) if vs else None,
                       ref.kernel_from_spec(es) if es else None, ref.SolverConfig(tolerance=1e-8), reorder=reorder,
                       operator_options=ops or None)
        cases.append({"name": name, "a": gjson(ga), "b": gjson(gb), "vkernel": vs, "ekernel": es, "tol": 1e-8,
                      "reorder": reorder, "options": opt, "iterations": r.iterations, "counters": rep(r.counters)})
    predict = []
    for model in ({"E": 0, "F": 4, "X": 3, "t": 8, "r": 8}, {"E": 8, "F": 4, "X": 10, "t": 8, "r": 4}):
        for n, m in ((16, 16), (24, 40), (13, 7)):
            for prim in ref.costs.PRIMITIVES:
                predict.append({"model": model, "n": n, "m": m, "primitive": prim,
                                "report": rep(ref.costs.predict_costs(ref.CostModel(**model), n, m, prim))})
    (HERE / "counters.json").write_text(json.dumps({"kernels": cases, "predict": predict}))


if __name__ == "__main__":
    main()
