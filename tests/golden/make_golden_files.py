"""Graph files written by the REAL reference (build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_files.py

``files/*.json`` come from the reference's ``save_graph`` (graphio.py:61-93) for a
categorical-labeled, a vector-labeled and an unlabeled graph; ``files/edges.txt`` is an
edge list; ``files/index.json`` records what the reference's ``load_graph`` /
``load_edge_list`` return for them and its ``kernel()`` nodewise field written the way the
CLI writes it (cli.py:65-69, ``files/nodewise.csv``).
"""
import json
from pathlib import Path

import numpy as np

from make_golden import gjson, random_graph, ref, to_ref

OUT = Path(__file__).resolve().parent / "files"


def main():
    OUT.mkdir(exist_ok=True)
    rng = np.random.default_rng(115)
    graphs = {"cat": random_graph(rng, 9, density=0.4, labeled=True),
              "vec": random_graph(rng, 7, density=0.5, edge_dim=3, vec_nodes=True),
              "plain": random_graph(rng, 6, density=0.5)}
    index = {}
    for name, g in graphs.items():
        rg = to_ref(g)
        ref.save_graph(rg, OUT / f"{name}.json")
        index[name] = gjson(ref.load_graph(OUT / f"{name}.json"))
    (OUT / "edges.txt").write_text("# comment line\n0 3 0.5\n3 1   # trailing comment\n\n2 4 1.25\n1 4\n")
    index["edges"] = gjson(ref.load_edge_list(OUT / "edges.txt"))
    ga, gb = ref.load_graph(OUT / "cat.json"), ref.load_graph(OUT / "plain.json")
    ga2 = ref.load_graph(OUT / "cat.json")
    r = ref.kernel(ga, ga2, ref.KroneckerDelta(0.5), ref.SquareExponential(1.0))
    with open(OUT / "nodewise.csv", "w") as fh:
        for row in r.nodewise:
            fh.write(",".join(repr(float(v)) for v in row) + "\n")
    index["nodewise_value"] = r.value
    (OUT / "index.json").write_text(json.dumps(index))


if __name__ == "__main__":
    main()
