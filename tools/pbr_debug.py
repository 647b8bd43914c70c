"""Compare device PBR candidates with the oracle restatement's, stage by stage."""
import os, sys, subprocess, json
sys.path.insert(0, ".")
import numpy as np
sys.path.insert(0, "tests")
from conftest import graph_from_json
from oracle import mgk_oracle as O
names = sys.argv[1].split(",")
recs = [r for r in json.load(open("tests/golden/structure.json")) if r["name"] in names]
graphs = [graph_from_json(r["graph"]) for r in recs]
if os.environ.get("MGK_PBR_DEBUG"):
    import paper_1910_06310_b200 as mgk
    perms = mgk.pbr_reorder_many(graphs, seed=0)
    for r, p in zip(recs, perms):
        print("DEVICE", r["name"], p.forward.tolist() == r["pbr"]["0"])
    sys.exit(0)
out = subprocess.run([sys.executable, __file__, sys.argv[1]], env={**os.environ, "MGK_PBR_DEBUG": "1"},
                     capture_output=True, text=True)
print(out.stdout)
dev = {}
for line in out.stderr.splitlines():
    if line.startswith("PBRDBG"):
        f = line.split()
        dev[int(f[1])] = np.array(list(map(int, f[2:])))
for gi, (r, g) in enumerate(zip(recs, graphs)):
    n = g.node_count
    k = -(-n // 8)
    adj = O.neighbour_lists(g)
    sizes = [8] * (k - 1) + [n - 8 * (k - 1)]
    for c, shuffled in enumerate((False, True)):
        nodes = list(range(n))
        if shuffled:
            O.SplitMix64(0).shuffle(nodes)
        parts = np.empty(n, dtype=np.int64)
        O._recursive(nodes, sizes, adj, 10, parts, 0)
        rp = parts.copy()
        fm = O.fm_refine(g, parts, k, np.array(sizes), 10, adj)
        d = dev.get(gi)
        dc = d[c * n:(c + 1) * n] if d is not None else None
        dp = d[2 * n + c * n: 2 * n + (c + 1) * n] if d is not None else None
        if dp is not None:
            print(r["name"], "cand", c, "recursive parts match:", bool(np.array_equal(dp, rp)))
            if not np.array_equal(dp, rp):
                print("  oracle rp:", rp.tolist())
                print("  device rp:", dp.tolist())
        print(r["name"], "cand", c, "fm match:", None if dc is None else bool(np.array_equal(dc, fm)),
              "obj oracle", O.pair_objective(g, fm), "obj dev", None if dc is None else O.pair_objective(g, dc))
        if dc is not None and not np.array_equal(dc, fm):
            print("  recursive parts (oracle):", rp.tolist())
            print("  fm (oracle):", fm.tolist())
            print("  device     :", dc.tolist())
