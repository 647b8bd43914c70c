import sys, numpy as np
sys.path.insert(0, '.')
import paper_1910_06310_b200 as mgk
from oracle import mgk_oracle as O
from paper_1910_06310_b200 import synth
ds = synth.config2(count=10, seed=1)
res = mgk.compute_gram(ds, "delta:0.5", "se:1.0")
for a in range(10):
    for b in range(a, 10):
        o = O.solve_pcg(ds[a], ds[b], ("delta", 0.5), ("se", 1.0))
        rel = abs(res.matrix[a, b] - o.value) / abs(o.value)
        flag = "" if (rel < 1e-5 and abs(int(res.iterations[a,b]) - o.iterations) <= 1) else "  <-- BAD"
        print(a, b, ds[a].node_count, ds[b].node_count, 2*ds[a].edge_count, 2*ds[b].edge_count, f"{res.matrix[a,b]:.8e} {o.value:.8e} rel={rel:.1e}", res.iterations[a,b], o.iterations, flag)
# single pair via kernel()
for a, b in [(0, 1), (2, 3)]:
    k = mgk.kernel(ds[a], ds[b], "delta:0.5", "se:1.0")
    o = O.solve_pcg(ds[a], ds[b], ("delta", 0.5), ("se", 1.0))
    print("kernel", a, b, k.value, o.value, k.iterations, o.iterations, np.max(np.abs(k.nodewise - o.nodewise)) / np.max(np.abs(o.nodewise)))
# unlabeled
res = mgk.compute_gram(ds[:4], cfg=mgk.SolverConfig(tolerance=1e-6))
for a in range(4):
    for b in range(a, 4):
        o = O.solve_pcg(ds[a], ds[b], None, None, tol=1e-6)
        print("unl", a, b, res.matrix[a,b], o.value, res.iterations[a,b], o.iterations)
