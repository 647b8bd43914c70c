"""Which small pairs need the FP64 tiny path?  Runs all pairs of small
config2-style molecules in FP32 (MGK_TINY_NM=0) and compares iteration
counts with the float64 oracle."""
import os, sys
os.environ["MGK_TINY_NM"] = sys.argv[1] if len(sys.argv) > 1 else "0"
sys.path.insert(0, ".")
import numpy as np
from paper_1910_06310_b200 import native, synth
from oracle import mgk_oracle as O
rng = np.random.default_rng(5)
ds = [synth.molecule(rng, int(n)) for n in rng.integers(4, 13, size=90)]
ctx = native.Context(0)
ctx.upload(native.PackedDataset(ds))
ctx.set_kernels("delta:0.5", "se:1.0")
K, it, cv = ctx.gram(1e-10)
bad = []
worst = 0
for a in range(len(ds)):
    for b in range(a, len(ds)):
        o = O.solve_pcg(ds[a], ds[b], ("delta", 0.5), ("se", 1.0))
        d = int(it[a, b]) - o.iterations
        worst = max(worst, abs(K[a, b] - o.value) / o.value)
        if abs(d) > 1:
            bad.append((ds[a].node_count, ds[b].node_count, a == b, o.iterations, d))
print("pairs", len(ds) * (len(ds) + 1) // 2, "bad", len(bad), "worst rel", worst)
for x in sorted(bad): print(x)
