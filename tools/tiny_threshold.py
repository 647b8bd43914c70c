"""Which small pairs need the FP64 tiny path?  All pairs of 200 config-2
molecules on the device at several MGK_TINY_NM thresholds, iteration counts
against the float64 oracle (pool of host cores).

usage: python tools/tiny_threshold.py [graphs]
"""
import multiprocessing as mp
import os
import subprocess
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from oracle import mgk_oracle as O  # noqa: E402
from paper_1910_06310_b200 import synth  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 200
DS = synth.config2(count=G, seed=99)


def oracle(ab):
    a, b = ab
    return O.solve_pcg(DS[a], DS[b], ("delta", 0.5), ("se", 1.0)).iterations


def device(tiny):
    code = ("import sys, numpy as np; sys.path.insert(0, '.');"
            "from paper_1910_06310_b200 import native, synth;"
            f"ds = synth.config2(count={G}, seed=99); ctx = native.Context(0);"
            "ctx.upload(native.PackedDataset(ds)); ctx.set_kernels('delta:0.5', 'se:1.0');"
            "K, it, cv = ctx.gram(1e-10); np.save('/tmp/it.npy', it)")
    subprocess.run([sys.executable, "-c", code], check=True, env={**os.environ, "MGK_TINY_NM": str(tiny)})
    return np.load("/tmp/it.npy")


if __name__ == "__main__":
    pairs = [(a, b) for a in range(G) for b in range(a, G)]
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        ref = np.array(pool.map(oracle, pairs, chunksize=64))
    n = np.array([g.node_count for g in DS])
    for tiny in (0, 64, 128):
        it = device(tiny)
        d = np.array([int(it[a, b]) for a, b in pairs]) - ref
        bad = np.abs(d) > 1
        nm = np.array([n[a] * n[b] for a, b in pairs])
        print(f"MGK_TINY_NM={tiny}: {len(pairs)} pairs, |d_iter|>1: {bad.sum()}, nm of those: "
              f"{sorted(set(nm[bad].tolist()))[:20]}, diff hist {np.unique(d, return_counts=True)}", flush=True)
