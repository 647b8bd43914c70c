"""Profiling driver for ncu: one mgk_pairs call of a config-3 or config-4 workload.

usage: python tools/prof_pairs.py c3 [npairs] | c4 [degree]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1910_06310_b200 import native, synth  # noqa: E402

which = sys.argv[1]
ctx = native.Context(0)
if which == "c3":
    ds = synth.config3(count=40)
    npairs = int(sys.argv[2]) if len(sys.argv) > 2 else 296
    rng = np.random.default_rng(0)
    pairs = [tuple(sorted(rng.choice(40, 2))) for _ in range(npairs)]
    vk, ek, tol = "delta:0.5", "se:1.0", 1e-10
else:
    deg = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    ds = synth.config4(count=2, degrees=(deg,))
    pairs = [(0, 1)]
    vk, ek, tol = None, "se:1.0", 1e-10
ctx.upload(native.PackedDataset(ds))
ctx.set_kernels(None, None)
ctx.reorder_pbr(0, True)
ctx.set_kernels(vk, ek)
a = np.array([p[0] for p in pairs], np.int32)
b = np.array([p[1] for p in pairs], np.int32)
val, it, res, cv, _ = ctx.pairs(a, b, tol)
print("solve ms", ctx.last_timing(), "iters", it.min(), it.max())
