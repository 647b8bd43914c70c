"""Probe: device solve time for medium / large pairs (configs 3-5 shapes).

usage: python tools/probe_sizes.py [c3pairs] [c4pairs]
Prints per-class pairs/s and effective GFLOP/s from mgk_pairs' device timing.
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1910_06310_b200 import native, synth  # noqa: E402


def run(name, ds, vk, ek, pairs, tol, reorder=False):
    ctx = native.Context(0)
    ctx.upload(native.PackedDataset(ds))
    ctx.set_kernels(vk, ek)
    if reorder:
        t0 = time.time()
        ctx.reorder_pbr(0, True)
        print(f"{name}: PBR reorder of {len(ds)} graphs {time.time() - t0:.2f} s", flush=True)
    a = np.array([p[0] for p in pairs], np.int32)
    b = np.array([p[1] for p in pairs], np.int32)
    t0 = time.time()
    val, it, res, cv, _ = ctx.pairs(a, b, tol)
    wall = time.time() - t0
    ms, launches = ctx.last_timing()
    S = np.array([2 * g.edge_count for g in ds])
    n = np.array([g.node_count for g in ds])
    x = 7 if ek else 3
    flops = float(np.sum(it * (x * S[a] * S[b] + 15.0 * n[a] * n[b])))
    print(f"{name}: {len(pairs)} pairs, device {ms:.1f} ms ({len(pairs) / ms * 1e3:.1f} pairs/s), wall {wall:.2f} s, "
          f"iters {it.min()}..{it.max()}, eff {flops / ms / 1e9:.1f} TFLOP/s, conv {cv.mean():.3f}",
          flush=True)


if __name__ == "__main__":
    c3 = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    c4 = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    rng = np.random.default_rng(0)
    ds3 = synth.config3(count=40)
    pairs = [tuple(sorted(rng.choice(40, 2))) for _ in range(c3)]
    run("C3", ds3, "delta:0.5", "se:1.0", pairs, 1e-10, reorder=True)
    ds5 = synth.config5(count=400, seed=1)
    pairs = [tuple(sorted(rng.choice(400, 2))) for _ in range(20000)]
    run("C5-mixed", ds5, "delta:0.5", "se:1.0", pairs, 1e-10)
    if c4:
        ds4 = synth.config4(count=8, degrees=(4, 8, 16, 32))
        pairs = [(2 * k, 2 * k + 1) for k in range(min(c4, 4))]
        run("C4-unlab", ds4, None, None, pairs, 1e-6, reorder=len(sys.argv) > 3)
        run("C4-se", ds4, None, "se:1.0", pairs, 1e-10, reorder=len(sys.argv) > 3)
