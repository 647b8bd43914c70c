"""Probe: device solve time for medium / large pairs (configs 3-5 shapes).

usage: python tools/probe_sizes.py [c3pairs] [c4pairs] [c4_reorder]
Prints per-class pairs/s and effective TFLOP/s from mgk_pairs' device timing.
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1910_06310_b200 import native, synth  # noqa: E402


def make_ctx(name, ds, reorder):
    ctx = native.Context(0)
    ctx.upload(native.PackedDataset(ds))
    ctx.set_kernels(None, None)
    if reorder:
        t0 = time.time()
        ctx.reorder_pbr(0, True)
        print(f"{name}: PBR reorder of {len(ds)} graphs {time.time() - t0:.2f} s", flush=True)
    return ctx


def run(name, ctx, ds, vk, ek, pairs, tol):
    ctx.set_kernels(vk, ek)
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
          f"iters {it.min()}..{it.max()}, eff {flops / ms / 1e9:.2f} TFLOP/s, conv {cv.mean():.3f}", flush=True)


if __name__ == "__main__":
    c3 = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    c4 = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    c4_reorder = len(sys.argv) > 3 and sys.argv[3] == "1"
    rng = np.random.default_rng(0)
    if c3:
        ds3 = synth.config3(count=40)
        ctx = make_ctx("C3", ds3, True)
        pairs = [tuple(sorted(rng.choice(40, 2))) for _ in range(c3)]
        run("C3", ctx, ds3, "delta:0.5", "se:1.0", pairs, 1e-10)
        ds5 = synth.config5(count=400, seed=1)
        ctx = make_ctx("C5", ds5, False)
        pairs = [tuple(sorted(rng.choice(400, 2))) for _ in range(20000)]
        run("C5-mixed", ctx, ds5, "delta:0.5", "se:1.0", pairs, 1e-10)
    if c4:
        ds4 = synth.config4(count=8, degrees=(4, 8, 16, 32))
        ctx = make_ctx("C4", ds4, c4_reorder)
        for k in range(min(c4, 4)):
            pairs = [(2 * k, 2 * k + 1)]
            run(f"C4-unlab deg{4 << k}", ctx, ds4, None, None, pairs, 1e-6)
            run(f"C4-se deg{4 << k}", ctx, ds4, None, "se:1.0", pairs, 1e-10)
