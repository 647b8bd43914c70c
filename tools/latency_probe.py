"""Per-call latency of the public API on small inputs (config 1 Gram, single-pair kernel()).

    python tools/latency_probe.py      (GPU)
Prints median wall times over repeated calls after one warm-up, with a phase breakdown of
compute_gram (validate+pack / upload / set_kernels / solve+D2H).
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1910_06310_b200 as mgk  # noqa: E402
from paper_1910_06310_b200 import native, synth  # noqa: E402
from paper_1910_06310_b200.gram import _validate  # noqa: E402
from paper_1910_06310_b200.solver import context  # noqa: E402


def med(f, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(ts))


def main():
    ds = synth.config1()
    mgk.compute_gram(ds, "delta:0.5", "se:1.0")
    print(f"compute_gram config 1 (136 pairs): {med(lambda: mgk.compute_gram(ds, 'delta:0.5', 'se:1.0'), 20):.2f} ms")
    ctx = context(0)
    pk = native.PackedDataset(ds)
    print(f"  validate        {med(lambda: _validate(ds), 20):.2f} ms")
    print(f"  pack            {med(lambda: native.PackedDataset(ds), 20):.2f} ms")
    print(f"  upload          {med(lambda: ctx.upload(pk), 20):.2f} ms")

    def solve():
        ctx.upload(pk)
        ctx.set_kernels("delta:0.5", "se:1.0")
        ctx.gram(1e-10)
    print(f"  upload+prepare+solve+D2H {med(solve, 20):.2f} ms  (device solve {ctx.last_timing()[0]:.3f} ms)")
    print(f"  solve only (prepared)    {med(lambda: ctx.gram(1e-10), 20):.2f} ms")
    ga, gb = ds[0], ds[1]
    mgk.kernel(ga, gb, "delta:0.5", "se:1.0")
    print(f"kernel() single pair: {med(lambda: mgk.kernel(ga, gb, 'delta:0.5', 'se:1.0'), 50):.2f} ms")


if __name__ == "__main__":
    main()
