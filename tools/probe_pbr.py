"""Probe: device PBR wall time on config-3/4 shaped graphs."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_1910_06310_b200 import native, synth  # noqa: E402


def run(name, ds):
    ctx = native.Context(0)
    ctx.upload(native.PackedDataset(ds))
    ctx.set_kernels(None, None)
    t0 = time.time()
    fwd = ctx.reorder_pbr(0, False)
    dt = time.time() - t0
    ident = sum(int(np.all(fwd[o:o + g.node_count] == np.arange(g.node_count)))
                for o, g in zip(np.cumsum([0] + [g.node_count for g in ds[:-1]]), ds))
    print(f"{name}: {len(ds)} graphs, n {min(g.node_count for g in ds)}..{max(g.node_count for g in ds)}, "
          f"PBR {dt:.2f} s, identity fallbacks {ident}", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c3", "c4"]
    if "c3" in which:
        run("C3x148", synth.config3(count=148))
    if "c4" in which:
        for d in (4, 8, 16, 32):
            run(f"C4 deg{d} x2", synth.config4(count=2, degrees=(d,)))
