"""Profiling driver: one device Gram of a config-5 subset (mixed sizes; for ncu launch lists)."""
import sys

sys.path.insert(0, ".")
from paper_1910_06310_b200 import native, synth  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
ds = synth.config5(count=count)
ctx = native.Context(0)
ctx.upload(native.PackedDataset(ds))
ctx.set_kernels("delta:0.5", "se:1.0")
ctx.gram(1e-10, fetch=False)
print("solve ms", ctx.last_timing(), flush=True)
