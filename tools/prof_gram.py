"""Profiling driver: one device Gram of a config2 subset (for ncu)."""
import sys, time
sys.path.insert(0, '.')
from paper_1910_06310_b200 import native, synth
count = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ds = synth.config2(count=count)
ctx = native.Context(0)
ctx.upload(native.PackedDataset(ds))
ctx.set_kernels("delta:0.5", "se:1.0")
for r in range(reps):
    ctx.gram(1e-10, fetch=False)
    print("solve ms", ctx.last_timing(), flush=True)
