"""Profiling driver: device Gram of the first `count` config-2 molecules, repeated.

    python tools/prof_gram.py [count] [reps]

Prints the device solve time of each repetition (CUDA events around the solver launches).
"""
import sys

sys.path.insert(0, ".")
from paper_1910_06310_b200 import native, synth  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ds = synth.config2(count=count)
ctx = native.Context(0)
ctx.upload(native.PackedDataset(ds))
ctx.set_kernels("delta:0.5", "se:1.0")
for _ in range(reps):
    ctx.gram(1e-10, fetch=False)
    ms, nl = ctx.last_timing()
    print(f"solve ms {ms:.1f} ({count * (count + 1) // 2 / ms * 1e3 / 1e6:.2f} M pairs/s, {nl} launches)", flush=True)
