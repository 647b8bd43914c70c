"""Profiling driver: device Gram of a config-3 subset (shuffled proteins, device PBR applied), repeated.

    python tools/prof_c3.py [count] [reps]
"""
import sys

sys.path.insert(0, ".")
from paper_1910_06310_b200 import apply_permutation, native, pbr_reorder_many, synth  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 150
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ds = synth.config3(count=count)
perms = pbr_reorder_many(ds, seed=0)
ds = [apply_permutation(g, p) for g, p in zip(ds, perms)]
ctx = native.Context(0)
ctx.upload(native.PackedDataset(ds))
ctx.set_kernels("delta:0.5", "se:1.0")
for _ in range(reps):
    ctx.gram(1e-10, fetch=False)
    ms, nl = ctx.last_timing()
    print(f"solve ms {ms:.1f} ({count * (count + 1) // 2 / ms * 1e3:.0f} pairs/s)", flush=True)
