"""Device Gram of one config-4 density bucket (25 RGGs, shuffled + device PBR): solve time per repetition.

    python tools/prof_c4.py [degree] [reps] [count] [se]
"""
import sys

sys.path.insert(0, ".")
from paper_1910_06310_b200 import apply_permutation, native, pbr_reorder_many, synth  # noqa: E402

deg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
count = int(sys.argv[3]) if len(sys.argv) > 3 else 25
se = len(sys.argv) > 4 and sys.argv[4] == "se"
ds = synth.config4(count=count, seed=100 + (4, 8, 16, 32).index(deg), degrees=(deg,))
perms = pbr_reorder_many(ds, seed=0)
ds = [apply_permutation(g, p) for g, p in zip(ds, perms)]
ctx = native.Context(0)
ctx.upload(native.PackedDataset(ds))
ctx.set_kernels(None, "se:1.0" if se else None)
for _ in range(reps):
    ctx.gram(1e-10 if se else 1e-6, fetch=False)
    ms, nl = ctx.last_timing()
    print(f"deg{deg}{' se' if se else ''}: solve ms {ms:.1f} ({count * (count + 1) // 2 / ms * 1e3:.2f} pairs/s)", flush=True)
