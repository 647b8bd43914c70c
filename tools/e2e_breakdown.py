"""Where the end-to-end config-2 Gram time goes: validation, packing, upload + octiles, device solve,
D2H of the N x N outputs (host wall clock per stage, after one warm-up call).

    python tools/e2e_breakdown.py [count]
"""
import sys
import time

sys.path.insert(0, ".")
import paper_1910_06310_b200 as mgk  # noqa: E402
from paper_1910_06310_b200 import gram as G, native, synth  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 7165
ds = synth.config2(count=count)
mgk.compute_gram(ds, "delta:0.5", "se:1.0")  # warm-up (context, kernels, pinned buffers)
for _ in range(2):
    t0 = time.perf_counter()
    G._validate(ds)
    t1 = time.perf_counter()
    packed = native.PackedDataset(ds)
    t2 = time.perf_counter()
    ctx = G.context(0)
    ctx.upload(packed)
    ctx.set_kernels("delta:0.5", "se:1.0")
    t3 = time.perf_counter()
    K, it, cv = ctx.gram(1e-10)
    t4 = time.perf_counter()
    ms, _ = ctx.last_timing()
    t5 = time.perf_counter()
    r = mgk.compute_gram(ds, "delta:0.5", "se:1.0")
    t6 = time.perf_counter()
    print(f"validate {1e3 * (t1 - t0):.1f} ms, pack {1e3 * (t2 - t1):.1f} ms, upload+kernels {1e3 * (t3 - t2):.1f} ms, "
          f"gram call {1e3 * (t4 - t3):.1f} ms (device solve {ms:.1f} ms), compute_gram total {1e3 * (t6 - t5):.1f} ms "
          f"[K {K.dtype} it {it.dtype} conv {cv.dtype}]", flush=True)
