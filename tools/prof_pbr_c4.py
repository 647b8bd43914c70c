"""Device PBR wall time on the config-4 graphs (100 RGGs, n 2k-5k, 4 density buckets)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1910_06310_b200 import pbr_reorder_many, synth  # noqa: E402

for d in (4, 8, 16, 32):
    gs = synth.config4(count=25, seed=100 + (4, 8, 16, 32).index(d), degrees=(d,))
    t0 = time.perf_counter()
    pbr_reorder_many(gs, seed=0)
    print(f"deg{d}: 25 graphs PBR {time.perf_counter() - t0:.2f} s", flush=True)
