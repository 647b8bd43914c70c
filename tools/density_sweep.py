"""Per-tile-density primitive sweep (BASELINE configs[3] "per-tile-density primitive
throughput"; the paper's tile-primitive analysis, PAPER.md:892-905 / product.py:38-66).

Synthetic graphs whose every non-empty octile holds exactly k nonzeros: n = 8R nodes, tile row I
has tiles (I, I-1) and (I, I+1) (mod R), each with k random positions (the mirrored tile gets the
transposed pattern).  For every (k_a, k_b) the device solves pairs of such graphs (mgk_pairs; warp
class at R = 3, panel class at R = 16) and we report the useful-work throughput

  effective TFLOP/s = sum I * (X S_a S_b + 15 n m) / t      (X = 7 SE-labeled, 3 unlabeled)

against the live FFMA peak, MUFU ex2/s against the live ex2 peak (SE), the dense-tile-equivalent
TFLOP/s (I X 4096 T_a T_b / t: what an 8x8 dense tile-pair primitive would issue) and the
reference's primitive choice for the cell (select_tile_kernel with its thresholds).

    python tools/density_sweep.py [out.json]       (GPU; ~1 min)
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1910_06310_b200 as mgk  # noqa: E402
from paper_1910_06310_b200 import native  # noqa: E402


def tile_graph(rng, R, k, labeled):
    ei, ej = [], []
    for I in range(R):
        J = (I + 1) % R
        if J == I:
            continue
        pos = rng.choice(64, size=k, replace=False)
        r, c = pos // 8, pos % 8
        a, b = 8 * I + r, 8 * J + c
        ei += np.minimum(a, b).tolist()
        ej += np.maximum(a, b).tolist()
    n = 8 * R
    key = np.unique(np.array(ei) * n + np.array(ej))
    ei, ej = key // n, key % n
    w = rng.uniform(0.3, 1.0, len(ei))
    lab = rng.uniform(1.0, 3.0, len(ei)) if labeled else None
    nl = rng.integers(0, 3, n) if labeled else None
    return mgk.LabeledGraph.from_arrays(n, ei, ej, w, node_labels=nl, edge_labels=lab)


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("out", nargs="?", default=str(ROOT / "profiles" / "r02_density_sweep.json"))
    ap.add_argument("--ks", default="1,2,4,8,16,32,48,64")
    ap.add_argument("--classes", default="warp,panel")
    ap.add_argument("--modes", default="labeled,unlabeled")
    args = ap.parse_args()
    out = Path(args.out)
    ctx = native.Context(0)
    fp32, ex2 = ctx.peaks(0)
    ks = [int(k) for k in args.ks.split(",")]
    th = {"labeled": mgk.SelectionThresholds.for_mode("labeled"),
          "unlabeled": mgk.SelectionThresholds.for_mode("unlabeled")}
    cells = []
    # enough pairs per cell to fill the device: 64 x 64 = 4096 warp-class pairs (2368 resident warps),
    # 32 x 32 = 1024 panel-class pairs (~3.5 waves of 296 CTAs)
    for cls, R, per in (("warp", 3, 64), ("panel", 16, 32)):
        if cls not in args.classes.split(","):
            continue
        for labeled in (True, False):
            if ("labeled" if labeled else "unlabeled") not in args.modes.split(","):
                continue
            mode = "labeled" if labeled else "unlabeled"
            X = 7 if labeled else 3
            vs, es = ("delta:0.5", "se:1.0") if labeled else (None, None)
            tol = 1e-10 if labeled else 1e-6
            rng = np.random.default_rng(1234 + R + labeled)
            groups = {k: [tile_graph(rng, R, k, labeled) for _ in range(per)] for k in ks}
            for ka in ks:
                for kb in ks:
                    if kb < ka:
                        continue
                    ga, gb = groups[ka], groups[kb]
                    if cls == "warp" and max(2 * g.edge_count for g in ga + gb) > 320:
                        continue
                    ds = ga + gb
                    pk = native.PackedDataset(ds)
                    ctx.upload(pk)
                    ctx.set_kernels(vs, es)
                    a = np.repeat(np.arange(per), per).astype(np.int32)
                    b = (per + np.tile(np.arange(per), per)).astype(np.int32)
                    ctx.pairs(a, b, tol)  # warm-up
                    best = None
                    for _ in range(3):
                        val, it, res, cv, _ = ctx.pairs(a, b, tol)
                        ms, _ = ctx.last_timing()
                        best = ms if best is None else min(best, ms)
                    S = np.array([2.0 * g.edge_count for g in ds])
                    n = np.array([float(g.node_count) for g in ds])
                    T = np.array([2.0 * R for _ in ds])
                    I = it.astype(np.float64)
                    flops = float(np.sum(I * (X * S[a] * S[b] + 15 * n[a] * n[b])))
                    contrib = float(np.sum(I * S[a] * S[b]))
                    dense = float(np.sum(I * X * 4096 * T[a] * T[b]))
                    t = best * 1e-3
                    cells.append({
                        "class": cls, "mode": mode, "nnz_a": ka, "nnz_b": kb, "n": 8 * R, "pairs": len(a),
                        "ms": best, "converged": bool(np.all(cv)), "mean_iterations": float(I.mean()),
                        "reference_primitive": mgk.select_tile_kernel(ka, kb, mode, th[mode]),
                        "eff_tflops": flops / t / 1e12, "fp32_frac": flops / t / 1e12 / fp32,
                        "contrib_per_s": contrib / t,
                        "ex2_frac": (contrib / t / 1e12 / ex2) if labeled else None,
                        "dense_tile_tflops": dense / t / 1e12,
                    })
                    c = cells[-1]
                    print(f"{cls:5s} {mode:9s} {ka:2d}x{kb:2d} {c['reference_primitive']:13s} "
                          f"{c['eff_tflops']:6.2f} TF/s ({100 * c['fp32_frac']:4.1f}% FP32"
                          + (f", {100 * c['ex2_frac']:4.1f}% ex2" if labeled else "") + ")"
                          f"  dense-eq {c['dense_tile_tflops']:7.1f} TF/s", flush=True)
    out.write_text(json.dumps({"fp32_peak_tflops": fp32, "ex2_peak_tops": ex2, "when": time.strftime("%F %T"),
                               "cells": cells, "doc": __doc__}, indent=1))


if __name__ == "__main__":
    main()
