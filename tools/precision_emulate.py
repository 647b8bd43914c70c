"""Numpy emulation of the device PCG precision schemes against the float64
reference scheme (oracle/mgk_oracle.py, solver.py:77-121), used to choose
kPreciseTol (csrc/mgk_internal.h) and the Laplacian-splitting switch.

    python tools/precision_emulate.py            # reference smallq goldens at tol 1e-8
    python tools/precision_emulate.py --sweep    # unlabeled molecules, q in {0.05, 5e-4}

Schemes: 'v32' FP32 vectors / FP32 XMV / FP64 dots (the warp, panel and grid
solvers), 'v64' FP64 vectors with an FP32 XMV, 'full' FP64 everything with
FP32-rounded weights (the block solver's precise mode).  split=True uses the
Laplacian splitting A p = s p - sum L (p_j - p_i) for the XMV.
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from oracle import mgk_oracle as O  # noqa: E402

f32 = np.float32


def solve(ga, gb, vs, es, tol, scheme, split):
    S = O.ProductSystem(ga, gb, vs, es)
    if scheme == "full":
        S.vals = S.vals.astype(f32).astype(float)
    rows = np.bincount(S.out_idx, weights=S.vals, minlength=S.size)
    s = S.diag - rows
    vals32, diag32 = S.vals.astype(f32), S.diag.astype(f32)

    def xmv32(p):
        p32 = p.astype(f32)
        acc = np.zeros(S.size, f32)
        if split:
            np.add.at(acc, S.out_idx, (vals32 * (p32[S.in_idx] - p32[S.out_idx]).astype(f32)).astype(f32))
            return s * p32.astype(float) - acc
        np.add.at(acc, S.out_idx, (vals32 * p32[S.in_idx]).astype(f32))
        return (diag32 * p32 - acc).astype(f32).astype(float)

    qa, qb = np.asarray(ga.stop_prob), np.asarray(gb.stop_prob)
    b = np.outer(S.d_a * qa, S.d_b * qb).ravel()
    px = np.outer(ga.start_prob, gb.start_prob).ravel()
    eps = tol * tol * float(b @ b)
    V = f32 if scheme == "v32" else float
    x = np.zeros(S.size, V)
    r = b.astype(V)
    rd = (1.0 / S.diag).astype(V)
    z = (r * rd).astype(V)
    p = z.copy()
    rho = float(r.astype(float) @ z.astype(float))
    done = float(r.astype(float) @ r.astype(float)) < eps
    it = 0
    while not done and it < 10 * S.size:
        a = S.apply(p) if scheme in ("ref", "full") else xmv32(p).astype(V)
        it += 1
        alpha = rho / float(p.astype(float) @ a.astype(float))
        x = (x + V(alpha) * p).astype(V)
        r = (r - V(alpha) * a).astype(V)
        if float(r.astype(float) @ r.astype(float)) < eps:
            break
        z = (r * rd).astype(V)
        rn = float(r.astype(float) @ z.astype(float))
        p = (z + V(rn / rho) * p).astype(V)
        rho = rn
    return float(px @ x.astype(float)), it


def goldens():
    from conftest import graph_from_json

    for rec in json.load(open(ROOT / "tests/golden/smallq.json")):
        if rec["tol"] != 1e-8:
            continue
        ga, gb = graph_from_json(rec["a"]), graph_from_json(rec["b"])
        vs = O.parse_spec(rec["vkernel"]) if rec["vkernel"] else None
        es = O.parse_spec(rec["ekernel"]) if rec["ekernel"] else None
        row = [rec["name"], rec["iterations"]]
        for scheme in ("v32", "v64", "full"):
            v, it = solve(ga, gb, vs, es, 1e-8, scheme, True)
            row += [scheme, it, f"{abs(v - rec['value']) / rec['value']:.1e}"]
        print(*row)


def sweep():
    import paper_1910_06310_b200 as mgk
    from paper_1910_06310_b200 import synth

    for q in (0.05, 5e-4):
        rng = np.random.default_rng(12)
        gs = []
        for n in (5, 8, 12, 16, 20, 23, 30, 45):
            g = synth.molecule(rng, n, q=q)
            gs.append(mgk.LabeledGraph.from_arrays(g.node_count, g.edges_i, g.edges_j, g.weights, default_q=q))
        for tol in (1e-6, 3e-7, 1e-7, 1e-8, 1e-10):
            worst = {}
            for i in range(len(gs)):
                for j in range(i, len(gs)):
                    ref = solve(gs[i], gs[j], None, None, tol, "ref", False)[1]
                    for scheme in ("v32", "v64", "full"):
                        d = abs(solve(gs[i], gs[j], None, None, tol, scheme, q < 0.01)[1] - ref)
                        worst[scheme] = max(worst.get(scheme, 0), d)
            print(f"q={q} tol={tol:g} worst iteration difference", worst)


if __name__ == "__main__":
    sweep() if "--sweep" in sys.argv else goldens()
