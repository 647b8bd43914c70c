"""Summarise an ncu source page (SASS) CSV: hottest instructions by stall samples."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = rows[2:]
def f(r, k):
    try: return float(r[idx[k]].replace(',', ''))
    except Exception: return 0.0
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_i = sum(f(r, "Instructions Executed") for r in data)
print("total samples", tot_s, "total warp instrs", tot_i)
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = Counter()
for r in data:
    for k in stall_cols: agg[k] += f(r, k)
print("stall totals:", [(k, round(v / tot_s * 100, 1)) for k, v in agg.most_common(8)])
# opcode mix
ops = Counter(); opi = Counter()
for r in data:
    op = r[idx["Source"]].split()[0] if r[idx["Source"]].strip() else ""
    if op.startswith("@"): op = r[idx["Source"]].split()[1]
    ops[op.split(".")[0]] += f(r, "Warp Stall Sampling (All Samples)")
    opi[op.split(".")[0]] += f(r, "Instructions Executed")
print("by opcode (samples%):", [(k, round(v / tot_s * 100, 1)) for k, v in ops.most_common(15)])
print("by opcode (instr%):", [(k, round(v / tot_i * 100, 1)) for k, v in opi.most_common(15)])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
top = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:n]
for r in top:
    st = sorted(((f(r, k), k[6:]) for k in stall_cols), reverse=True)[:3]
    print(f"{r[idx['Address']]:>6} {f(r,'Warp Stall Sampling (All Samples)')/tot_s*100:5.2f}% ex={f(r,'Instructions Executed'):.3g} "
          f"thr={f(r,'Avg. Predicated-On Threads Executed'):4.1f} {r[idx['Source']][:60]:60s} {[(s[1], int(s[0])) for s in st]}")
