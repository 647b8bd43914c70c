"""Attribute ncu SASS-level stall samples / executed instructions to CUDA source lines.

usage: ncu_by_line.py <ncu sass csv> <object .o> <kernel-name substring> [top]
The ncu report's SASS addresses are offset from the function start, which is
matched to nvdisasm --print-line-info of the same object build.
"""
import csv, os, re, subprocess, sys, tempfile
from collections import Counter, defaultdict

sass_csv, obj, pat = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
rows = list(csv.reader(open(sass_csv)))
h = rows[1]; ix = {k: i for i, k in enumerate(h)}
data = rows[2:]
addr = [int(r[ix["Address"]], 16) for r in data]
base = min(addr)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
out = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)], capture_output=True, text=True).stdout
line_of = {}; cur = None; fn = None
for line in out.splitlines():
    m = re.search(r"\.text\.(\S+):", line)
    if m: fn = m.group(1)
    m = re.search(r'//## File "[^"]*/([^"/]+)", line (\d+)', line)
    if m: cur = f"{m.group(1)}:{m.group(2)}"; continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
    if m and fn and pat in fn: line_of[int(m.group(1), 16)] = cur
def f(r, k):
    try: return float(r[ix[k]].replace(",", ""))
    except Exception: return 0.0
samp = Counter(); inst = Counter(); stalls = defaultdict(Counter)
sc = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
for r, a in zip(data, addr):
    ln = line_of.get(a - base, "?")
    samp[ln] += f(r, "Warp Stall Sampling (All Samples)")
    inst[ln] += f(r, "Instructions Executed")
    for k in sc: stalls[ln][k[6:]] += f(r, k)
ts = sum(samp.values()); ti = sum(inst.values())
print(f"mapped {sum(1 for a in addr if (a-base) in line_of)}/{len(addr)} instructions")
for ln, v in samp.most_common(top):
    st = ", ".join(f"{k}:{int(100*x/v)}%" for k, x in stalls[ln].most_common(3)) if v else ""
    print(f"{ln:28s} samples {100*v/ts:5.1f}%  instrs {100*inst[ln]/ti:5.1f}%   {st}")
