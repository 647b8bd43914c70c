"""Instruction count per source line of one kernel in a cubin/object (code-size triage)."""
import re, subprocess, sys, tempfile, os
from collections import Counter
obj, pat = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
out = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)], capture_output=True, text=True).stdout
c = Counter(); cur = None; fn = None
for line in out.splitlines():
    m = re.search(r"\.text\.(\S+):", line)
    if m: fn = m.group(1)
    m = re.search(r'//## File "[^"]*/([^"/]+)", line (\d+)', line)
    if m: cur = (m.group(1), int(m.group(2))); continue
    if fn and pat in fn and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line): c[cur] += 1
print("total instrs", sum(c.values()))
for k, v in c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25): print(k, v)
