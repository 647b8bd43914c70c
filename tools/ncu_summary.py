"""Summarise an ncu --set full report into JSON (committed under profiles/).

usage: ncu_summary.py <report.ncu-rep> <out.json> [kernel-substring]
Records per kernel launch: duration, DRAM bytes read+written, SM / memory
throughput, issue activity, occupancy, registers.  bench.py reads
``solver_dram_bytes_per_launch`` from the newest summary as roofline.traffic.
"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
pat = sys.argv[3] if len(sys.argv) > 3 else "k_pcg_warp"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "shared_wavefronts",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}
idx = {k: hdr.index(k) for k in want if k in hdr}
launches = []
for r in data:
    name = r[hdr.index("Kernel Name")]
    if pat not in name:
        continue
    rec = {"kernel": name[:120]}
    for k, i in idx.items():
        v = r[i].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            pass
        rec[want[k]] = v
        rec[want[k] + "_unit"] = units[i]
    launches.append(rec)


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return v * scale.get(u, 1)


summary = {"report": rep, "kernel_filter": pat, "launches": launches}
if launches:
    L = launches[0]
    rd = to_bytes(L.get("dram_read", 0), L.get("dram_read_unit", "byte"))
    wr = to_bytes(L.get("dram_write", 0), L.get("dram_write_unit", "byte"))
    summary["solver_dram_bytes_per_launch"] = rd + wr
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "launches"}, indent=1))
for L in launches:
    print({k: v for k, v in L.items() if not k.endswith("_unit")})
