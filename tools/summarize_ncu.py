#!/usr/bin/env python3
"""Summarise an ncu --set full report of one kernel into profiles/ (markdown +
json): duration, pipe utilisation, stall reasons, DRAM traffic, occupancy.
Usage: python tools/summarize_ncu.py <report.ncu-rep> <out-prefix> [kernel-regex] [source-note]"""
import csv
import io
import json
import re
import subprocess
import sys

rep, prefix = sys.argv[1], sys.argv[2]
kre = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
if kre:
    ki = hdr.index("Kernel Name")
    data = [r for r in data if kre.search(r[ki])]
d = dict(zip(hdr, data[0]))
u = dict(zip(hdr, units))


def num(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


def to_bytes(k):
    v, unit = num(k), u.get(k, "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return None if v is None else v * scale


dur_ns = num("gpu__time_duration.sum") * ({"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
                                          .get(u.get("gpu__time_duration.sum", "ns"), 1))
rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
stalls = {k.split("issue_stalled_")[1].split("_per_issue")[0]: num(k) for k in hdr
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
top = dict(sorted(((k, v) for k, v in stalls.items() if v), key=lambda kv: -kv[1])[:8])
summary = {
    "kernel": d.get("Kernel Name"), "grid": d.get("Grid Size"), "block": d.get("Block Size"),
    "duration_ms": dur_ns / 1e6,
    "dram_read_bytes": rd, "dram_write_bytes": wr,
    "dram_bytes_per_launch": (rd or 0) + (wr or 0),
    "warp_instructions": num("smsp__inst_executed.sum"),
    "ipc_active": num("sm__inst_executed.avg.per_cycle_active"),
    "issue_active_pct": num("sm__inst_executed.sum.pct_of_peak_sustained_elapsed"),
    "pipe_alu_pct": num("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    "pipe_fma_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "pipe_fmaheavy_pct": num("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    "pipe_lsu_inst_pct": num("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "occupancy_achieved_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
    "l1tex_throughput_pct": num("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
    "l2_throughput_pct": num("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    "l1tex_hit_pct": num("l1tex__t_sector_hit_rate.pct"),
    "top_stalls_per_issue": top,
}
if len(sys.argv) > 4:
    summary["source"] = sys.argv[4]
json.dump(summary, open(prefix + ".json", "w"), indent=1)
with open(prefix + ".md", "w") as f:
    f.write(f"# ncu --set full summary: {summary['kernel']}\n\n")
    f.write(f"source report: `{rep}` (clock-control none)\n\n| metric | value |\n|---|---|\n")
    for k, v in summary.items():
        if k != "top_stalls_per_issue":
            f.write(f"| {k} | {v} |\n")
    f.write("\n## top stall reasons (warps per issued instruction)\n\n| reason | value |\n|---|---|\n")
    for k, v in top.items():
        f.write(f"| {k} | {v:.3f} |\n")
print(json.dumps(summary, indent=1))
