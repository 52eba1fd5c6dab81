#!/usr/bin/env python
"""Summarise ncu --set full captures (.ncu-rep) into a markdown table for
profiles/: time, DRAM traffic, issue activity, and the shared-memory atomic /
bank-conflict counters the north star asks for.

    python tools/ncu_summary.py OUT.md label=path.ncu-rep [label=path ...]
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "smem atomic wavefronts"),
    ("smsp__inst_executed_op_shared_atom.sum", "smem atomic instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "smem bank conflicts (atom)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem bank conflicts (ld)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem bank conflicts (st)"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
]


def raw(path: str):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {h: (v, u) for h, v, u in zip(hdr, r, units)}
        res.append(d)
    return res


def main():
    out = sys.argv[1]
    lines = ["| kernel (capture) | " + " | ".join(n for _, n in METRICS) + " |",
             "|---|" + "---|" * len(METRICS)]
    for arg in sys.argv[2:]:
        label, path = arg.split("=", 1)
        for d in raw(path):
            name = d.get("Kernel Name", ("?", ""))[0].split("(")[0][:60]
            cells = []
            for m, _ in METRICS:
                v, u = d.get(m, ("n/a", ""))
                cells.append(f"{v} {u}".strip())
            lines.append(f"| {label}: `{name}` | " + " | ".join(cells) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
