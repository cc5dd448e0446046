"""Summarise ncu reports (.ncu-rep) into the tracked profiles/ directory.

    python scripts/ncu_summary.py gpurun_out/prof_c2.ncu-rep [...] > profiles/r1_<name>.md
    python scripts/ncu_summary.py gpurun_out/prof_r2c_c2 [...]   # exported pages (gpu_round_profile.sh)

Reads the `details` and `raw` pages with `ncu -i` (no GPU needed) -- or the
pages gpu_round_profile.sh exported (<prefix>_details.txt, <prefix>_raw.csv)
when the report itself did not travel back -- and prints a
markdown table of the numbers DESIGN.md cites: duration, DRAM bytes and
throughput, FP64-pipe activity, occupancy, issue statistics, top stall reasons.
"""

from __future__ import annotations

import csv
import os
import re
import subprocess
import sys

DETAILS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
           "Grid Size", "Block Size", "Theoretical Occupancy", "Achieved Occupancy", "Executed Ipc Active",
           "Issue Slots Busy", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
           "Static Shared Memory Per Block", "Dynamic Shared Memory Per Block"]
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu_csv(path: str, page: str):
    out = subprocess.run(["ncu", "-i", path, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def exported(prefix: str):
    """(kernel, details values, raw rows) from the exported text/CSV pages."""
    vals, kernel = {}, None
    for line in open(prefix + "_details.txt"):
        m = re.match(r"^\s{4}(\S.*?)\s{2,}(\S+(?: \S+)?)?\s+([-\d.,]+)\s*$", line)
        if m and m.group(1).strip() in DETAILS:
            vals[m.group(1).strip()] = f"{m.group(3)} {m.group(2) or ''}".strip()
        elif kernel is None and line.strip() and not line.startswith(" ") and "(" in line:
            kernel = line.strip()
    with open(prefix + "_raw.csv") as f:
        raw = list(csv.reader(f))
    return kernel, vals, raw


def summarize(path: str) -> list[str]:
    lines = [f"### `{path.split('/')[-1]}`", ""]
    if not path.endswith(".ncu-rep") and os.path.exists(path + "_raw.csv"):
        kernel, vals, raw = exported(path)
        if len(raw) >= 3 and "Kernel Name" in raw[0]:
            kernel = raw[2][raw[0].index("Kernel Name")]
        return finish(lines, kernel, vals, raw)
    rows = ncu_csv(path, "details")
    hdr = rows[0]
    kernel = None
    vals = {}
    for row in rows[1:]:
        d = dict(zip(hdr, row))
        kernel = kernel or d.get("Kernel Name")
        if d.get("Metric Name") in DETAILS:
            vals[d["Metric Name"]] = f"{d['Metric Value']} {d.get('Metric Unit', '')}".strip()
    return finish(lines, kernel, vals, ncu_csv(path, "raw"))


def finish(lines, kernel, vals, raw) -> list[str]:
    lines.append(f"kernel: `{(kernel or '')[:160]}`")
    lines.append("")
    lines.append("| metric | value |")
    lines.append("|---|---|")
    for k in DETAILS:
        if k in vals:
            lines.append(f"| {k} | {vals[k]} |")
    if len(raw) >= 3:
        h, units, v = raw[0], raw[1], raw[2]
        for k in RAW:
            if k in h:
                i = h.index(k)
                lines.append(f"| {k} | {v[i]} {units[i]} |")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(v[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        lines.append(f"| top stall samples | {', '.join(f'{n} {int(c)}' for c, n in stalls[:6])} |")
    lines.append("")
    return lines


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("\n".join(summarize(p)))
