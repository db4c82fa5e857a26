"""Export what the judge reads from an `ncu --set full` report into small text
files (the .ncu-rep itself is too large to bring back from the GPU box):

  <out>/<stem>_details.txt   `ncu --page details` (every section of every kernel)
  <out>/<stem>_stalls.txt    per kernel: the SASS lines with the most warp-stall
                             samples (source page)
and appends the per-kernel metrics to profiles/ncu_summary.json through
tools/ncu_summary.py (kernel key = the kernel's base name, workload = argv).

usage: python tools/ncu_export.py <report.ncu-rep> <workload> <out_dir>
"""

from __future__ import annotations

import csv
import io
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402


def base_name(full: str) -> str:
    n = full.replace("void ", "").split("(")[0].split("<")[0]
    return n.split("::")[-1]


def main(rep, workload, out):
    os.makedirs(out, exist_ok=True)
    stem = os.path.basename(rep).replace(".ncu-rep", "")
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    with open(os.path.join(out, f"{stem}_details.txt"), "w") as fh:
        fh.write(det)
    # per-kernel metrics -> ncu_summary.json (one entry per kernel base name)
    rows = ncu_summary.raw_rows(rep)
    seen = {}
    args = []
    for row, _unit in rows:
        nm = base_name(row.get("Kernel Name", ""))
        seen[nm] = seen.get(nm, 0) + 1
    ncu_summary.main_named(rep, workload, base_name)
    # stalls per kernel (source page is per kernel: --print-kernel-base / -k filters)
    with open(os.path.join(out, f"{stem}_stalls.txt"), "w") as fh:
        for nm in seen:
            src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{re.escape(nm)}"],
                                 capture_output=True, text=True).stdout
            lines = list(csv.reader(io.StringIO(src)))
            if len(lines) < 3:
                continue
            hdr = lines[1] if lines[0] and lines[0][0] == "Kernel Name" else lines[0]
            data = lines[2:] if hdr is lines[1] else lines[1:]
            try:
                si = hdr.index("Warp Stall Sampling (All Samples)")
                sc = hdr.index("Source")
            except ValueError:
                continue
            tot = sum(float(r[si] or 0) for r in data if len(r) > si)
            fh.write(f"== {nm}: {tot:.0f} warp-stall samples; top SASS lines\n")
            top = sorted((r for r in data if len(r) > si), key=lambda r: -float(r[si] or 0))[:25]
            for r in top:
                fh.write(f"{float(r[si] or 0):7.0f}  {r[sc][:120]}\n")
            fh.write("\n")
    del args


if __name__ == "__main__":
    main(*sys.argv[1:4])
