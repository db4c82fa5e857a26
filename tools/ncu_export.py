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
            sections, cur, hdr = [], None, None
            for r in csv.reader(io.StringIO(src)):
                if not r:
                    continue
                if r[0] == "Kernel Name":
                    cur = []
                    sections.append(cur)
                    hdr = None
                elif r[0] == "Address":
                    hdr = r
                elif hdr is not None and cur is not None:
                    cur.append(dict(zip(hdr, r)))
            if not sections or not sections[0]:
                continue
            data = sections[0]  # first launch of this kernel in the report
            key = "Warp Stall Sampling (All Samples)"

            def num(r):
                try:
                    return float(r.get(key) or 0)
                except ValueError:
                    return 0.0
            tot = sum(num(r) for r in data)
            fh.write(f"== {nm}: {tot:.0f} warp-stall samples; top SASS lines\n")
            for r in sorted(data, key=lambda r: -num(r))[:25]:
                fh.write(f"{num(r):7.0f}  {r.get('Source', '')[:120]}\n")
            fh.write("\n")
    del args


if __name__ == "__main__":
    main(*sys.argv[1:4])
