"""Summarise ncu captures into profiles/ncu_summary.json (read by bench.py for
roofline.traffic) and per-capture text summaries.

usage: python tools/ncu_summary.py <report.ncu-rep> <kernel-name> <workload> [<report> <kernel> <workload> ...]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "gpc__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def _record(row, unit, kernel, workload, rep):
    rec = {"kernel": kernel, "workload": workload, "name": row.get("Kernel Name", "")[:120],
           "report": os.path.basename(rep)}
    for k in KEYS:
        if k in row and row[k] not in ("", None):
            v = float(row[k].replace(",", ""))
            u = unit.get(k, "")
            if u in SCALE:
                v *= SCALE[u]
            rec[k] = v
            rec[k + ".unit"] = "byte" if u in SCALE else u
    rec["dram_bytes_per_launch"] = rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
    return rec


def _save(keep):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    data = {"kernels": keep,
            "note": ("one `ncu --set full --clock-control none` capture per kernel/workload (cold-cache, serialised "
                     "replays); dram_bytes_per_launch = dram__bytes_read.sum + dram__bytes_write.sum")}
    with open(path, "w") as fh:
        json.dump(data, fh, indent=1)


def _load():
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    return json.load(open(path))["kernels"] if os.path.exists(path) else []


def main_named(rep, workload, name_of):
    """Every kernel of `rep` under its base name (name_of(full name)); the first
    launch of each name wins (the report holds one layer call)."""
    keep = _load()
    done = set()
    for row, unit in raw_rows(rep):
        kernel = name_of(row.get("Kernel Name", ""))
        if kernel in done:
            continue
        done.add(kernel)
        rec = _record(row, unit, kernel, workload, rep)
        keep = [k for k in keep if not (k["kernel"] == kernel and k["workload"] == workload)]
        keep.append(rec)
        print(json.dumps({k: rec[k] for k in ("kernel", "workload", "gpu__time_duration.sum", "dram_bytes_per_launch")
                          if k in rec}))
    _save(keep)


def main(args):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    data = json.load(open(path)) if os.path.exists(path) else {"kernels": []}
    keep = [k for k in data["kernels"]]
    for i in range(0, len(args), 3):
        rep, kernel, workload = args[i:i + 3]
        for n, (row, unit) in enumerate(raw_rows(rep)):
            rec = {"kernel": kernel if n == 0 else f"{kernel}#{n}", "workload": workload,
                   "name": row.get("Kernel Name", "")[:120], "report": os.path.basename(rep)}
            for k in KEYS:
                if k in row and row[k] not in ("", None):
                    v = float(row[k].replace(",", ""))
                    u = unit.get(k, "")
                    if u in SCALE:
                        v *= SCALE[u]
                    rec[k] = v
                    rec[k + ".unit"] = "byte" if u in SCALE else u
            rec["dram_bytes_per_launch"] = rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
            keep = [k for k in keep if not (k["kernel"] == rec["kernel"] and k["workload"] == workload)]
            keep.append(rec)
            print(json.dumps(rec))
    data["kernels"] = keep
    data["note"] = ("one `ncu --set full --clock-control none` capture per kernel/workload (cold-cache, serialised "
                    "replays); dram_bytes_per_launch = dram__bytes_read.sum + dram__bytes_write.sum")
    with open(path, "w") as fh:
        json.dump(data, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
