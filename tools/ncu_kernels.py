"""Median per-kernel duration / DRAM bytes of the repo's kernels from an ncu CSV
(`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv`).
usage: python tools/ncu_kernels.py <csv> [label]"""
import csv
import sys


def main(path, label=""):
    agg = {}
    for r in csv.reader(open(path)):
        if len(r) < 15 or not r[0].isdigit():
            continue
        k = r[4].replace("void ", "").split("(")[0]
        agg.setdefault(k, {}).setdefault(r[12], []).append(float(r[14].replace(",", "")))
    for k, ms in agg.items():
        med = {m: sorted(v)[len(v) // 2] for m, v in ms.items()}
        t = med.get("gpu__time_duration.sum", 0.0)
        rd = med.get("dram__bytes_read.sum", 0.0)
        print(f"{label} {k[:70]:70s} n={len(ms.get('gpu__time_duration.sum', []))} us={t / 1e3:.1f} "
              f"MB_read={rd / 1e6:.1f} GB/s={rd / max(t, 1):.0f}")


if __name__ == "__main__":
    main(*sys.argv[1:3])
