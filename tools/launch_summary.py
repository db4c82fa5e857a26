"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): mean
duration per kernel name (beam kernels only unless --all)."""
import collections
import csv
import sys


def main(path, all_kernels=False):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki]
        if not all_kernels and "beam::" not in name:
            continue
        short = name.split("(")[0].replace("void ", "")[:70]
        d.setdefault(short, []).append(float(r[vi].replace(",", "")) / 1e3)
    for k, v in d.items():
        print(f"  {k:70s} n={len(v):3d} mean={sum(v)/len(v):8.2f} us  min={min(v):8.2f}")


if __name__ == "__main__":
    main(sys.argv[1], "--all" in sys.argv)
