"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass)
by CUDA source line: warp-stall samples by reason and executed instructions."""
import collections
import csv
import sys


def main(path, top=40, filt=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    cur_file = cur_line = None
    agg = collections.defaultdict(lambda: collections.Counter())
    src = {}
    reasons = None
    for r in rows:
        if r and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if not hdr or len(r) < 8:
            continue
        if r[0] != "":
            cur_line = (cur_file, int(r[0]))
            src[cur_line] = r[1]
            continue
        try:
            c = agg[cur_line]
            c["samples"] += float(r[4] or 0)
            c["inst"] += float(r[7] or 0)
            for i, h in reasons:
                c[h] += float(r[i] or 0)
        except ValueError:
            continue
    tot = sum(v["samples"] for v in agg.values()) or 1
    toti = sum(v["inst"] for v in agg.values()) or 1
    items = sorted(agg.items(), key=lambda kv: -kv[1]["samples"])
    for k, v in items[:top]:
        if filt and filt not in k[0]:
            continue
        rs = sorted(((h[6:], v[h]) for _, h in reasons if v[h] > 0), key=lambda x: -x[1])[:3]
        rs = " ".join(f"{n}:{x / tot * 100:.1f}" for n, x in rs)
        print(f"{k[0]}:{k[1]} {v['samples'] / tot * 100:5.1f}% {v['inst'] / toti * 100:5.1f}%i [{rs}] | {src[k].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
