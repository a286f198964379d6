"""Top source lines by warp-stall samples (with their top reasons) from an ncu
cuda,sass source export.   python tools/line_stalls.py file.csv [top]"""
import csv
import sys
from collections import defaultdict


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = None
    cur = None
    f = "?"
    agg = defaultdict(lambda: defaultdict(int))
    src = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            cols = [h for h in r if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if hdr is None or not r[0].isdigit() and r[0] != "":
            continue
        if r[0] != "":
            cur = (f, int(r[0]))
            src[cur] = r[1].strip()[:70]
            continue
        if len(r) < len(hdr) or not r[8].isdigit():
            continue
        for h in cols:
            v = r[hdr[h]]
            if v.isdigit():
                agg[cur][h[6:]] += int(v)
    tot = sum(sum(d.values()) for d in agg.values())
    for k, d in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
        s = sum(d.values())
        t3 = sorted(d.items(), key=lambda kv: -kv[1])[:3]
        print(f"{k[0]:14s}:{k[1]:4d} {100 * s / tot:5.1f}%  {', '.join(f'{a}={100 * b / s:.0f}' for a, b in t3)}  | {src[k]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
