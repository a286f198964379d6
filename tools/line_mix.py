"""Per-source-line instruction attribution from an ncu cuda,sass source export
(ncu -i rep --page source --csv --print-source cuda,sass --launch-skip S --launch-count 1).

    python tools/line_mix.py file.csv cells [top]
Prints, per (file, line): thread-instructions per cell, split FP64 / other, stall share.
"""
import csv
import sys
from collections import defaultdict

FP64 = ("DFMA", "DMUL", "DADD")


def main(path, cells, top=40):
    rows = list(csv.reader(open(path)))
    cur_file, cur_line, cur_src = "?", "?", ""
    agg = defaultdict(lambda: [0, 0, 0, ""])
    ops = defaultdict(lambda: defaultdict(int))
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0] != "":
            cur_line, cur_src = r[0], r[1]
            continue
        sass = r[3].strip().split()
        if not sass or not r[8].isdigit():
            continue
        op = sass[1] if sass[0].startswith("@") else sass[0]
        base = op.split(".")[0]
        n = int(r[8])
        st = int(r[4] or 0)
        key = (cur_file, cur_line)
        a = agg[key]
        a[3] = cur_src.strip()[:70]
        if base in FP64:
            a[0] += n
        else:
            a[1] += n
        a[2] += st
        ops[key][op] += n
    tot = sum(a[0] + a[1] for a in agg.values())
    sts = sum(a[2] for a in agg.values())
    print(f"total {tot / cells:.1f} thread-inst/cell")
    for key, a in sorted(agg.items(), key=lambda kv: -(kv[1][0] + kv[1][1]))[:top]:
        o = sorted(ops[key].items(), key=lambda kv: -kv[1])[:4]
        os_ = " ".join(f"{k}:{v / cells:.1f}" for k, v in o if not k.startswith(FP64))
        print(f"{key[0]:14s}:{key[1]:>4s} fp64 {a[0] / cells:6.1f} other {a[1] / cells:6.1f} stall {100 * a[2] / sts:5.1f}%  {a[3]}  | {os_}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 40)
