"""Per-opcode thread-instruction mix of one kernel from an ncu source-page CSV
(ncu -i rep --page source --csv --print-source sass --launch-skip S --launch-count 1).

    python tools/sass_mix.py /tmp/sass_y.csv [cells]
"""
import csv
import sys
from collections import Counter


def main(path, cells=None):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    ix = {h: i for i, h in enumerate(hdr)}
    start = rows.index(hdr) + 1
    mix, warp = Counter(), Counter()
    stall = Counter()
    for r in rows[start:]:
        if len(r) < len(hdr) or not r[ix["Instructions Executed"]].isdigit():
            continue
        op = r[ix["Source"]].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1]
        o = o.split(".")[0]
        mix[o] += int(r[ix["Thread Instructions Executed"]] or 0)
        warp[o] += int(r[ix["Instructions Executed"]] or 0)
        stall[o] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot = sum(mix.values())
    wt = sum(warp.values())
    st = sum(stall.values())
    print(f"total thread-inst {tot:.4g}  warp-inst {wt:.4g}" + (f"  per cell {tot / cells:.1f}" if cells else ""))
    for o, v in mix.most_common(40):
        pc = f"{v / cells:9.1f}/cell" if cells else ""
        print(f"{o:10s} {v:14d} {100 * v / tot:6.2f}% warp {100 * warp[o] / wt:6.2f}% stall {100 * stall[o] / st:6.2f}% {pc}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
