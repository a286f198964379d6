"""Per-phase instruction and stall-sample totals of a k_march kernel from an ncu source-page
export with SASS (ncu -i rep --page source --csv --print-source cuda,sass): every SASS row is
attributed to the CUDA (file, line) block above it, and the line to a pipeline phase by the
function it falls in (echo_dev.cuh) or the phase markers of march_impl.cuh.

    python tools/src_phases.py gpurun_out/src_sweep_1.csv CELLS
"""
import csv
import re
import sys
from collections import defaultdict

ROOT = "paper_1810_04597_b200/csrc/"
FP64 = ("DFMA", "DMUL", "DADD", "DSETP")


def spans():
    out = []
    dev = open(ROOT + "echo_dev.cuh").read().splitlines()

    def span(lines, pat, fname, ph):
        i0 = next(i for i, l in enumerate(lines) if re.search(pat, l))
        depth, started = 0, False
        for j in range(i0, len(lines)):
            depth += lines[j].count("{") - lines[j].count("}")
            started = started or "{" in lines[j]
            if started and depth == 0:
                out.append((fname, i0 + 1, j + 1, ph))
                return
    for pat, ph in ((r"void weno5_both", "A:weno"), (r"void make_state", "B:hll"), (r"void speeds", "B:hll"),
                    (r"void hll_face", "B:hll"), (r"void cons_flux", "B:hll"), (r"double der5", "D1:der"),
                    (r"double frcp", "rcp/rsqrt"), (r"double frsqrt", "rcp/rsqrt"), (r"int map_index", "index")):
        span(dev, pat, "echo_dev.cuh", ph)
    m = open(ROOT + "march_impl.cuh").read().splitlines()
    marks = [(r"---- A: WENO5", "A:march"), (r"---- D1: DER", "D1:march"), (r"prefetch: the next chunk", "prefetch"),
             (r"---- D2: cell", "D2:march"), (r"---- B: face", "B:march")]
    idx = [(next(i for i, l in enumerate(m) if re.search(p, l)), ph) for p, ph in marks]
    kend = next(i for i, l in enumerate(m) if "__launch_bounds__" in l and i > idx[-1][0])
    for (a, ph), nxt in zip(idx, idx[1:] + [(kend, None)]):
        out.append(("march_impl.cuh", a + 1, nxt[0], ph))
    return out


def main(path, cells):
    sp = spans()

    def phase(f, ln):
        for fn, a, b, ph in sp:
            if f == fn and a <= ln <= b:
                return ph
        return f"other:{f}"
    rows = list(csv.reader(open(path)))
    hdr = {}
    cur_f, cur_l = "?", 0
    inst = defaultdict(lambda: [0, 0])
    st = defaultdict(lambda: defaultdict(int))
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if not hdr or len(r) < len(hdr):
            continue
        if r[0]:
            cur_l = int(r[0]) if r[0].isdigit() else 0
            continue
        sass = r[3].strip().split()
        if not sass:
            continue
        op = (sass[1] if sass[0].startswith("@") else sass[0]).split(".")[0]
        ph = phase(cur_f, cur_l)
        v = r[hdr["Thread Instructions Executed"]]
        n = int(v) if v.isdigit() else 0
        inst[ph][0 if op in FP64 else 1] += n
        for h, i in hdr.items():
            if h.startswith("stall_") and "Not Issued" not in h and r[i].isdigit():
                st[ph][h[6:]] += int(r[i])
    tot = sum(sum(d.values()) for d in st.values())
    print(f"{'phase':28s} {'fp64/cell':>9s} {'other/cell':>10s} {'samples%':>8s}  top stall reasons (% of the phase's samples)")
    for ph in sorted(inst, key=lambda p: -sum(st[p].values())):
        s = sum(st[ph].values())
        top = sorted(st[ph].items(), key=lambda kv: -kv[1])[:5]
        print(f"{ph:28s} {inst[ph][0] / cells:9.1f} {inst[ph][1] / cells:10.1f} {100 * s / max(tot, 1):8.1f}  " +
              ", ".join(f"{k}={100 * v / max(s, 1):.0f}" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
