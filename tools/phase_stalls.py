"""Stall reasons and instruction counts per pipeline phase of a k_march kernel
from an ncu cuda,sass source export (tools/line_mix.py format).

    python tools/phase_stalls.py file.csv cells
Phases are assigned by source file + function-line ranges found by pattern.
"""
import csv
import re
import sys
from collections import defaultdict

FP64 = ("DFMA", "DMUL", "DADD")


def ranges():
    """(file, first, last, phase) from the sources' markers."""
    out = []
    root = "paper_1810_04597_b200/csrc/"
    dev = open(root + "echo_dev.cuh").read().splitlines()
    def span(lines, start_pat, fname, phase):
        i0 = next(i for i, l in enumerate(lines) if re.search(start_pat, l))
        depth, started = 0, False
        for j in range(i0, len(lines)):
            depth += lines[j].count("{") - lines[j].count("}")
            if "{" in lines[j]:
                started = True
            if started and depth == 0:
                out.append((fname, i0 + 1, j + 1, phase))
                return
    span(dev, r"void weno5_both", "echo_dev.cuh", "A:weno")
    span(dev, r"void make_state", "echo_dev.cuh", "B:hll")
    span(dev, r"void speeds", "echo_dev.cuh", "B:hll")
    span(dev, r"void hll_face", "echo_dev.cuh", "B:hll")
    span(dev, r"void cons_flux", "echo_dev.cuh", "B:hll")
    span(dev, r"double der5", "echo_dev.cuh", "D1:der")
    span(dev, r"double frcp", "echo_dev.cuh", "rcp/rsqrt")
    span(dev, r"double frsqrt", "echo_dev.cuh", "rcp/rsqrt")
    m = open(root + "march.cu").read().splitlines()
    marks = [(r"---- A: WENO5", "A:march"), (r"---- D1: DER", "D1:march"), (r"prefetch: the next chunk", "prefetch"),
             (r"---- D2: cell", "D2:march"), (r"---- B: face", "B:march")]
    idx = [(next(i for i, l in enumerate(m) if re.search(p, l)), ph) for p, ph in marks]
    kend = next(i for i, l in enumerate(m) if l.startswith("template <int AX, bool KS, int DER, int REC, bool DN>\nstatic") or "static cudaError_t launch_one" in l)
    for (a, ph), nxt in zip(idx, idx[1:] + [(kend, None)]):
        out.append(("march.cu", a + 1, nxt[0], ph))
    return out


def main(path, cells):
    rng = ranges()
    def phase(f, ln):
        try:
            ln = int(ln)
        except ValueError:
            return "?"
        for fn, a, b, ph in rng:
            if f == fn and a <= ln <= b:
                return ph
        return f"other:{f}"
    rows = list(csv.reader(open(path)))
    hdr = None
    cur_f, cur_l = "?", "?"
    inst = defaultdict(lambda: [0, 0])
    stalls = defaultdict(lambda: defaultdict(int))
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            cols = [h for h in r if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if hdr is None:
            continue
        if r[0] != "":
            cur_l = r[0]
            continue
        if len(r) < len(hdr) or not r[8].isdigit():
            continue
        sass = r[3].strip().split()
        op = (sass[1] if sass[0].startswith("@") else sass[0]).split(".")[0]
        ph = phase(cur_f, cur_l)
        n = int(r[8])
        inst[ph][0 if op in FP64 else 1] += n
        for h in cols:
            v = r[hdr[h]]
            if v.isdigit():
                stalls[ph][h[6:]] += int(v)
    tot_st = sum(sum(d.values()) for d in stalls.values())
    tot_i = sum(a + b for a, b in inst.values())
    print(f"{'phase':24s} {'fp64/cell':>9s} {'other/cell':>10s} {'samples%':>8s}  top stall reasons (% of phase samples)")
    for ph in sorted(inst, key=lambda p: -sum(stalls[p].values())):
        st = stalls[ph]
        s = sum(st.values())
        top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
        print(f"{ph:24s} {inst[ph][0] / cells:9.1f} {inst[ph][1] / cells:10.1f} {100 * s / tot_st:8.1f}  " +
              ", ".join(f"{k}={100 * v / max(s, 1):.0f}" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
