"""Bitwise fingerprint of the library's results on a set of cases, to compare two builds:

    ECHO_LIB_VARIANT=      python tools/variant_bitwise.py > a.txt
    ECHO_LIB_VARIANT=xold  python tools/variant_bitwise.py > b.txt ; diff a.txt b.txt

Each case: set_prims, rhs, 2 steps at a fixed dt, the final U^n and P; one sha256 line each.
"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import echo_inputs as I  # noqa: E402
from paper_1810_04597_b200 import echo as E  # noqa: E402

CASES = [
    # (config, grid, overrides)
    (0, (32, 32, 32), {}),
    (0, (150, 13, 70), {}),
    (0, (3, 7, 5), {}),            # n < g along x (periodic wrap mod n)
    (2, (45, 38, 41), {}),         # outflow blast
    (2, (63, 9, 7), {}),           # odd outflow
    (2, (1, 20, 12), {}),          # degenerate x
    (3, (130, 20, 18), {}),        # ragged tail, several chunks
    (4, (72, 35, 24), {}),         # Kerr-Schild
    (0, (66, 20, 20), {"divb": 1}),
    (2, (70, 24, 20), {"divb": 2}),
    (4, (40, 20, 16), {"divb": 2}),
    (2, (70, 24, 20), {"rec": 2}),
    (2, (70, 24, 20), {"rec": 3}),
    (2, (70, 24, 20), {"rec": 4}),
    (2, (70, 24, 20), {"rec": 5}),
    (2, (70, 24, 20), {"der": 4}),
]


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main():
    for cfg, n, kw in CASES:
        p = I.problem(cfg, n=n)
        for k, v in kw.items():
            setattr(p, k, v)
        P8 = I.initial_prims(p)
        try:
            run_case(p, P8, cfg, n, kw)
        except Exception as ex:  # noqa: BLE001
            print(cfg, n, kw, "ERROR", ex, flush=True)


def run_case(p, P8, cfg, n, kw):
    if True:
        g = E.Echo(p)
        g.set_prims(P8)
        if p.divb == 2:
            g.set_face_field(I.face_field(p))
        L = g.rhs()
        dt = 0.25 * g.max_dt(p.cfl)
        g.step(dt)
        g.step(dt)
        un, us, p5 = g.get_state()
        print(cfg, n, kw, "rhs", h(L), "Un", h(un), "P", h(p5), flush=True)
        g.close()


if __name__ == "__main__":
    main()
