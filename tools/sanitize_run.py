"""A small run of every path for compute-sanitizer (SURVEY §4 "Sanitizers", §5 race
detection): config 0 at 32^3 (host steps + the CUDA-graph device loop), a Kerr-Schild
32 x 16 x 32 patch, rec = 6, UCT, 2 slabs with the copy exchange (split halves) and with the
fused ghost stores, and the debug NaN scan.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import echo_inputs as I
    from paper_1810_04597_b200 import echo
    from paper_1810_04597_b200.slab import LocalSlabs

    def run(p, steps=1, adv=0, faces=False, debug=False):
        g = echo.Echo(p)
        g.set_prims(I.initial_prims(p))
        if faces:
            g.set_face_field(I.face_field(p))
        if debug:
            g.set_debug()
        for _ in range(steps):
            g.step(g.max_dt(p.cfl))
        if adv:
            g.advance(adv, p.cfl)
        g.rhs()
        g.get_prims()
        g.close()

    run(I.problem(0, n=(32, 32, 32)), steps=2, adv=2)
    run(I.problem(4, n=(32, 16, 32)), steps=1)
    p = I.problem(0, n=(24, 20, 16))
    p.rec = 6
    run(p, steps=1, adv=1)
    q = I.problem(2, n=(20, 16, 12))
    q.divb = 2
    run(q, steps=1, adv=1, faces=True)
    run(I.problem(0, n=(16, 12, 10)), steps=1, adv=1, debug=True)
    for fused, split in ((False, True), (True, False)):
        s = LocalSlabs(I.problem(0, n=(24, 20, 32)), 2, fused=fused)
        s.set_prims(I.initial_prims(I.problem(0, n=(24, 20, 32))))
        for _ in range(2):
            s.step(s.max_dt(0.4), split=split)
        s.close()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
