"""Diagnostic (development): where a UCT slab run departs from the single-domain run."""
import sys
import numpy as np
sys.path.insert(0, '.')
import echo_inputs as I
from paper_1810_04597_b200 import echo as E
from paper_1810_04597_b200.slab import LocalSlabs

for n, ns in (((20, 16, 27), 3), ((24, 20, 32), 2)):
    p = I.problem(0, n=n); p.divb = 2
    P8, b3 = I.initial_prims(p), I.face_field(p)
    one = E.Echo(p); one.set_prims(P8); one.set_face_field(b3)
    sl = LocalSlabs(p, ns); sl.set_prims(P8); sl.set_face_field(b3)
    u1, _, p1 = one.get_state()
    for name, a, b in (("U0", sl.gather(lambda g: g.get_state()[0]), u1), ("P0", sl.gather(lambda g: g.get_state()[2]), p1),
                       ("prims", sl.gather(lambda g: g.get_prims()), one.get_prims())):
        d = np.abs(a - b)
        print(n, ns, name, "max", d.max(), "planes", sorted(set(np.argwhere(d > 0)[:, 1].tolist()))[:20])
    dt = one.max_dt(0.4)
    print("dt one", dt, "slabs", [g.max_dt(0.4) for g, _, _ in sl.parts])
    for s in (1, 2, 3):
        one.stage(s, dt)
        sl.exchange()
        for g, _, _ in sl.parts:
            E.stage_sweeps(g.ctx, s); E.stage_update_field(g.ctx, s, dt)
        sl.exchange_field()
        for g, _, _ in sl.parts:
            E.stage_update_cells(g.ctx, s, dt)
        bo, bs = one.get_face_field(), sl.gather(lambda g: g.get_face_field())
        uo, us = one.get_state(), sl.gather(lambda g: g.get_state()[1 if s < 3 else 0])
        u_one = uo[1 if s < 3 else 0]
        for name, a, b in (("b", bs, bo), ("U", us, u_one)):
            d = np.abs(a - b)
            if d.max() > 0:
                idx = np.argwhere(d > 0)
                print(n, ns, "stage", s, name, "max", d.max(), "count", len(idx), "k planes", sorted(set(idx[:, 1].tolist()))[:20], "vars", sorted(set(idx[:, 0].tolist())))
            else:
                print(n, ns, "stage", s, name, "bitwise")
