"""one UCT step at 256^3 (config 3's turbulence recipe) for kernel timing under ncu"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import echo_inputs as I
from paper_1810_04597_b200 import echo as E
p = I.problem(3, n=(256, 256, 256)); p.divb = 2
g = E.Echo(p)
g.set_prims(I.initial_prims(p))
g.set_face_field(I.face_field(p))
g.step(g.max_dt(p.cfl))
print("ok", os.environ.get("ECHO_LIB_VARIANT", ""))
