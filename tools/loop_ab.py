"""A/B of the host time loop (echo_max_dt + echo_step per step) against echo_advance
(dt on the device, one CUDA-graph replay per step), alternated in one process.

    python tools/loop_ab.py --config 1 --steps 20 --reps 5
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import echo_inputs as I  # noqa: E402
from paper_1810_04597_b200 import echo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    p = I.problem(a.config)
    st = torch.cuda.current_stream()
    g = echo.Echo(p)
    echo.set_stream(g.ctx, st.cuda_stream)
    g.set_prims(I.initial_prims(p, device=torch.device("cuda")))
    g.advance(3, p.cfl)
    for _ in range(3):
        g.step(g.max_dt(p.cfl))
    res = {"host": [], "device": []}
    for _ in range(a.reps):
        for mode in ("host", "device"):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            if mode == "device":
                g.advance(a.steps, p.cfl, log=False)
            else:
                for _ in range(a.steps):
                    g.step(g.max_dt(p.cfl))
            e1.record(st)
            torch.cuda.synchronize()
            res[mode].append(e0.elapsed_time(e1) / a.steps)
    print(json.dumps({"config": a.config, "grid": list(p.n), "steps": a.steps,
                      "ms_per_step_median": {k: statistics.median(v) for k, v in res.items()},
                      "all": res}))


if __name__ == "__main__":
    main()
