"""torchrun helper for tests/test_gpu_multi.py: the z-slab decomposition over N GPUs (one rank
per GPU, NCCL ghost exchange overlapped by the interior sweeps, DistSlab.step) against the
single-domain run on rank 0's GPU, bit for bit, after `steps` steps.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        tools/multi_gpu_slab_check.py --config 0 --n 48 40 36 --steps 2 --out result.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=0)
    ap.add_argument("--n", type=int, nargs=3, default=[48, 40, 36])
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--fused", action="store_true")
    ap.add_argument("--divb", type=int, default=0)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    import echo_inputs as I
    from paper_1810_04597_b200 import echo, slab

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    p = I.problem(a.config, n=tuple(a.n))
    p.divb = a.divb
    P8 = I.initial_prims(p)
    B3 = I.face_field(p) if a.divb == 2 else None
    sp, (z0, nz) = slab.slab_problem(p, rank, world)
    g = echo.Echo(sp)
    echo.set_stream(g.ctx, torch.cuda.current_stream(dev).cuda_stream)
    g.set_prims(np.ascontiguousarray(P8[:, z0:z0 + nz]))
    D = slab.DistSlab(slab.CtxIO(g), rank, world, p.bc[2][0] == 0, dev, uct=a.divb == 2)
    if B3 is not None:
        D.set_face_field(np.ascontiguousarray(B3[:, z0:z0 + nz]))
    if a.fused:
        D.link_fused()
    dts = []
    for _ in range(a.steps):
        dt = D.min_dt(g.max_dt(p.cfl))
        dts.append(dt)
        (D.step_fused if a.fused else D.step)(dt)
    un, _, pp = g.get_state()
    bb = g.get_face_field() if B3 is not None else np.zeros(1)
    parts = [None] * world
    dist.all_gather_object(parts, (z0, nz, un, pp, bb))
    if rank == 0:
        ref = echo.Echo(p)
        ref.set_prims(P8)
        if B3 is not None:
            ref.set_face_field(B3)
        rdts = []
        for _ in range(a.steps):
            dt = ref.max_dt(p.cfl)
            rdts.append(dt)
            ref.step(dt)
        run, _, rpp = ref.get_state()
        un_all = np.concatenate([x[2] for x in sorted(parts, key=lambda x: x[0])], axis=1)
        pp_all = np.concatenate([x[3] for x in sorted(parts, key=lambda x: x[0])], axis=1)
        res = {"world": world, "dt_equal": dts == rdts, "U_bitwise": bool(np.array_equal(un_all, run)),
               "P_bitwise": bool(np.array_equal(pp_all, rpp)),
               "max_abs_dU": float(np.max(np.abs(un_all - run)))}
        if B3 is not None:
            b_all = np.concatenate([x[4] for x in sorted(parts, key=lambda x: x[0])], axis=1)
            res["b_bitwise"] = bool(np.array_equal(b_all, ref.get_face_field()))
        with open(a.out, "w") as f:
            json.dump(res, f)
        ref.close()
    g.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
