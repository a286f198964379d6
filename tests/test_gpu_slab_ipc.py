"""Cross-process fused slab exchange: one process per
slab, the neighbours' arrays mapped by CUDA IPC, every K3 update storing its edge
planes straight into them (echo_ipc_export / echo_halo_link_ipc / echo_halo_pull,
slab.DistSlab.link_fused / step_fused).  On this one-GPU box the 2-3 processes share
cuda:0 (IPC works within a device; their kernels never wait on each other — the
stage ordering is host barriers over gloo).  The gathered state must equal the
single-domain run bit for bit.  Marked gpu."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, n, steps, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    import echo_inputs as I
    from paper_1810_04597_b200 import echo as E
    from paper_1810_04597_b200 import slab

    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = I.problem(cfg, n=n)
    P8 = I.initial_prims(p)
    sp, (z0, nz) = slab.slab_problem(p, rank, world)
    g = E.Echo(sp)
    g.set_prims(np.ascontiguousarray(P8[:, z0:z0 + nz]))
    D = slab.DistSlab(slab.CtxIO(g), rank, world, p.bc[2][0] == 0, "cpu")
    D.link_fused()
    dts = []
    for _ in range(steps):
        dt = D.min_dt(g.max_dt(p.cfl))
        dts.append(dt)
        D.step_fused(dt)
    un, _, pp = g.get_state()
    parts = [None] * world
    dist.all_gather_object(parts, (z0, un, pp, dts))
    D.barrier()  # nobody unmaps while a neighbour may still store into it
    for side in (0, 1):
        E.halo_link_ipc(g.ctx, side, None, 0)
    g.close()
    if rank == 0:
        out["parts"] = parts
    dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("cfg,n,world,steps", [(0, (32, 24, 32), 2, 2), (2, (24, 20, 36), 3, 2)])
def test_ipc_fused_slabs_bitwise(cfg, n, world, steps):
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, ROOT)
    from paper_1810_04597_b200 import build

    build.build()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _port(), cfg, n, steps, out), nprocs=world, join=True)
    parts = sorted(out["parts"], key=lambda t: t[0])
    import echo_inputs as I
    from paper_1810_04597_b200 import echo as E

    p = I.problem(cfg, n=n)
    one = E.Echo(p)
    one.set_prims(I.initial_prims(p))
    for dt in parts[0][3]:
        assert one.max_dt(p.cfl) == dt
        one.step(dt)
    un1, _, p1 = one.get_state()
    assert np.array_equal(np.concatenate([t[1] for t in parts], axis=-3), un1)
    assert np.array_equal(np.concatenate([t[2] for t in parts], axis=-3), p1)
    one.close()
