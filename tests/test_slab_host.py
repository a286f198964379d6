"""z-slab decomposition host logic, CPU only:
the split of the planes, the neighbour map, and the point-to-point ghost exchange
of paper_1810_04597_b200/slab.py over torch.distributed with world_size 2 and 3 on
gloo, with a host stand-in for the library's export/import (planes carry their
global index, so every ghost plane must end up holding the right neighbour plane)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

H = 6  # ghost planes per side (echo.h ECHO_HALO_PLANES)


def _slab_module():
    # slab.py imports the library lazily; import the module file without the package __init__
    import importlib.util

    spec = importlib.util.spec_from_file_location("slab", os.path.join(ROOT, "paper_1810_04597_b200", "slab.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_decompose_z():
    S = _slab_module()
    assert S.decompose_z(512, 8) == [(64 * r, 64) for r in range(8)]
    parts = S.decompose_z(100, 7)
    assert sum(nz for _, nz in parts) == 100 and max(nz for _, nz in parts) - min(nz for _, nz in parts) <= 1
    assert all(parts[r + 1][0] == parts[r][0] + parts[r][1] for r in range(6))
    with pytest.raises(ValueError):
        S.decompose_z(20, 4)  # 5-plane slabs are thinner than the halo


def test_neighbours():
    S = _slab_module()
    assert S.neighbours(0, 4, True) == (3, 1)
    assert S.neighbours(3, 4, True) == (2, 0)
    assert S.neighbours(0, 4, False) == (None, 1)
    assert S.neighbours(3, 4, False) == (2, None)
    assert S.neighbours(0, 1, True) == (0, 0)


class HostIO:
    """Stand-in for the library: a slab of nz planes (value = global plane index + 0.5 x variable)
    with H stored ghost planes per side; export / import / fill as echo.h specifies."""

    def __init__(self, z0, nz, nzg, nvar=3):
        self.z0, self.nz, self.nvar = z0, nz, nvar
        self.a = np.full((nz + 2 * H, nvar), np.nan)
        for k in range(nz):
            self.a[H + k] = z0 + k + 0.5 * np.arange(nvar)

    def halo_doubles(self):
        return H * self.nvar

    def export(self, side, buf):
        k0 = 0 if side == 0 else self.nz - H
        buf.copy_(torch.from_numpy(self.a[H + k0:H + k0 + H].ravel().copy()))

    def import_(self, side, buf):
        k0 = 0 if side == 0 else H + self.nz
        self.a[k0:k0 + H] = buf.numpy().reshape(H, self.nvar)

    def fill(self, side):
        if side == 0:
            self.a[:H] = self.a[H]
        else:
            self.a[H + self.nz:] = self.a[H + self.nz - 1]

    def sync(self):
        pass


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nzg, periodic, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    S = _slab_module()
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z0, nz = S.decompose_z(nzg, world)[rank]
    io = HostIO(z0, nz, nzg)
    slab = S.DistSlab(io, rank, world, periodic, "cpu")
    slab.exchange()
    dt = slab.min_dt(0.1 * (rank + 1))
    out[rank] = (io.a.copy(), z0, nz, dt)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nzg,periodic", [(2, 24, True), (3, 40, True), (2, 24, False), (3, 37, False)])
def test_dist_ghost_exchange_gloo(world, nzg, periodic):
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _port(), nzg, periodic, out), nprocs=world, join=True)
    for r in range(world):
        a, z0, nz, dt = out[r]
        assert dt == pytest.approx(0.1)  # the min over ranks
        for h in range(1, H + 1):
            for side, k_local, k_global in ((0, H - h, z0 - h), (1, H + nz - 1 + h, z0 + nz - 1 + h)):
                if periodic:
                    want = k_global % nzg
                else:  # physical outflow ends replicate the edge plane
                    want = min(max(k_global, 0), nzg - 1)
                assert a[k_local, 0] == want, (r, side, h, a[k_local])
                assert np.array_equal(a[k_local], want + 0.5 * np.arange(3))


class LogIO(HostIO):
    """HostIO that records the call order of DistSlab.step."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.log = []

    def export(self, side, buf):
        self.log.append(("export", side))
        super().export(side, buf)

    def import_(self, side, buf):
        self.log.append(("import", side))
        super().import_(side, buf)

    def fill(self, side):
        self.log.append(("fill", side))
        super().fill(side)

    def sweeps_interior(self, s):
        self.log.append(("interior", s))

    def sweeps_boundary(self, s):
        self.log.append(("boundary", s))

    def update(self, s, dt):
        self.log.append(("update", s))


def _step_worker(rank, world, port, nzg, periodic, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    S = _slab_module()
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z0, nz = S.decompose_z(nzg, world)[rank]
    io = LogIO(z0, nz, nzg)
    slab = S.DistSlab(io, rank, world, periodic, "cpu")
    slab.step(0.01)
    out[rank] = (io.log, io.a.copy(), z0, nz)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,periodic", [(2, True), (3, False)])
def test_dist_step_overlaps_exchange_with_interior_sweeps(world, periodic):
    """DistSlab.step, per stage: both exports, the interior sweeps (issued while the messages are
    in flight), then the imports / outflow fills, the boundary sweeps and the update, in this
    order; the ghost planes hold the neighbours' planes (echo.h, echo_stage_sweeps_interior)."""
    nzg = 30
    out = mp.Manager().dict()
    mp.spawn(_step_worker, args=(world, _port(), nzg, periodic, out), nprocs=world, join=True)
    for r in range(world):
        log, a, z0, nz = out[r]
        for s in (1, 2, 3):
            i_int = log.index(("interior", s))
            i_bnd = log.index(("boundary", s))
            i_upd = log.index(("update", s))
            exports = [k for k, e in enumerate(log) if e[0] == "export" and k < i_int and
                       (s == 1 or k > log.index(("update", s - 1)))]
            ins = [k for k, e in enumerate(log) if e[0] in ("import", "fill") and i_int < k < i_bnd]
            assert len(ins) == 2 and i_int < i_bnd < i_upd, log
            nb = S_neighbours(r, world, periodic)
            assert len(exports) == sum(x is not None for x in nb), log
        for h in range(1, H + 1):
            k_global = z0 - h
            want = k_global % nzg if periodic else min(max(k_global, 0), nzg - 1)
            assert a[H - h, 0] == want


def S_neighbours(r, world, periodic):
    return _slab_module().neighbours(r, world, periodic)
