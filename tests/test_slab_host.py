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
