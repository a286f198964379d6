"""Maximum sizes (the north star's edge cases): a grid near the largest one a B200's HBM holds
(256 B of state per cell, ~820^3) steps correctly -- conserved sums, no floor or
Newton failure, a finite CFL step -- and a grid beyond it is refused loudly (ECHO_E_OOM) with
everything it allocated given back.  Marked gpu; skipped on a device with less free memory."""
import math

import numpy as np
import pytest

import echo_inputs as I

pytestmark = pytest.mark.gpu

N_MAX = 800  # 5.1e8 cells: 131 GB of state + a 33 GB input / output tensor (of ~820^3 at most)


@pytest.fixture(scope="module")
def E():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1810_04597_b200 import build

    build.build()
    from paper_1810_04597_b200 import echo

    return echo


def smooth_state(torch, n, dev):
    """a smooth periodic MHD state [8][n][n][n] built plane-broadcast on the device (one full-size
    temporary at a time): rho, p ~ 1 +- 20 %, |v| <= 0.3, B = 0.5 + a divergence-free sinusoid"""
    x = (torch.arange(n, device=dev, dtype=torch.float64) + 0.5) / n
    s = torch.sin(2 * math.pi * x)
    c = torch.cos(2 * math.pi * x)
    X, Y, Z = s.view(1, 1, n), s.view(1, n, 1), s.view(n, 1, 1)
    CX, CY, CZ = c.view(1, 1, n), c.view(1, n, 1), c.view(n, 1, 1)
    P8 = torch.empty((8, n, n, n), device=dev, dtype=torch.float64)
    P8[0] = 1.0 + 0.2 * X * Y * CZ
    P8[1] = 0.3 * Y * CZ
    P8[2] = 0.3 * Z * CX
    P8[3] = 0.3 * X * CY
    P8[4] = 1.0 + 0.2 * CX * CY * Z
    P8[5] = 0.5 + 0.1 * Y * Z   # B^x independent of x, etc.: divergence free
    P8[6] = 0.5 + 0.1 * Z * X
    P8[7] = 0.5 + 0.1 * X * Y
    return P8


def test_near_maximum_grid_steps_and_conserves(E):
    import torch

    n = N_MAX
    need = n ** 3 * (256 + 64) + (8 << 30)
    free, _ = torch.cuda.mem_get_info()
    if free < need:
        pytest.skip(f"needs {need / 2**30:.0f} GiB free, {free / 2**30:.0f} GiB available")
    dev = torch.device("cuda", 0)
    p = I.problem(3, n=(n, n, n))
    g = E.Echo(p)
    P8 = smooth_state(torch, n, dev)
    g.set_prims(P8)
    del P8
    torch.cuda.empty_cache()
    U = torch.empty((8, n, n, n), device=dev, dtype=torch.float64)
    E.get_cons(g.ctx, U)
    before = np.array([float(U[v].sum()) for v in range(8)])  # (one variable's temporary at a time)
    scale = np.array([float(U[v].abs().sum()) for v in range(8)])
    dt = g.max_dt(p.cfl)
    assert math.isfinite(dt) and dt > 0.0
    g.step(dt)
    g.step(g.max_dt(p.cfl))
    E.get_cons(g.ctx, U)
    after = np.array([float(U[v].sum()) for v in range(8)])
    assert all(bool(torch.isfinite(U[v]).all()) for v in range(8))
    del U
    st = g.stats()
    g.close()
    torch.cuda.empty_cache()
    assert st["floor_events"] == 0 and st["c2p_failures"] == 0 and st["steps"] == 2
    # periodic: every conserved sum (D, S_i, tau, B^i) changes by roundoff only
    assert np.all(np.abs(after - before) <= 1e-12 * scale), (before, after, scale)


def test_beyond_memory_is_refused_and_released(E):
    import torch

    torch.cuda.empty_cache()
    free0, total = torch.cuda.mem_get_info()
    n = int(round((total / 200.0) ** (1.0 / 3.0))) + 64  # > total / 256 B cells
    p = I.problem(3, n=(n, n, n))
    with pytest.raises(E.EchoError) as ei:
        E.Echo(p)
    assert "alloc" in str(ei.value).lower() or "memory" in str(ei.value).lower()
    free1, _ = torch.cuda.mem_get_info()
    assert free1 >= free0 - (256 << 20), (free0, free1)  # nothing left behind
    q = I.problem(0, n=(32, 32, 32))  # and the library still works
    g = E.Echo(q)
    g.set_prims(I.initial_prims(q))
    g.step(g.max_dt(q.cfl))
    g.close()
