"""z-slab domain decomposition of the time step.

The paper's code scales by a Cartesian MPI domain decomposition with a ghost
exchange per stage.  Here every rank (one process per GPU)
owns a contiguous block of z planes of the global grid; its context has z
boundaries of kind BC_HALO (stored ghost planes, echo.h) and, before every RK
stage, the 6 boundary planes of P and U^s travel to the neighbours:

    for s in 1, 2, 3:  exchange()  ->  echo_stage(s, dt)

with dt = the minimum over ranks of each slab's CFL dt (the max signal speed is
a max over cells, so the decomposed dt equals the single-domain one bit for bit).
The library does the arithmetic (export/import are stream-ordered device copies);
this module only pairs the messages: torch.distributed point-to-point (NCCL over
NVLink on GPUs, gloo on CPU) between ranks, or direct copies between slabs held by
one process (`LocalSlabs`, which makes the decomposed step testable on one GPU).
"""
from __future__ import annotations

import math
from dataclasses import replace

LOWER, UPPER = 0, 1


def decompose_z(n3: int, nranks: int, min_planes: int = 6) -> list[tuple[int, int]]:
    """(z0, nz) of each rank: contiguous, balanced (sizes differ by at most one plane),
    every slab at least HALO_PLANES = 6 planes thick (UCT: HALO_PLANES_UCT = 8)."""
    if nranks < 1:
        raise ValueError("nranks >= 1")
    base, extra = divmod(n3, nranks)
    if base < min_planes:
        raise ValueError(f"{n3} planes cannot give {nranks} slabs of >= {min_planes} planes")
    out, z0 = [], 0
    for r in range(nranks):
        nz = base + (1 if r < extra else 0)
        out.append((z0, nz))
        z0 += nz
    return out


def neighbours(rank: int, nranks: int, periodic: bool) -> tuple[int | None, int | None]:
    """(lower, upper) neighbour ranks along z; None at a physical (outflow) end."""
    lo = rank - 1 if rank > 0 else (nranks - 1 if periodic else None)
    hi = rank + 1 if rank < nranks - 1 else (0 if periodic else None)
    return lo, hi


def slab_problem(problem, rank: int, nranks: int):
    """The rank's slab of an echo_inputs.Problem: its z planes and coordinate range, z
    boundaries BC_HALO towards neighbours and the global rule at physical ends."""
    from .echo import BC_HALO

    z0, nz = decompose_z(problem.n[2], nranks, 8 if getattr(problem, "divb", 0) == 2 else 6)[rank]
    dz = (problem.hi[2] - problem.lo[2]) / problem.n[2]
    periodic = problem.bc[2][0] == 0
    lo_nb, hi_nb = neighbours(rank, nranks, periodic)
    bcz = (BC_HALO if lo_nb is not None else problem.bc[2][0], BC_HALO if hi_nb is not None else problem.bc[2][1])
    bc = (tuple(problem.bc[0]), tuple(problem.bc[1]), bcz)
    # the slab's Delta_z is the global one bit for bit (every z difference and the CFL rate divide
    # by it; (hi - lo) / nz of the slab's own bounds can differ in the last bits): echo_grid.dz
    return replace(problem, n=(problem.n[0], problem.n[1], nz), lo=(problem.lo[0], problem.lo[1], problem.lo[2] + z0 * dz),
                   hi=(problem.hi[0], problem.hi[1], problem.lo[2] + (z0 + nz) * dz), bc=bc, dz=dz), (z0, nz)


class LocalSlabs:
    """All slabs of one grid in one process (one GPU): the decomposed step with the
    ghost exchange done by device-to-device copies between the contexts, or, fused=True,
    by the update kernels storing their edge planes straight into the neighbours' ghost
    planes (echo_halo_link; per stage all sweeps, then all updates)."""

    def __init__(self, problem, nslabs: int, device="cuda", fused: bool = False):
        import torch

        from . import echo as E

        self.E = E
        self.problem = problem
        self.periodic = problem.bc[2][0] == 0
        self.parts = []
        for r in range(nslabs):
            sp, (z0, nz) = slab_problem(problem, r, nslabs)
            self.parts.append((E.Echo(sp), z0, nz))
        nd = E.halo_doubles(self.parts[0][0].ctx)
        self.buf = torch.empty(nd, dtype=torch.float64, device=device)
        self.uct = getattr(problem, "divb", 0) == 2 and nd > 0  # UCT slabs: the two-part update
        self.fbuf = torch.empty(E.halo_field_doubles(self.parts[0][0].ctx), dtype=torch.float64, device=device)
        self.fused = fused
        if fused:
            for r, (g, _, _) in enumerate(self.parts):
                lo, hi = neighbours(r, nslabs, self.periodic)
                for side, nb in ((LOWER, lo), (UPPER, hi)):
                    if nb is not None:
                        E.halo_link(g.ctx, side, self.parts[nb][0].ctx)

    def set_face_field(self, b3):
        """UCT (divb = 2): the global staggered field [3][n3][n2][n1].  Each slab's centring
        U_B = I6(b) reads b^z of 3 faces beyond its planes: set, exchange, and set again (the
        second pass centres the edge cells with the neighbours' faces in the ghost planes)."""
        for _ in range(2):
            for g, z0, nz in self.parts:
                x = b3[:, z0:z0 + nz]
                g.set_face_field(x.contiguous() if hasattr(x, "contiguous") else x.copy())
            self.exchange()

    def set_prims(self, p8):
        """p8: the global user prims [8][n3][n2][n1] (numpy, or a torch CUDA tensor)."""
        for g, z0, nz in self.parts:
            x = p8[:, z0:z0 + nz]
            g.set_prims(x.contiguous() if hasattr(x, "contiguous") else x.copy())
        if self.fused:  # the first stage's ghosts; later ones are written by the updates
            self.exchange()

    def exchange(self):
        E, n = self.E, len(self.parts)
        if self.buf.numel() == 0:  # one slab of a non-periodic z axis: no halo side at all
            return
        for r, (g, _, _) in enumerate(self.parts):
            lo, hi = neighbours(r, n, self.periodic)
            for side, nb in ((LOWER, lo), (UPPER, hi)):
                if nb is None:
                    E.halo_fill(g.ctx, side)
                else:  # my side-`side` ghosts = the neighbour's planes next to its opposite side
                    E.halo_export(self.parts[nb][0].ctx, 1 - side, self.buf)
                    E.halo_import(g.ctx, side, self.buf)

    def exchange_field(self):
        """UCT slabs: the new b^z of the 3 edge planes of every slab, after the inductions."""
        E, n = self.E, len(self.parts)
        for r, (g, _, _) in enumerate(self.parts):
            lo, hi = neighbours(r, n, self.periodic)
            for side, nb in ((LOWER, lo), (UPPER, hi)):
                if nb is None:
                    E.halo_fill_field(g.ctx, side)
                else:
                    E.halo_export_field(self.parts[nb][0].ctx, 1 - side, self.fbuf)
                    E.halo_import_field(g.ctx, side, self.fbuf)

    def max_dt(self, cfl: float) -> float:
        return min(g.max_dt(cfl) for g, _, _ in self.parts)

    def step(self, dt: float, split: bool = False):
        """split=True (copy exchange): each slab's interior sweeps first, then the exchange, the
        boundary sweeps and the updates -- DistSlab.step's order, on one GPU."""
        E = self.E
        for s in (1, 2, 3):
            if self.fused:
                for g, _, _ in self.parts:
                    E.stage_sweeps(g.ctx, s)
                for g, _, _ in self.parts:
                    E.stage_update(g.ctx, s, dt)
            elif self.uct:  # sweeps + EMFs, induction, new-field exchange, cell update
                self.exchange()
                for g, _, _ in self.parts:
                    E.stage_sweeps(g.ctx, s)
                    E.stage_update_field(g.ctx, s, dt)
                self.exchange_field()
                for g, _, _ in self.parts:
                    E.stage_update_cells(g.ctx, s, dt)
            elif split and self.buf.numel() > 0 and getattr(self.problem, "divb", 0) != 2:
                for g, _, _ in self.parts:
                    E.stage_sweeps_interior(g.ctx, s)
                self.exchange()
                for g, _, _ in self.parts:
                    E.stage_sweeps_boundary(g.ctx, s)
                    E.stage_update(g.ctx, s, dt)
            else:
                self.exchange()
                for g, _, _ in self.parts:
                    g.stage(s, dt)

    def gather(self, getter):
        import numpy as np

        return np.concatenate([getter(g) for g, _, _ in self.parts], axis=-3)

    def close(self):
        for g, _, _ in self.parts:
            for side in (LOWER, UPPER):
                try:
                    self.E.halo_link(g.ctx, side, None)
                except Exception:
                    pass
        for g, _, _ in self.parts:
            g.close()


class DistSlab:
    """This rank's slab under torch.distributed: point-to-point ghost exchange with the
    z neighbours (send my boundary planes, receive theirs), min-reduced CFL dt.
    `io` supplies export(side, buf) / import_(side, buf) / fill(side) / halo_doubles
    (the library context by default; a host stand-in in the CPU tests).

    Fused mode (`link_fused`, GPUs): the neighbours' arrays are mapped by CUDA IPC and
    every update stores its edge planes straight into them (NVLink peer stores); a
    step is then, per stage, sweeps -> stream sync + barrier -> update -> sync +
    barrier, with no data messages at all."""

    def __init__(self, io, rank: int, nranks: int, periodic: bool, device, split: bool = True, uct: bool = False):
        """split=False: the exchange precedes the whole stage (no interior/boundary halves).
        uct=True (UCT slabs, echo.h): per stage the exchange, the sweeps, the induction, the
        new-field exchange (io.export_field / import_field / fill_field), the cell update."""
        import torch

        self.io, self.rank, self.n, self.split, self.uct = io, rank, nranks, split and not uct, uct
        self.lo, self.hi = neighbours(rank, nranks, periodic)
        nd = io.halo_doubles()
        self.send = [torch.empty(nd, dtype=torch.float64, device=device) for _ in range(2)]
        self.recv = [torch.empty(nd, dtype=torch.float64, device=device) for _ in range(2)]
        nf = io.halo_field_doubles() if uct else 0
        self.fsend = [torch.empty(nf, dtype=torch.float64, device=device) for _ in range(2)]
        self.frecv = [torch.empty(nf, dtype=torch.float64, device=device) for _ in range(2)]

    def exchange(self, overlap=None):
        self._pair(self.send, self.recv, self.io.export, self.io.import_, self.io.fill, overlap)

    def exchange_field(self):
        """UCT slabs: the new b^z of the 3 edge planes, after this stage's induction."""
        self._pair(self.fsend, self.frecv, self.io.export_field, self.io.import_field, self.io.fill_field)

    def _pair(self, send, recv, export, import_, fill, overlap=None):
        """The ghost exchange of one stage, stream-ordered: the exports are kernels on the
        compute stream, and NCCL's stream waits for them (torch orders a collective after the
        work already issued on the current stream), so the host never synchronises; `overlap`
        (e.g. the stage's interior sweeps, echo_stage_sweeps_interior) is issued on the compute
        stream while the messages are in flight; req.wait() then makes the compute stream wait
        for NCCL before the imports.  (gloo, the CPU tests: wait() blocks the host.)"""
        import torch.distributed as dist

        if send[0].numel() == 0:  # a single rank on a non-periodic z axis: no halo side
            if overlap is not None:
                overlap()
            return
        # sends in the order (upper planes, lower planes), receives (lower ghosts, upper ghosts),
        # tagged with the side of the sender's planes: with two ranks both neighbours are the
        # same peer, and NCCL ignores tags and matches point-to-point messages in issue order
        for side, nb in ((LOWER, self.lo), (UPPER, self.hi)):
            if nb is not None:
                export(side, send[side])
        ops = []
        for side, nb in ((UPPER, self.hi), (LOWER, self.lo)):
            if nb is not None and nb != self.rank:
                ops.append(dist.P2POp(dist.isend, send[side], nb, tag=side))
        for side, nb in ((LOWER, self.lo), (UPPER, self.hi)):
            if nb is not None and nb != self.rank:
                ops.append(dist.P2POp(dist.irecv, recv[side], nb, tag=1 - side))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        if overlap is not None:
            overlap()
        for req in reqs:
            req.wait()
        for side, nb in ((LOWER, self.lo), (UPPER, self.hi)):
            if nb is None:
                fill(side)
            elif nb == self.rank:
                import_(side, send[1 - side])
            else:
                import_(side, recv[side])

    def step(self, dt: float):
        """One SSP-RK3 step with the exchange overlapped by each stage's interior sweeps."""
        for s in (1, 2, 3):
            if self.send[0].numel() == 0:  # no halo side (one rank, non-periodic z): a plain stage
                self.io.sweeps(s)
            elif self.uct:
                self.exchange()
                self.io.sweeps(s)
                self.io.update_field(s, dt)
                self.exchange_field()
                self.io.update_cells(s, dt)
                continue
            elif not self.split:
                self.exchange()
                self.io.sweeps(s)
            else:
                self.exchange(overlap=lambda s=s: self.io.sweeps_interior(s))
                self.io.sweeps_boundary(s)
            self.io.update(s, dt)

    def link_fused(self):
        """Exchange the slabs' IPC handles and link both z sides (a self-neighbour, i.e. a
        single periodic rank, links in-process); then pull the first stage's ghosts."""
        import torch.distributed as dist

        mine = self.io.ipc_export()
        allh = [None] * self.n
        dist.all_gather_object(allh, mine)
        for side, nb in ((LOWER, self.lo), (UPPER, self.hi)):
            if nb is None:
                continue
            if nb == self.rank:
                self.io.link_self(side)
            else:
                self.io.link_ipc(side, *allh[nb])
        self.fused = True
        self.barrier()
        for side, nb in ((LOWER, self.lo), (UPPER, self.hi)):
            if nb is None:
                self.io.fill(side)
            else:
                self.io.pull(side)
        self.barrier()

    def barrier(self):
        import torch.distributed as dist

        self.io.sync()
        dist.barrier()

    def set_face_field(self, b3_slab):
        """UCT: this rank's part of the staggered field; set, exchange, set again (the centring of
        the edge cells reads the neighbours' faces, see LocalSlabs.set_face_field)."""
        for _ in range(2):
            self.io.set_face_field(b3_slab)
            self.exchange()

    def step_fused(self, dt: float):
        for s in (1, 2, 3):
            self.io.sweeps(s)
            self.barrier()   # every neighbour finished reading the ghost planes my update overwrites
            self.io.update(s, dt)
            self.barrier()   # my ghost planes hold the neighbours' new edge planes

    def min_dt(self, dt_local: float) -> float:
        import torch
        import torch.distributed as dist

        t = torch.tensor([dt_local], dtype=torch.float64, device=self.send[0].device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return float(t.item())


class CtxIO:
    """DistSlab's io over a library context (device buffers on the context stream)."""

    def __init__(self, echo_obj):
        from . import echo as E

        self.E, self.g = E, echo_obj

    def halo_doubles(self):
        return self.E.halo_doubles(self.g.ctx)

    def export(self, side, buf):
        self.E.halo_export(self.g.ctx, side, buf)

    def import_(self, side, buf):
        self.E.halo_import(self.g.ctx, side, buf)

    def fill(self, side):
        self.E.halo_fill(self.g.ctx, side)

    def sync(self):
        import torch

        torch.cuda.current_stream().synchronize()

    def ipc_export(self):
        return self.E.ipc_export(self.g.ctx)

    def link_ipc(self, side, handles, nz):
        self.E.halo_link_ipc(self.g.ctx, side, handles, nz)

    def link_self(self, side):
        self.E.halo_link(self.g.ctx, side, self.g.ctx)

    def pull(self, side):
        self.E.halo_pull(self.g.ctx, side)

    def sweeps(self, s):
        self.E.stage_sweeps(self.g.ctx, s)

    def set_face_field(self, b3):
        self.g.set_face_field(b3)

    def halo_field_doubles(self):
        return self.E.halo_field_doubles(self.g.ctx)

    def export_field(self, side, buf):
        self.E.halo_export_field(self.g.ctx, side, buf)

    def import_field(self, side, buf):
        self.E.halo_import_field(self.g.ctx, side, buf)

    def fill_field(self, side):
        self.E.halo_fill_field(self.g.ctx, side)

    def update_field(self, s, dt):
        self.E.stage_update_field(self.g.ctx, s, dt)

    def update_cells(self, s, dt):
        self.E.stage_update_cells(self.g.ctx, s, dt)

    def sweeps_interior(self, s):
        self.E.stage_sweeps_interior(self.g.ctx, s)

    def sweeps_boundary(self, s):
        self.E.stage_sweeps_boundary(self.g.ctx, s)

    def update(self, s, dt):
        self.E.stage_update(self.g.ctx, s, dt)
