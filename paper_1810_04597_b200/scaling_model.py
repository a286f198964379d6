"""Analytic strong-scaling model of the z-slab decomposition (SPEC.md's
performance model — Amdahl, halo strong scaling, sweet spot, SPEC.md:383-418 — re-targeted
from MPI on Xeon nodes to one NVSwitch box of B200s).

Per rank of an N-slab run of an n1 x n2 x n3 grid (nz = n3 / N planes):

    T(N) = t_plane * (nz + g) + t_launch * L + T_xchg(N)

  t_plane  device time per owned plane and step (all kernels), from the 1-GPU bench
  g        ghost-plane work per slab: the x/y sweeps also run on one ghost plane per
           side and the z sweep's lines are 2 cells longer (calibrated, below)
  L        kernel launches per step and slab (12 + the exchange launches)
  T_xchg   ghost exchange per step: 3 stages x 2 sides x 6 planes of halo messages, over
           NVLink.  Round 1's messages were whole P and U records (2 x 64 B per cell); round
           2's hold what the sweeps read (8 doubles per cell, `exchange_bytes(layout="r02")`).
           "copy": the exchange in series with the stage; "overlap" (round 2's default,
           DistSlab.step): the NCCL messages in flight while the stage's interior x/y sweeps
           run (a fraction f_xy of the stage's compute), only the excess exposed; "fused":
           folded into the update's stores (only the part that does not overlap the update,
           f_exposed)

Calibration (`calibrate`) fits t_plane, g and the exchange cost per byte to the measured
1-GPU runs (profiles/r01_bench_default.json and r01_bench_decomp_*.json, where the
"exchange" is a device copy or the update's own stores); `predict` then replaces the
device-copy bandwidth by NVLink's.  The model is a reported explanation, not a
measurement: the cross-GPU numbers await a multi-GPU box.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

HALO = 6
RECORD_BYTES = 64  # one 8-variable fp64 record


def amdahl(f: float, n: int) -> float:
    """Amdahl speed-up with serial fraction f on n workers (SPEC.md [OP] amdahl)."""
    if not 0.0 <= f <= 1.0 or n < 1:
        raise ValueError("f in [0, 1], n >= 1")
    return 1.0 / (f + (1.0 - f) / n)


def plane_bytes(n1: int, n2: int) -> int:
    """Bytes of one z plane of one record array (row-interleaved, padded rows)."""
    vs = n1 + (n1 & 1)
    return (8 * vs + 8) * n2 * 8


def exchange_bytes(n1: int, n2: int, layout: str = "r01") -> int:
    """Bytes a slab sends per step: 3 stages x 2 sides x 6 planes.  layout "r01": the P and U
    records (round 1); "r02": per row 8 x vs doubles (rho, u~, p from P, B from U)."""
    if layout == "r01":
        return 3 * 2 * HALO * 2 * plane_bytes(n1, n2)
    vs = n1 + (n1 & 1)
    return 3 * 2 * HALO * n2 * 8 * vs * 8


@dataclass
class Model:
    t_plane: float          # s per owned plane and step
    g: float                # ghost-plane equivalents per slab
    t_launch: float = 4e-6  # s per kernel launch (stream-ordered, no sync)
    copy_bw: float = 3.0e12     # B/s of the 1-GPU device-copy exchange (read + write in HBM)
    fused_exposed: float = 0.5  # fraction of the fused ghost stores not hidden by the update
    nvlink_bw: float = 0.7e12   # B/s per direction and GPU pair, effective (900 GB/s nominal)
    f_xy: float = 0.51          # x + y sweeps' share of a stage (profiles/r02_launch_shares.txt)
    plane_cells: int = 512 * 512  # cells of the calibration plane: t_plane scales with n1 n2

    def step_time(self, n: tuple, nslabs: int, mode: str = "copy", link: str = "nvlink") -> dict:
        """Per-step time of one slab (= the job, all slabs in parallel on separate GPUs)."""
        n1, n2, n3 = n
        nz = n3 / nslabs
        tp = self.t_plane * (n1 * n2) / self.plane_cells
        compute = tp * (nz + (self.g if nslabs > 1 else 0.0))
        layout = "r02" if mode == "overlap" else "r01"
        xb = exchange_bytes(n1, n2, layout) if nslabs > 1 else 0
        bw = self.nvlink_bw if link == "nvlink" else self.copy_bw
        if mode == "copy":
            xchg = xb / bw + 12 * self.t_launch
        elif mode == "overlap":  # per stage: the messages against the interior x/y sweeps
            per_stage = xb / 3 / bw
            hidden = self.f_xy * (tp * nz) / 3
            xchg = 3 * max(0.0, per_stage - hidden) + (12 * self.t_launch if nslabs > 1 else 0.0)
        elif mode == "fused":
            xchg = self.fused_exposed * xb / bw
        else:
            raise ValueError(mode)
        launches = 12 * self.t_launch
        total = compute + launches + xchg
        return {"nslabs": nslabs, "sec_per_step": total, "compute": compute, "launch": launches, "exchange": xchg}

    def curve(self, n, ranks, mode="copy") -> list[dict]:
        return [self.step_time(n, r, mode) for r in ranks]


def sweet_spot(curve: list[dict]) -> int:
    """Rank count at minimal time per step; ties go to fewer ranks (SPEC.md [OP] sweet_spot)."""
    if not curve:
        raise ValueError("empty curve")
    best = min(curve, key=lambda p: (p["sec_per_step"], p["nslabs"]))
    return best["nslabs"]


def calibrate(profiles_dir: str) -> Model:
    """t_plane from the 1-GPU bench; g and the copy bandwidth from the 1-GPU slab runs
    (S slabs on one GPU do S x the ghost work and S x the exchange of one slab)."""
    def ms(name):
        with open(os.path.join(profiles_dir, name)) as f:
            return json.load(f)["ms_per_step"] * 1e-3
    n = (512, 512, 512)
    t1 = ms("r01_bench_default.json")
    t_plane = t1 / n[2]
    m = Model(t_plane=t_plane, g=0.0)
    # one process holding S slabs on one GPU: S (nz + g) planes + S x the exchange, serialised
    s2, s4 = ms("r01_bench_decomp_slabs2.json"), ms("r01_bench_decomp_slabs4.json")
    xb = exchange_bytes(n[0], n[1])
    # two equations (S = 2, 4): extra = S g t_plane + S xb / copy_bw + 12 S t_launch
    e2, e4 = s2 - t1, s4 - t1
    per_slab_launch = 12 * m.t_launch
    # solve e_S = S (g t_plane + xb / bw + launch) for the S-independent per-slab cost c
    c = (e2 / 2 + e4 / 4) / 2 - per_slab_launch
    # split c between ghost work and the copies with the fused runs (no copies)
    f2, f4 = ms("r01_bench_decomp_slabs2_fused.json"), ms("r01_bench_decomp_slabs4_fused.json")
    cf = ((f2 - t1) / 2 + (f4 - t1) / 4) / 2 - per_slab_launch
    m.g = max(cf, 0.0) / t_plane
    copy_cost = max(c - cf, 1e-6)
    m.copy_bw = xb / copy_cost
    return m
