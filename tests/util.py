"""Shared test helpers: the normwise per-group parity metric of DESIGN.md reading A16."""
from __future__ import annotations

import json
import os

import numpy as np

CONS_GROUPS = {"D": [0], "S": [1, 2, 3], "tau": [4], "B": [5, 6, 7]}
PRIM5_GROUPS = {"rho": [0], "u": [1, 2, 3], "p": [4]}
PRIM8_GROUPS = {"rho": [0], "v": [1, 2, 3], "p": [4], "B": [5, 6, 7]}


def group_errors(got, ref, groups, axis=0) -> dict:
    """max_cells |got - ref| / max_cells |ref| per variable group (scale shared inside a group)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    out = {}
    for name, idx in groups.items():
        g = np.take(got, idx, axis=axis)
        r = np.take(ref, idx, axis=axis)
        scale = float(np.max(np.abs(r))) if r.size else 0.0
        err = float(np.max(np.abs(g - r))) if r.size else 0.0
        out[name] = err / scale if scale > 0 else err
    return out


def assert_groups(got, ref, groups, tol, axis=0, what=""):
    errs = group_errors(got, ref, groups, axis)
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"{what}: normwise group error above {tol:g}: {errs}"
    return errs


def flux_scale(orc, oc, U, P5, groups=CONS_GROUPS, nsample=512, seed=0) -> dict:
    """Per group: max over sampled cells and the three axes of |sqrt(g) F^a_q| / Delta_a,
    the size of one flux difference term of L (a4).  A max over a SAMPLE is <= the max
    over the grid, so a scale from it is never looser than the grid's max |F| / Delta.
    Fluxes from the oracle's pinned physical flux (orc_flux_pt) at the cell centres."""
    U, P5 = np.asarray(U), np.asarray(P5)
    n3, n2, n1 = P5.shape[1:]
    rng = np.random.default_rng(seed)
    cnt = min(nsample, n1 * n2 * n3)
    lin = rng.choice(n1 * n2 * n3, size=cnt, replace=False)
    dx = [oc.dx(a) for a in range(3)]
    best = np.zeros(8)
    for m in lin:
        k, r = divmod(int(m), n1 * n2)
        j, i = divmod(r, n1)
        x = [oc.lo[0] + (i + 0.5) * dx[0], oc.lo[1] + (j + 0.5) * dx[1], oc.lo[2] + (k + 0.5) * dx[2]]
        sg = orc.metric(oc, x)["sqrtg"]
        pr = [*P5[:, k, j, i], *(U[5:8, k, j, i] / sg)]
        for a in range(3):
            f = orc.flux_pt(oc, x, pr, a)
            best = np.maximum(best, np.abs(f) * sg / dx[a])
    return {name: float(np.max(best[idx])) for name, idx in groups.items()}


def assert_rhs_groups(got, ref, U, dt, groups, tol, what="", fscale=None):
    """L comparisons (A16 for residuals).  Three group scales are computed:
      'L'     max |L_ref|                      (A16 as SURVEY states it)
      'F'     max(max |L|, max |F| / Delta)    (the size of one flux-difference term)
      'U/dt'  max(max |L|, max |U| / dt)       (round 1's scale)
    The asserted one is 'F' when the caller passes `fscale` (flux_scale()), else 'U/dt'.
    The L of a group near equilibrium (D in the CP Alfven wave) is a truncation-level residual
    of cancelling flux differences; its rounding scales with |F|/Delta, not with |L|, so 'L'
    alone is reported, not asserted.  With ECHO_PARITY_LOG=path every call appends all three."""
    got, ref, U = np.asarray(got), np.asarray(ref), np.asarray(U)
    errs, rep = {}, {}
    for name, idx in groups.items():
        g, r, u = got[idx], ref[idx], U[idx]
        d = float(np.max(np.abs(g - r)))
        sL = float(np.max(np.abs(r)))
        sU = max(sL, float(np.max(np.abs(u))) / dt)
        sF = max(sL, fscale[name]) if fscale is not None else None
        rep[name] = {"L": d / sL if sL > 0 else d, "U/dt": d / sU if sU > 0 else d}
        if sF is not None:
            rep[name]["F"] = d / sF if sF > 0 else d
        errs[name] = rep[name]["F" if sF is not None else "U/dt"]
    log = os.environ.get("ECHO_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps({"what": what, "tol": tol, "asserted": "F" if fscale is not None else "U/dt",
                                "errors": rep}) + "\n")
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"{what}: rhs group error above {tol:g}: {rep}"
    return errs
