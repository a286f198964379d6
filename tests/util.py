"""Shared test helpers: the normwise per-group parity metric of DESIGN.md reading A16."""
from __future__ import annotations

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


def assert_rhs_groups(got, ref, U, dt, groups, tol, what=""):
    """L comparisons (A16 for residuals): the group scale is max(max|L|, max|U|/dt), because
    the L of a group near equilibrium is a truncation-level residual of cancelling flux
    differences whose rounding scales with |U|/dt, not with |L|."""
    got, ref, U = np.asarray(got), np.asarray(ref), np.asarray(U)
    errs = {}
    for name, idx in groups.items():
        g, r, u = got[idx], ref[idx], U[idx]
        scale = max(float(np.max(np.abs(r))), float(np.max(np.abs(u))) / dt)
        errs[name] = float(np.max(np.abs(g - r))) / scale if scale > 0 else float(np.max(np.abs(g - r)))
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"{what}: rhs group error above {tol:g}: {errs}"
    return errs
