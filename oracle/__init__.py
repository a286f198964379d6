"""CPU fp64 oracle of the ECHO-3DHPC time-step hot path — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_1810_04597_b200`` never imports it and shares no code with it.

This module is a ctypes loader for ``liboracle.so`` (plain C, see oracle.h for
what every function computes and which DESIGN.md reading it follows).  All
array arguments are C-contiguous float64 numpy arrays in the public layout
``[var][n3][n2][n1]`` (x1 fastest).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = ["oracle_metric.c", "oracle_physics.c", "oracle_scheme.c"]
LIB_PATH = os.path.join(_HERE, "liboracle.so")

# -O2 -ffp-contract=off: no fused multiply-add contraction, no fast-math
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (cheap; done on demand)."""
    srcs = [os.path.join(_HERE, s) for s in _SRC]
    hdrs = [os.path.join(_HERE, h) for h in ("oracle.h", "oracle_internal.h")]
    if not force and os.path.exists(LIB_PATH):
        t = os.path.getmtime(LIB_PATH)
        if all(os.path.getmtime(s) <= t for s in srcs + hdrs):
            return LIB_PATH
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", *CFLAGS, *srcs, "-o", tmp, "-lm"])
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class _Cfg(C.Structure):
    _fields_ = [
        ("n", C.c_int * 3),
        ("lo", C.c_double * 3),
        ("hi", C.c_double * 3),
        ("bc", (C.c_int * 2) * 3),
        ("metric", C.c_int),
        ("M", C.c_double),
        ("a", C.c_double),
        ("gamma", C.c_double),
        ("rho_floor", C.c_double),
        ("p_floor", C.c_double),
        ("w_max", C.c_double),
        ("c2p_max_iter", C.c_int),
        ("c2p_tol", C.c_double),
        ("rec", C.c_int),
        ("der", C.c_int),
        ("divb", C.c_int),
        ("der_jump", C.c_double),
        ("nthreads", C.c_int),
    ]


class _Counts(C.Structure):
    _fields_ = [("floor_events", C.c_longlong), ("c2p_failures", C.c_longlong)]


PERIODIC, OUTFLOW = 0, 1
MINKOWSKI, KERR_SCHILD = 0, 1


@dataclass
class Cfg:
    """Problem description for the oracle (mirrors echo_grid/echo_metric/echo_eos)."""

    n: tuple = (8, 8, 8)
    lo: tuple = (0.0, 0.0, 0.0)
    hi: tuple = (1.0, 1.0, 1.0)
    bc: tuple = ((PERIODIC, PERIODIC),) * 3
    metric: int = MINKOWSKI
    M: float = 1.0
    a: float = 0.0
    gamma: float = 4.0 / 3.0
    rho_floor: float = 1e-8
    p_floor: float = 1e-10
    w_max: float = 50.0
    c2p_max_iter: int = 30
    c2p_tol: float = 1e-13
    rec: int = 0
    der: int = 6
    divb: int = 0
    der_jump: float = 0.5
    nthreads: int = 0

    def c(self) -> _Cfg:
        s = _Cfg()
        for i in range(3):
            s.n[i] = int(self.n[i])
            s.lo[i] = float(self.lo[i])
            s.hi[i] = float(self.hi[i])
            s.bc[i][0] = int(self.bc[i][0])
            s.bc[i][1] = int(self.bc[i][1])
        for k in ("metric", "c2p_max_iter", "rec", "der", "divb", "nthreads"):
            setattr(s, k, int(getattr(self, k)))
        for k in ("M", "a", "gamma", "rho_floor", "p_floor", "w_max", "c2p_tol", "der_jump"):
            setattr(s, k, float(getattr(self, k)))
        return s

    @property
    def ncells(self) -> int:
        return int(self.n[0]) * int(self.n[1]) * int(self.n[2])

    def shape(self, nvar: int) -> tuple:
        return (nvar, int(self.n[2]), int(self.n[1]), int(self.n[0]))

    def dx(self, a: int) -> float:
        return (self.hi[a] - self.lo[a]) / self.n[a]


_lib = None
_D = C.POINTER(C.c_double)
_LL = C.POINTER(C.c_longlong)


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P = C.POINTER(_Cfg)
        sig = {
            "orc_metric": (C.c_int, [P, _D, _D]),
            "orc_metric_deriv": (C.c_int, [P, _D, _D]),
            "orc_prim2cons_pt": (C.c_int, [P, _D, _D, _D]),
            "orc_flux_pt": (C.c_int, [P, _D, _D, C.c_int, _D]),
            "orc_speeds_pt": (C.c_int, [P, _D, _D, C.c_int, _D]),
            "orc_hll_pt": (C.c_int, [P, _D, _D, _D, C.c_int, _D]),
            "orc_sources_pt": (C.c_int, [P, _D, _D, _D]),
            "orc_weno5_left": (C.c_double, [_D, C.c_int]),
            "orc_mp5_left": (C.c_double, [_D]),
            "orc_wenoz_left": (C.c_double, [_D]),
            "orc_mc2_left": (C.c_double, [_D]),
            "orc_ppm_left": (C.c_double, [_D]),
            "orc_der": (C.c_double, [_D, C.c_int]),
            "orc_charrec_face_pt": (C.c_int, [P, _D, C.c_int, _D, _D]),
            "orc_c2p_pt": (C.c_int, [P, _D, _D, _D, _D, C.POINTER(C.c_int)]),
            "orc_set_prims": (C.c_int, [P, _D, _D, _D, _LL]),
            "orc_get_prims": (C.c_int, [P, _D, _D, _D]),
            "orc_rhs": (C.c_int, [P, _D, _D, _D]),
            "orc_rhs_cells": (C.c_int, [P, _D, _D, C.c_longlong, _LL, _D]),
            "orc_stage": (C.c_int, [P, C.c_int, C.c_double, _D, _D, _D, _D, _D, C.POINTER(_Counts)]),
            "orc_stage_cells": (C.c_int, [P, C.c_int, C.c_double, _D, _D, _D, C.c_longlong, _LL, _D, _D,
                                          C.POINTER(_Counts)]),
            "orc_step": (C.c_int, [P, C.c_double, _D, _D, C.POINTER(_Counts)]),
            "orc_max_dt": (C.c_int, [P, _D, _D, C.c_double, _D]),
            "orc_con2prim": (C.c_int, [P, _D, _D, C.POINTER(_Counts)]),
            "orc_divb": (C.c_double, [P, _D]),
            "orc_uct_centre": (C.c_int, [P, _D, _D]),
            "orc_set_prims_uct": (C.c_int, [P, _D, _D, _D, _D, _LL]),
            "orc_uct_divh": (C.c_int, [P, _D, _D]),
            "orc_rhs_uct": (C.c_int, [P, _D, _D, _D, _D]),
            "orc_stage_uct": (C.c_int, [P, C.c_int, C.c_double, _D, _D, _D, _D, _D, _D, _D, _D,
                                        C.POINTER(_Counts)]),
            "orc_step_uct": (C.c_int, [P, C.c_double, _D, _D, _D, C.POINTER(_Counts)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "need C-contiguous float64"
    return a.ctypes.data_as(_D)


def _v(x, n=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if n is not None:
        assert a.size == n
    return a


# ------------------------------------------------------------ point-wise
def metric(cfg: Cfg, x) -> dict:
    out = np.zeros(23)
    lib().orc_metric(C.byref(cfg.c()), _p(_v(x, 3)), _p(out))
    return {"alpha": out[0], "beta": out[1:4].copy(), "g": out[4:13].reshape(3, 3).copy(),
            "gi": out[13:22].reshape(3, 3).copy(), "sqrtg": out[22]}


def metric_deriv(cfg: Cfg, x) -> dict:
    out = np.zeros(39)
    lib().orc_metric_deriv(C.byref(cfg.c()), _p(_v(x, 3)), _p(out))
    return {"dalpha": out[0:3].copy(), "dbeta": out[3:12].reshape(3, 3).copy(),
            "dg": out[12:39].reshape(3, 3, 3).copy()}


def prim2cons_pt(cfg: Cfg, x, pr) -> np.ndarray:
    out = np.zeros(8)
    lib().orc_prim2cons_pt(C.byref(cfg.c()), _p(_v(x, 3)), _p(_v(pr, 8)), _p(out))
    return out


def flux_pt(cfg: Cfg, x, pr, d: int) -> np.ndarray:
    out = np.zeros(8)
    lib().orc_flux_pt(C.byref(cfg.c()), _p(_v(x, 3)), _p(_v(pr, 8)), d, _p(out))
    return out


def speeds_pt(cfg: Cfg, x, pr, d: int) -> tuple:
    out = np.zeros(2)
    lib().orc_speeds_pt(C.byref(cfg.c()), _p(_v(x, 3)), _p(_v(pr, 8)), d, _p(out))
    return float(out[0]), float(out[1])


def hll_pt(cfg: Cfg, x, pl, pr, d: int) -> np.ndarray:
    out = np.zeros(8)
    lib().orc_hll_pt(C.byref(cfg.c()), _p(_v(x, 3)), _p(_v(pl, 8)), _p(_v(pr, 8)), d, _p(out))
    return out


def sources_pt(cfg: Cfg, x, pr) -> np.ndarray:
    out = np.zeros(8)
    lib().orc_sources_pt(C.byref(cfg.c()), _p(_v(x, 3)), _p(_v(pr, 8)), _p(out))
    return out


def weno5_left(u, rec: int = 0) -> float:
    return float(lib().orc_weno5_left(_p(_v(u, 5)), rec))


def mp5_left(u) -> float:
    return float(lib().orc_mp5_left(_p(_v(u, 5))))


def wenoz_left(u) -> float:
    return float(lib().orc_wenoz_left(_p(_v(u, 5))))


def mc2_left(u) -> float:
    return float(lib().orc_mc2_left(_p(_v(u, 5))))


def ppm_left(u) -> float:
    return float(lib().orc_ppm_left(_p(_v(u, 5))))


def charrec_face(cfg: Cfg, st, a: int):
    """rec = 6 (A44) at one face: st[6][8] prims of cells i-2..i+3 -> (qL, qR) hydro slots 0..4."""
    st = np.ascontiguousarray(np.asarray(st, dtype=np.float64).reshape(6, 8))
    qL, qR = np.zeros(8), np.zeros(8)
    lib().orc_charrec_face_pt(C.byref(cfg.c()), _p(st), int(a), _p(qL), _p(qR))
    return qL[:5].copy(), qR[:5].copy()


def der(F, order: int = 6) -> float:
    return float(lib().orc_der(_p(_v(F, 5)), order))


def c2p_pt(cfg: Cfg, x, u, guess):
    out = np.zeros(8)
    it = C.c_int(0)
    st = lib().orc_c2p_pt(C.byref(cfg.c()), _p(_v(x, 3)), _p(_v(u, 8)), _p(_v(guess, 8)), _p(out), C.byref(it))
    return st, out, it.value


# ------------------------------------------------------------ grid level
class OracleError(RuntimeError):
    pass


def set_prims(cfg: Cfg, P8: np.ndarray):
    """user prims (rho, v^i, p, B^i) -> (U8 densitised, P5 = rho, u~^i, p)."""
    P8 = _v(P8)
    assert P8.shape == cfg.shape(8)
    U8 = np.zeros(cfg.shape(8))
    P5 = np.zeros(cfg.shape(5))
    bad = C.c_longlong(-1)
    rc = lib().orc_set_prims(C.byref(cfg.c()), _p(P8), _p(U8), _p(P5), C.byref(bad))
    if rc:
        raise OracleError(f"unphysical primitive state at linear cell {bad.value}")
    return U8, P5


def get_prims(cfg: Cfg, U8, P5) -> np.ndarray:
    out = np.zeros(cfg.shape(8))
    lib().orc_get_prims(C.byref(cfg.c()), _p(_v(U8)), _p(_v(P5)), _p(out))
    return out


def rhs(cfg: Cfg, U8, P5) -> np.ndarray:
    out = np.zeros(cfg.shape(8))
    rc = lib().orc_rhs(C.byref(cfg.c()), _p(_v(U8)), _p(_v(P5)), _p(out))
    if rc:
        raise OracleError(f"orc_rhs rc={rc}")
    return out


def _idx(cells) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(cells, dtype=np.int64).reshape(-1, 3))


def rhs_cells(cfg: Cfg, U8, P5, cells) -> np.ndarray:
    idx = _idx(cells)
    out = np.zeros((idx.shape[0], 8))
    lib().orc_rhs_cells(C.byref(cfg.c()), _p(_v(U8)), _p(_v(P5)), idx.shape[0], idx.ctypes.data_as(_LL), _p(out))
    return out


def stage(cfg: Cfg, s: int, dt: float, Un, Us, Ps):
    Uo = np.zeros(cfg.shape(8))
    Po = np.zeros(cfg.shape(5))
    cnt = _Counts()
    rc = lib().orc_stage(C.byref(cfg.c()), s, dt, _p(_v(Un)), _p(_v(Us)), _p(_v(Ps)), _p(Uo), _p(Po),
                         C.byref(cnt))
    if rc:
        raise OracleError(f"orc_stage rc={rc}")
    return Uo, Po, (cnt.floor_events, cnt.c2p_failures)


def stage_cells(cfg: Cfg, s: int, dt: float, Un, Us, Ps, cells):
    idx = _idx(cells)
    m = idx.shape[0]
    Uo = np.zeros((m, 8))
    Po = np.zeros((m, 5))
    cnt = _Counts()
    lib().orc_stage_cells(C.byref(cfg.c()), s, dt, _p(_v(Un)), _p(_v(Us)), _p(_v(Ps)), m, idx.ctypes.data_as(_LL),
                          _p(Uo), _p(Po), C.byref(cnt))
    return Uo, Po, (cnt.floor_events, cnt.c2p_failures)


def step(cfg: Cfg, dt: float, U8, P5):
    """one SSP-RK3 step; returns new copies (U8, P5, counts)."""
    U = _v(U8).copy()
    P = _v(P5).copy()
    cnt = _Counts()
    rc = lib().orc_step(C.byref(cfg.c()), dt, _p(U), _p(P), C.byref(cnt))
    if rc:
        raise OracleError(f"orc_step rc={rc}")
    return U, P, (cnt.floor_events, cnt.c2p_failures)


def max_dt(cfg: Cfg, U8, P5, cfl: float) -> float:
    out = C.c_double(0.0)
    rc = lib().orc_max_dt(C.byref(cfg.c()), _p(_v(U8)), _p(_v(P5)), cfl, C.byref(out))
    if rc:
        raise OracleError("static field, dt unbounded")
    return out.value


def con2prim(cfg: Cfg, U8, P5):
    U = _v(U8).copy()
    P = _v(P5).copy()
    cnt = _Counts()
    lib().orc_con2prim(C.byref(cfg.c()), _p(U), _p(P), C.byref(cnt))
    return U, P, (cnt.floor_events, cnt.c2p_failures)


def divb(cfg: Cfg, U8) -> float:
    return float(lib().orc_divb(C.byref(cfg.c()), _p(_v(U8))))


# ---------------------------------------------------- UCT (divb = 2, A37-A41)
def uct_centre(cfg: Cfg, b3) -> np.ndarray:
    """cell-centred field I6(b3) (A37), [3][n3][n2][n1]"""
    out = np.zeros(cfg.shape(3))
    rc = lib().orc_uct_centre(C.byref(cfg.c()), _p(_v(b3)), _p(out))
    if rc:
        raise OracleError(f"orc_uct_centre rc={rc}")
    return out


def uct_divh(cfg: Cfg, b3) -> np.ndarray:
    """the divergence UCT preserves, sum_a delta_a Dh_a b^a, per cell (A41)"""
    out = np.zeros(cfg.shape(1))[0]
    lib().orc_uct_divh(C.byref(cfg.c()), _p(_v(b3)), _p(out))
    return out


def set_prims_uct(cfg: Cfg, P8, b3):
    """state of a UCT run: the hydro primitives of P8 and the staggered field b3 (the
    cell-centred sqrt(gamma) B of the state is I6(b3); P8's B slots are ignored)."""
    P8 = _v(P8)
    b = _v(b3).copy()
    U8 = np.zeros(cfg.shape(8))
    P5 = np.zeros(cfg.shape(5))
    bad = C.c_longlong(-1)
    rc = lib().orc_set_prims_uct(C.byref(cfg.c()), _p(P8), _p(b), _p(U8), _p(P5), C.byref(bad))
    if rc:
        raise OracleError(f"orc_set_prims_uct rc={rc} (cell {bad.value})")
    return U8, P5, b


def rhs_uct(cfg: Cfg, U8, P5, b3) -> np.ndarray:
    out = np.zeros(cfg.shape(8))
    rc = lib().orc_rhs_uct(C.byref(cfg.c()), _p(_v(U8)), _p(_v(P5)), _p(_v(b3)), _p(out))
    if rc:
        raise OracleError(f"orc_rhs_uct rc={rc}")
    return out


def stage_uct(cfg: Cfg, s: int, dt: float, Un, Us, Ps, bn, bs):
    Uo = np.zeros(cfg.shape(8))
    Po = np.zeros(cfg.shape(5))
    bo = np.zeros(cfg.shape(3))
    cnt = _Counts()
    rc = lib().orc_stage_uct(C.byref(cfg.c()), s, dt, _p(_v(Un)), _p(_v(Us)), _p(_v(Ps)), _p(_v(bn)), _p(_v(bs)),
                             _p(Uo), _p(Po), _p(bo), C.byref(cnt))
    if rc:
        raise OracleError(f"orc_stage_uct rc={rc}")
    return Uo, Po, bo, (cnt.floor_events, cnt.c2p_failures)


def step_uct(cfg: Cfg, dt: float, U8, P5, b3):
    """one SSP-RK3 step with the staggered field; returns new copies (U8, P5, b3, counts)."""
    U = _v(U8).copy()
    P = _v(P5).copy()
    b = _v(b3).copy()
    cnt = _Counts()
    rc = lib().orc_step_uct(C.byref(cfg.c()), dt, _p(U), _p(P), _p(b), C.byref(cnt))
    if rc:
        raise OracleError(f"orc_step_uct rc={rc}")
    return U, P, b, (cnt.floor_events, cnt.c2p_failures)
