"""Thin ctypes binding of include/echo.h (argument marshalling only).

Every function has the C name without the ``echo_`` prefix; every step of the
path runs in the sm_100a kernels of libecho_b200.so.  There is no fallback:
if the library is missing or fails to load, importing this module raises.

Buffers: numpy float64 C-contiguous arrays are host buffers (``on_device=0``);
torch CUDA float64 contiguous tensors are device buffers (``on_device=1``,
stream-ordered on the context stream).  Layouts are those of echo.h.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ECHO_LIB_VARIANT=<name> loads libecho_b200_<name>.so (a tuning build, build.py --variant)
_VAR = os.environ.get("ECHO_LIB_VARIANT", "")
LIB_PATH = os.path.join(HERE, "libecho_b200.so" if not _VAR else f"libecho_b200_{_VAR}.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1810_04597_b200.build` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

OK, E_ARG, E_CUDA, E_OOM, E_ORDER, E_UNPHYSICAL, E_NONFINITE = 0, -1, -2, -3, -4, -5, -6
DEBUG_NANSCAN = 1
BC_PERIODIC, BC_OUTFLOW, BC_HALO = 0, 1, 2
HALO_PLANES = 6
METRIC_MINKOWSKI, METRIC_KERR_SCHILD = 0, 1


class Grid(C.Structure):
    _fields_ = [("n", C.c_int * 3), ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("bc", (C.c_int * 2) * 3),
                ("rec", C.c_int), ("der", C.c_int), ("divb", C.c_int), ("der_jump", C.c_double), ("dz", C.c_double)]


class Metric(C.Structure):
    _fields_ = [("kind", C.c_int), ("M", C.c_double), ("a", C.c_double)]


class Eos(C.Structure):
    _fields_ = [("gamma", C.c_double), ("rho_floor", C.c_double), ("p_floor", C.c_double), ("w_max", C.c_double),
                ("c2p_max_iter", C.c_int), ("c2p_tol", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("floor_events", C.c_ulonglong), ("c2p_failures", C.c_ulonglong), ("steps", C.c_ulonglong),
                ("stages", C.c_ulonglong)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_sig = {
    "echo_create": (C.c_int, [C.POINTER(Grid), C.POINTER(Metric), C.POINTER(Eos), C.POINTER(_P)]),
    "echo_destroy": (None, [_P]),
    "echo_set_stream": (C.c_int, [_P, _P]),
    "echo_set_prims": (C.c_int, [_P, _P, C.c_int]),
    "echo_get_prims": (C.c_int, [_P, _P, C.c_int]),
    "echo_set_cons": (C.c_int, [_P, _P, C.c_int]),
    "echo_set_face_field": (C.c_int, [_P, _P, C.c_int]),
    "echo_get_face_field": (C.c_int, [_P, _P, C.c_int]),
    "echo_get_cons": (C.c_int, [_P, _P, C.c_int]),
    "echo_get_state": (C.c_int, [_P, _P, _P, _P, C.c_int]),
    "echo_rhs": (C.c_int, [_P, _P, C.c_int]),
    "echo_con2prim": (C.c_int, [_P, C.POINTER(Stats)]),
    "echo_stage": (C.c_int, [_P, C.c_int, C.c_double]),
    "echo_step": (C.c_int, [_P, C.c_double]),
    "echo_max_dt": (C.c_int, [_P, C.c_double, _D]),
    "echo_advance": (C.c_int, [_P, C.c_int, C.c_double, _D, C.POINTER(C.c_int)]),
    "echo_stats": (C.c_int, [_P, C.POINTER(Stats)]),
    "echo_last_error": (C.c_char_p, [_P]),
    "echo_profile": (C.c_int, [_P, C.c_int]),
    "echo_profile_read": (C.c_int, [_P, C.c_int, _D, C.POINTER(C.c_longlong)]),
    "echo_kernel_classes": (C.c_int, []),
    "echo_kernel_name": (C.c_char_p, [C.c_int]),
    "echo_launch_count": (C.c_longlong, [_P]),
    "echo_halo_doubles": (C.c_longlong, [_P]),
    "echo_halo_link": (C.c_int, [_P, C.c_int, _P]),
    "echo_ipc_export": (C.c_int, [_P, _P, C.POINTER(C.c_int)]),
    "echo_halo_link_ipc": (C.c_int, [_P, C.c_int, _P, C.c_int]),
    "echo_halo_pull": (C.c_int, [_P, C.c_int]),
    "echo_stage_sweeps": (C.c_int, [_P, C.c_int]),
    "echo_stage_update": (C.c_int, [_P, C.c_int, C.c_double]),
    "echo_stage_sweeps_interior": (C.c_int, [_P, C.c_int]),
    "echo_stage_update_field": (C.c_int, [_P, C.c_int, C.c_double]),
    "echo_stage_update_cells": (C.c_int, [_P, C.c_int, C.c_double]),
    "echo_halo_field_doubles": (C.c_longlong, [_P]),
    "echo_halo_export_field": (C.c_int, [_P, C.c_int, _P, C.c_int]),
    "echo_halo_import_field": (C.c_int, [_P, C.c_int, _P, C.c_int]),
    "echo_halo_fill_field": (C.c_int, [_P, C.c_int]),
    "echo_stage_sweeps_boundary": (C.c_int, [_P, C.c_int]),
    "echo_halo_export": (C.c_int, [_P, C.c_int, _P, C.c_int]),
    "echo_halo_import": (C.c_int, [_P, C.c_int, _P, C.c_int]),
    "echo_halo_fill": (C.c_int, [_P, C.c_int]),
    "echo_set_debug": (C.c_int, [_P, C.c_int]),
    "echo_check_finite": (C.c_int, [_P]),
    "echo_check_guards": (C.c_int, [_P]),
    "echo_checkpoint_doubles": (C.c_longlong, [_P]),
    "echo_checkpoint_save": (C.c_int, [_P, _P, C.c_int]),
    "echo_checkpoint_load": (C.c_int, [_P, _P, C.c_int]),
}
for _n, (_r, _a) in _sig.items():
    _f = getattr(_lib, _n)
    _f.restype = _r
    _f.argtypes = _a

EXPORTED = tuple(_sig)


class EchoError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(ctx, rc: int):
    if rc != OK:
        raise EchoError(rc, last_error(ctx))
    return rc


def _buf(a, writable=False):
    """(pointer, on_device) of a numpy array (host) or a torch CUDA tensor (device)."""
    if isinstance(a, np.ndarray):
        assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "need C-contiguous float64"
        if writable:
            assert a.flags["WRITEABLE"]
        return a.ctypes.data, 0
    # torch tensor
    assert a.dtype.is_floating_point and a.element_size() == 8 and a.is_contiguous(), "need contiguous float64"
    assert a.is_cuda, "torch tensors must be on the GPU"
    return a.data_ptr(), 1


def _grid(n, lo, hi, bc, rec=0, der=6, divb=0, der_jump=0.5, dz=0.0) -> Grid:
    g = Grid()
    for i in range(3):
        g.n[i] = int(n[i])
        g.lo[i] = float(lo[i])
        g.hi[i] = float(hi[i])
        g.bc[i][0] = int(bc[i][0])
        g.bc[i][1] = int(bc[i][1])
    g.rec, g.der, g.divb = int(rec), int(der), int(divb)
    g.der_jump = float(der_jump)
    g.dz = float(dz)
    return g


# ------------------------------------------------------------- C names
def create(n, lo, hi, bc, metric=METRIC_MINKOWSKI, M=1.0, a=0.0, gamma=4.0 / 3.0, rho_floor=1e-8, p_floor=1e-10,
           w_max=50.0, c2p_max_iter=30, c2p_tol=1e-13, rec=0, der=6, divb=0, der_jump=0.5, dz=0.0):
    g = _grid(n, lo, hi, bc, rec, der, divb, der_jump, dz)
    m = Metric(int(metric), float(M), float(a))
    e = Eos(float(gamma), float(rho_floor), float(p_floor), float(w_max), int(c2p_max_iter), float(c2p_tol))
    out = _P()
    rc = _lib.echo_create(C.byref(g), C.byref(m), C.byref(e), C.byref(out))
    if rc != OK:
        raise EchoError(rc, _lib.echo_last_error(None).decode())
    return out


def destroy(ctx):
    _lib.echo_destroy(ctx)


def set_stream(ctx, stream_handle: int):
    return _check(ctx, _lib.echo_set_stream(ctx, _P(stream_handle)))


def set_prims(ctx, p8):
    p, d = _buf(p8)
    return _check(ctx, _lib.echo_set_prims(ctx, p, d))


def get_prims(ctx, out8):
    p, d = _buf(out8, True)
    return _check(ctx, _lib.echo_get_prims(ctx, p, d))


def set_cons(ctx, u8):
    p, d = _buf(u8)
    return _check(ctx, _lib.echo_set_cons(ctx, p, d))


def set_face_field(ctx, b3):
    """divb = 2 (UCT): the staggered field sqrt(gamma) B^a at the faces i_a + 1/2, [3][n3][n2][n1]"""
    p, d = _buf(b3)
    return _check(ctx, _lib.echo_set_face_field(ctx, p, d))


def get_face_field(ctx, out3):
    p, d = _buf(out3, True)
    return _check(ctx, _lib.echo_get_face_field(ctx, p, d))


def get_cons(ctx, out8):
    p, d = _buf(out8, True)
    return _check(ctx, _lib.echo_get_cons(ctx, p, d))


def get_state(ctx, un8=None, us8=None, p5=None):
    ptrs, dev = [], 0
    for a in (un8, us8, p5):
        if a is None:
            ptrs.append(None)
        else:
            p, dev = _buf(a, True)
            ptrs.append(p)
    return _check(ctx, _lib.echo_get_state(ctx, *ptrs, dev))


def rhs(ctx, out8):
    p, d = _buf(out8, True)
    return _check(ctx, _lib.echo_rhs(ctx, p, d))


def con2prim(ctx):
    s = Stats()
    _check(ctx, _lib.echo_con2prim(ctx, C.byref(s)))
    return s.floor_events, s.c2p_failures


def stage(ctx, s: int, dt: float):
    return _check(ctx, _lib.echo_stage(ctx, int(s), float(dt)))


def step(ctx, dt: float):
    return _check(ctx, _lib.echo_step(ctx, float(dt)))


def max_dt(ctx, cfl: float) -> float:
    out = C.c_double(0.0)
    _check(ctx, _lib.echo_max_dt(ctx, float(cfl), C.byref(out)))
    return out.value


def advance(ctx, nsteps: int, cfl: float, log: bool = True):
    """nsteps x (max_dt + step) with dt computed on the device (one CUDA-graph replay per
    step, one synchronisation): returns the dt of every step (numpy) or None."""
    buf = np.zeros(max(int(nsteps), 1), np.float64) if log else None
    done = C.c_int(0)
    ptr = buf.ctypes.data_as(_D) if log else None
    _check(ctx, _lib.echo_advance(ctx, int(nsteps), float(cfl), ptr, C.byref(done)))
    return buf[: done.value] if log else None


def stats(ctx) -> dict:
    s = Stats()
    _check(ctx, _lib.echo_stats(ctx, C.byref(s)))
    return {"floor_events": s.floor_events, "c2p_failures": s.c2p_failures, "steps": s.steps, "stages": s.stages}


def last_error(ctx) -> str:
    return _lib.echo_last_error(ctx).decode()


def profile(ctx, enable: bool):
    return _check(ctx, _lib.echo_profile(ctx, int(bool(enable))))


def profile_read(ctx) -> dict:
    out = {}
    for i in range(_lib.echo_kernel_classes()):
        ms = C.c_double(0.0)
        n = C.c_longlong(0)
        _check(ctx, _lib.echo_profile_read(ctx, i, C.byref(ms), C.byref(n)))
        out[_lib.echo_kernel_name(i).decode()] = (ms.value, n.value)
    return out


def kernel_classes() -> int:
    return _lib.echo_kernel_classes()


def kernel_name(i: int) -> str:
    return _lib.echo_kernel_name(i).decode()


def set_debug(ctx, flags: int):
    return _check(ctx, _lib.echo_set_debug(ctx, int(flags)))


def check_finite(ctx):
    return _check(ctx, _lib.echo_check_finite(ctx))


def check_guards(ctx):
    return _check(ctx, _lib.echo_check_guards(ctx))


def launch_count(ctx) -> int:
    return int(_lib.echo_launch_count(ctx))


def halo_link(ctx, side: int, peer):
    return _check(ctx, _lib.echo_halo_link(ctx, int(side), peer))


def ipc_export(ctx):
    """(bytes of the 3 CUDA IPC handles of P, Un, Us, n[2]) of a slab context."""
    buf = C.create_string_buffer(3 * 64)
    nz = C.c_int(0)
    _check(ctx, _lib.echo_ipc_export(ctx, buf, C.byref(nz)))
    return buf.raw, nz.value


def halo_link_ipc(ctx, side: int, handles, peer_nz: int):
    if handles is None:
        return _check(ctx, _lib.echo_halo_link_ipc(ctx, int(side), None, 0))
    buf = C.create_string_buffer(bytes(handles), len(handles))
    return _check(ctx, _lib.echo_halo_link_ipc(ctx, int(side), buf, int(peer_nz)))


def halo_pull(ctx, side: int):
    return _check(ctx, _lib.echo_halo_pull(ctx, int(side)))


def stage_sweeps(ctx, s: int):
    return _check(ctx, _lib.echo_stage_sweeps(ctx, int(s)))


def stage_update(ctx, s: int, dt: float):
    return _check(ctx, _lib.echo_stage_update(ctx, int(s), float(dt)))


def stage_update_field(ctx, s: int, dt: float):
    return _check(ctx, _lib.echo_stage_update_field(ctx, int(s), float(dt)))


def stage_update_cells(ctx, s: int, dt: float):
    return _check(ctx, _lib.echo_stage_update_cells(ctx, int(s), float(dt)))


def halo_field_doubles(ctx) -> int:
    return int(_lib.echo_halo_field_doubles(ctx))


def halo_export_field(ctx, side: int, buf):
    p, d = _buf(buf, True)
    return _check(ctx, _lib.echo_halo_export_field(ctx, int(side), p, d))


def halo_import_field(ctx, side: int, buf):
    p, d = _buf(buf)
    return _check(ctx, _lib.echo_halo_import_field(ctx, int(side), p, d))


def halo_fill_field(ctx, side: int):
    return _check(ctx, _lib.echo_halo_fill_field(ctx, int(side)))


def stage_sweeps_interior(ctx, s: int):
    return _check(ctx, _lib.echo_stage_sweeps_interior(ctx, int(s)))


def stage_sweeps_boundary(ctx, s: int):
    return _check(ctx, _lib.echo_stage_sweeps_boundary(ctx, int(s)))


def halo_doubles(ctx) -> int:
    return int(_lib.echo_halo_doubles(ctx))


def halo_export(ctx, side: int, buf):
    p, d = _buf(buf, True)
    return _check(ctx, _lib.echo_halo_export(ctx, int(side), p, d))


def halo_import(ctx, side: int, buf):
    p, d = _buf(buf)
    return _check(ctx, _lib.echo_halo_import(ctx, int(side), p, d))


def halo_fill(ctx, side: int):
    return _check(ctx, _lib.echo_halo_fill(ctx, int(side)))


def checkpoint_doubles(ctx) -> int:
    return int(_lib.echo_checkpoint_doubles(ctx))


def checkpoint_save(ctx, buf):
    p, d = _buf(buf, True)
    return _check(ctx, _lib.echo_checkpoint_save(ctx, p, d))


def checkpoint_load(ctx, buf):
    p, d = _buf(buf)
    return _check(ctx, _lib.echo_checkpoint_load(ctx, p, d))


# ------------------------------------------------------- convenience
class Echo:
    """Owns one context; `problem` is an echo_inputs.Problem (or anything with grid_kwargs())."""

    def __init__(self, problem=None, **kw):
        args = dict(problem.grid_kwargs()) if problem is not None else {}
        args.update(kw)
        self.n = tuple(args["n"])
        self.N = self.n[0] * self.n[1] * self.n[2]
        self.ctx = create(**args)
        try:
            import torch  # device memory and streams are torch's (plumbing only)
            if torch.cuda.is_available():
                set_stream(self.ctx, torch.cuda.current_stream().cuda_stream)
        except ImportError:
            pass

    def close(self):
        if self.ctx:
            destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shape(self, nvar):
        return (nvar, self.n[2], self.n[1], self.n[0])

    def set_prims(self, p8):
        return set_prims(self.ctx, p8)

    def get_prims(self, out=None):
        out = np.zeros(self.shape(8)) if out is None else out
        get_prims(self.ctx, out)
        return out

    def set_face_field(self, b3):
        return set_face_field(self.ctx, b3)

    def get_face_field(self, out=None):
        out = np.zeros(self.shape(3)) if out is None else out
        get_face_field(self.ctx, out)
        return out

    def get_cons(self, out=None):
        out = np.zeros(self.shape(8)) if out is None else out
        get_cons(self.ctx, out)
        return out

    def get_state(self):
        un, us, p = np.zeros(self.shape(8)), np.zeros(self.shape(8)), np.zeros(self.shape(5))
        get_state(self.ctx, un, us, p)
        return un, us, p

    def rhs(self, out=None):
        out = np.zeros(self.shape(8)) if out is None else out
        rhs(self.ctx, out)
        return out

    def stage(self, s, dt):
        return stage(self.ctx, s, dt)

    def step(self, dt):
        return step(self.ctx, dt)

    def max_dt(self, cfl):
        return max_dt(self.ctx, cfl)

    def advance(self, nsteps, cfl, log=True):
        return advance(self.ctx, nsteps, cfl, log)

    def con2prim(self):
        return con2prim(self.ctx)

    def stats(self):
        return stats(self.ctx)

    def set_debug(self, flags=DEBUG_NANSCAN):
        return set_debug(self.ctx, flags)

    def check_finite(self):
        return check_finite(self.ctx)

    def check_guards(self):
        return check_guards(self.ctx)

    def checkpoint(self, out=None):
        """the raw state at a step boundary (echo_checkpoint_save): a host array, or `out`"""
        out = np.zeros(checkpoint_doubles(self.ctx)) if out is None else out
        checkpoint_save(self.ctx, out)
        return out

    def restore(self, buf):
        """continue bit for bit from a checkpoint of a context with the same configuration"""
        return checkpoint_load(self.ctx, buf)
