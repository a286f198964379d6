"""CPU-side checks of the boundary: the C-ABI library builds, loads without a
GPU, and exports every symbol include/echo.h declares (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "echo.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(echo_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1810_04597_b200 import build

    return build.build()


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for name in ("echo_create", "echo_set_prims", "echo_rhs", "echo_con2prim", "echo_step", "echo_max_dt",
                 "echo_get_prims"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (echo_[a-z0-9_]+)\b", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_without_gpu(lib_path):
    lib = ctypes.CDLL(lib_path)
    for s in declared_symbols():
        assert hasattr(lib, s)
    lib.echo_kernel_classes.restype = ctypes.c_int
    assert lib.echo_kernel_classes() == 16
    lib.echo_kernel_name.restype = ctypes.c_char_p
    assert lib.echo_kernel_name(0) == b"sweep_x"


def test_binding_names_match_header(lib_path):
    from paper_1810_04597_b200 import echo

    assert sorted(echo.EXPORTED) == declared_symbols()
    for s in declared_symbols():
        assert callable(getattr(echo, s[len("echo_"):]))


def test_sass_is_sm100a(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1810_04597_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.h" not in txt, f


def build_c_demo(lib_path, out_dir):
    """examples/echo_c_demo.c against include/echo.h as plain C99 (-Wall -Wextra -Werror), linked
    to the library: the boundary needs no CUDA header, C++ or Python"""
    exe = os.path.join(out_dir, "echo_c_demo")
    libdir = os.path.dirname(lib_path)
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "echo_c_demo.c"), "-L" + libdir, "-lecho_b200",
           "-Wl,-rpath," + libdir, "-lm", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_demo_builds_and_reports_no_device(lib_path, tmp_path):
    import torch

    exe = build_c_demo(lib_path, str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    if torch.cuda.is_available():  # (the GPU run of the same program: tests/test_gpu_c_demo.py)
        assert r.returncode == 0, r.stdout + r.stderr
    else:  # echo_create -> ECHO_E_CUDA, named; the demo's "skipped" exit
        assert r.returncode == 77, r.stdout + r.stderr
        assert "no CUDA device" in r.stdout


def test_current_library_needs_no_objects(lib_path, tmp_path, monkeypatch):
    """A library newer than every source is current without its object dir (which does not travel
    to the GPU boxes, .gpurunignore): build() must not recompile it on every box and rank."""
    import time

    from paper_1810_04597_b200 import build

    monkeypatch.setattr(build, "BUILD", str(tmp_path / "no_objects"))
    t = time.time()
    assert build.build() == lib_path
    assert time.time() - t < 5.0
    assert not (tmp_path / "no_objects").exists()
