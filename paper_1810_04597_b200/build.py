"""Build libecho_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1810_04597_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import concurrent.futures as cf
import fcntl
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libecho_b200.so")
SOURCES = ["march.cu", "fused.cu", "update.cu", "uct.cu", "api.cu", "metric_tables.cpp"]
HEADERS = ["echo_dev.cuh", "echo_kernels.h", "metric_tables.h", "cell_physics.cuh", "march_impl.cuh", "march_pair.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _includes(path: str, seen: set) -> None:
    """the csrc headers `path` includes, recursively (quoted includes only)"""
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line.startswith("#include \""):
                h = line.split("\"")[1]
                hp = os.path.join(CSRC, h)
                if h in HEADERS and hp not in seen:
                    seen.add(hp)
                    _includes(hp, seen)


def _compile(src: str, verbose: bool, build_dir: str = BUILD, defines: tuple = ()) -> str:
    obj = os.path.join(build_dir, os.path.basename(src) + ".o")
    hdrs: set = set()
    _includes(os.path.join(CSRC, src), hdrs)
    deps = [os.path.join(CSRC, src)] + sorted(hdrs) + [os.path.join(ROOT, "include", "echo.h")]
    if not _stale(obj, deps):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *defines, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(build_dir, os.path.basename(src) + ".ptxas.log")
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
    if verbose:
        print(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, variant: str = "", defines: tuple = ()) -> str:
    """Build libecho_b200.so; a named `variant` (tuning runs only) builds
    libecho_b200_<variant>.so with extra -D `defines` in its own object dir."""
    build_dir = BUILD if not variant else BUILD + "_" + variant
    lib = LIB if not variant else LIB.replace(".so", f"_{variant}.so")
    # The object dir is not shipped to the GPU boxes (.gpurunignore): a library newer than
    # every source and header is current without its objects, so no rank recompiles it.
    if not force and not variant and not _stale(lib, _all_deps()):
        return lib
    os.makedirs(build_dir, exist_ok=True)
    # one builder at a time: torchrun starts N ranks that all call build() (bench.py)
    with open(os.path.join(build_dir, ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if force:
            for f in os.listdir(build_dir):
                if f != ".lock":
                    os.remove(os.path.join(build_dir, f))
        with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
            objs = list(ex.map(lambda s: _compile(s, verbose, build_dir, tuple(defines)), SOURCES))
        if _stale(lib, objs):
            tmp = lib + f".tmp{os.getpid()}"
            cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
            os.replace(tmp, lib)
    return lib


def _all_deps() -> list[str]:
    return ([os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
            + [os.path.join(ROOT, "include", "echo.h")])


if __name__ == "__main__":
    # python -m paper_1810_04597_b200.build [--force] [--verbose] [--variant NAME -DX=Y ...]
    var = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else ""
    defs = tuple(a for a in sys.argv if a.startswith("-D"))
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, variant=var, defines=defs))
