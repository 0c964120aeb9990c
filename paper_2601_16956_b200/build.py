"""Builds libts_b200.so (the C-ABI + sm_100a kernels) in-tree with nvcc.

    python -m paper_2601_16956_b200.build

Sources: paper_2601_16956_b200/csrc/*.{cu,cpp}. Every translation unit goes
through nvcc with `-gencode arch=compute_100a,code=sm_100a -lineinfo`; the
runtime is linked statically so the library carries no torch dependency.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libts_b200.so")
BUILD = os.path.join(os.path.dirname(HERE), "build", "ts_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3,-pthread,-Wall",
          "-I" + os.path.join(os.path.dirname(HERE), "include")]


PYFAST_SRC = os.path.join(CSRC, "pyfast", "pyfast.cpp")


def pyfast_path() -> str:
    import sysconfig

    return os.path.join(HERE, "_pyfast" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_pyfast() -> str:
    """The Python mirror's CPython fast path (csrc/pyfast): a host-only
    extension linked against libts_b200.so (rpath $ORIGIN/_lib)."""
    import sysconfig

    out = pyfast_path()
    deps = [PYFAST_SRC, LIB, os.path.join(os.path.dirname(HERE), "include", "ts_b200.h")]
    if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps):
        return out
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-shared", "-fPIC", "-Wall",
           "-I" + sysconfig.get_paths()["include"], "-I" + os.path.join(os.path.dirname(HERE), "include"),
           PYFAST_SRC, "-o", out + ".tmp", "-L" + OUT_DIR, "-lts_b200", "-Wl,-rpath,$ORIGIN/_lib"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"pyfast build failed:\n{r.stderr}")
    os.replace(out + ".tmp", out)
    return out


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    deps = [src] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".hpp", ".cuh"))]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "ts_b200.h"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    lang = [] if src.endswith(".cu") else ["-x", "cu"]
    cmd = [NVCC] + ARCH + COMMON + lang + ["-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(OUT_DIR, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), sources()))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB + ".tmp"] + objs + ["-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    build_pyfast()
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
