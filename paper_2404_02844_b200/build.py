"""Build libqdt.so (the C-ABI library, include/qdt.h) in-tree with nvcc for sm_100a.

Each .cu is compiled to an object in parallel (the kernel templates dominate the build time),
then nvcc links the shared library.  ptxas register / spill reports go to build_ptxas.log.
"""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libqdt.so")
SRCS = [os.path.join(HERE, "csrc", f) for f in ("qdt_api.cu", "qdt_kernels.cu", "qdt_sweep.cu", "qdt_newton.cu",
                                                            "qdt_wide.cu", "qdt_small.cu", "qdt_coop.cu")]
DEPS = SRCS + glob.glob(os.path.join(HERE, "csrc", "*.h")) + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "qdt.h"),
                                                              os.path.abspath(__file__)]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
         "-Xptxas", "-v"]


def nvcc_cmd(out: str = LIB, extra=()):
    """Single-shot command (documentation / tests): every source, one nvcc invocation."""
    return [NVCC, *ARCH, *FLAGS, "-shared", *extra, "-o", out, *SRCS, "-ldl"]


def _obj(src: str) -> str:
    return os.path.join(HERE, "build", os.path.basename(src).replace(".cu", ".o"))


def _compile(src: str):
    obj = _obj(src)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(
            os.path.getmtime(d) for d in DEPS if d == src or not d.endswith(".cu")):
        return src, 0, ""
    tmp = obj + f".tmp{os.getpid()}"
    r = subprocess.run([NVCC, *ARCH, *FLAGS, "-c", src, "-o", tmp], capture_output=True, text=True)
    if r.returncode == 0:
        os.replace(tmp, obj)
    return src, r.returncode, r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return LIB
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    if force:
        for s in SRCS:
            if os.path.exists(_obj(s)):
                os.remove(_obj(s))
    with ThreadPoolExecutor(len(SRCS)) as ex:
        res = list(ex.map(_compile, SRCS))
    log = os.path.join(HERE, "build_ptxas.log")
    with open(log, "w") as f:
        for src, rc, out in res:
            f.write(f"==== {os.path.basename(src)} rc={rc}\n{out}\n")
    bad = [(s, out) for s, rc, out in res if rc != 0]
    if bad:
        raise RuntimeError("nvcc failed:\n" + "\n".join(f"{s}:\n{o[-6000:]}" for s, o in bad))
    tmp = LIB + f".tmp{os.getpid()}"
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *[_obj(s) for s in SRCS], "-ldl"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + r.stderr[-6000:])
    os.replace(tmp, LIB)
    if verbose:
        print(open(log).read()[-3000:])
    return LIB


def build_variant(tag: str, defines, src: str = "qdt_sweep.cu") -> str:
    """A/B build: `src` recompiled with extra -D flags, linked with the main objects into
    libqdt_<tag>.so (load it with QDT_LIB=<path>)."""
    build()
    out_dir = os.path.join(HERE, "build_" + tag)
    os.makedirs(out_dir, exist_ok=True)
    s = os.path.join(HERE, "csrc", src)
    obj = os.path.join(out_dir, src.replace(".cu", ".o"))
    r = subprocess.run([NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", s, "-o", obj],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-6000:])
    with open(os.path.join(out_dir, "ptxas.log"), "w") as f:
        f.write(r.stdout + r.stderr)
    objs = [obj if os.path.basename(x) == src else _obj(x) for x in SRCS]
    lib = os.path.join(HERE, f"libqdt_{tag}.so")
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", lib, *objs, "-ldl"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-6000:])
    return lib


if __name__ == "__main__":
    build(force=True, verbose=True)
