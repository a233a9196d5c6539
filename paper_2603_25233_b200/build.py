"""Builds the sm_100a shared library paper_2603_25233_b200/lib/librtlr_cu.so.

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU
container too.  Explicit -gencode arch=compute_100a,code=sm_100a (plain
-arch=sm_100a would also emit a generic compute_100 PTX image that ptxas
rejects for arch-specific instructions).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
OBJ_DIR = os.path.join(PKG, "lib", "obj")
LIB = os.path.join(LIB_DIR, "librtlr_cu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-lineinfo", "-I", CSRC,
          "-I", os.path.join(os.path.dirname(PKG), "include")]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers_mtime():
    ts = [os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    ts.append(os.path.getmtime(os.path.join(os.path.dirname(PKG), "include", "rtlr_cu.h")))
    return max(ts)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ_DIR, src + ".o")
    srcp = os.path.join(CSRC, src)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(srcp), _headers_mtime()):
        return obj
    cmd = [NVCC, *GENCODE, *COMMON, "-c", srcp, "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose else []
    else:
        cmd += ["-x", "cu"] if False else []
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    return obj


def _nccl_link():
    """Link the NCCL that torch itself loads (the venv's nvidia-nccl wheel)
    when present: a process that loads this library before `import torch`
    would otherwise bind the older system libnccl.so.2 first and torch's
    libtorch_cuda.so then fails on symbols only the newer NCCL exports."""
    try:
        import nvidia.nccl  # type: ignore
        for root in nvidia.nccl.__path__:
            d = os.path.join(root, "lib")
            if os.path.exists(os.path.join(d, "libnccl.so.2")):
                return ["-L" + d, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + d]
    except ImportError:
        pass
    return ["-L/usr/lib/x86_64-linux-gnu", "-lnccl"]


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), _sources()))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC, *GENCODE, "-shared", "-o", LIB, *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread",
               *_nccl_link()]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    _build_cli()
    _build_facade_test()
    return LIB


CLI_SRC = os.path.join(PKG, "cli", "rtlr_cu_bench.cpp")
CLI = os.path.join(LIB_DIR, "rtlr_cu_bench")


def _build_cli():
    """The rtlr_bench driver (C ABI only) next to the library it links."""
    if os.path.exists(CLI) and os.path.getmtime(CLI) >= max(os.path.getmtime(CLI_SRC), os.path.getmtime(LIB)):
        return
    nccl = [a for a in _nccl_link() if a.startswith("-L")]
    cmd = ["g++", "-O2", "-std=c++17", "-I", os.path.join(os.path.dirname(PKG), "include"), CLI_SRC, "-o", CLI,
           "-L" + LIB_DIR, "-lrtlr_cu", "-Wl,-rpath,$ORIGIN"] + ["-Wl,-rpath-link," + a[2:] for a in nccl]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"cli build failed:\n{r.stdout}\n{r.stderr}")


FACADE_SRC = os.path.join(os.path.dirname(PKG), "tests", "cpp", "facade_test.cpp")
FACADE = os.path.join(LIB_DIR, "rtlr_cu_facade_test")


def _build_facade_test():
    """The C++ consumer of include/rtlr_cu.hpp (the rtlr::cuda façade), built
    against the header and the library only (tests/cpp/facade_test.cpp)."""
    hdrs = [os.path.join(os.path.dirname(PKG), "include", f) for f in ("rtlr_cu.h", "rtlr_cu.hpp")]
    if os.path.exists(FACADE) and os.path.getmtime(FACADE) >= max(os.path.getmtime(p) for p in
                                                                  [FACADE_SRC, LIB] + hdrs):
        return
    nccl = [a for a in _nccl_link() if a.startswith("-L")]
    cmd = ["g++", "-O2", "-std=c++17", "-Wall", "-Wextra", "-I", os.path.join(os.path.dirname(PKG), "include"),
           FACADE_SRC, "-o", FACADE, "-L" + LIB_DIR, "-lrtlr_cu", "-Wl,-rpath,$ORIGIN"] + \
          ["-Wl,-rpath-link," + a[2:] for a in nccl]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"facade test build failed:\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
