"""Build libcycb200.so in-tree for sm_100a (nvcc; no torch, no JIT cache).

    python -m paper_2405_16911_b200.build [--force]

The library is the product: the C-ABI of include/cycb200.h over the CUDA
kernels in csrc/.  It is written next to this file so it travels to the GPU
box with the repository snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libcycb200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# CYC_NVCC_EXTRA (diagnostic builds: traces, ablations) never touches the
# product library: its objects and library go to a directory keyed by a hash of
# the extra flags, loaded with CYC_LIB=<that path>.
EXTRA = os.environ.get("CYC_NVCC_EXTRA", "").split()
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include"),
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"] + EXTRA
if EXTRA:
    import hashlib
    _tag = hashlib.sha1(" ".join(EXTRA).encode()).hexdigest()[:10]
    BUILD = os.path.join(HERE, "_diag", _tag)
    LIB = os.path.join(BUILD, "libcycb200.so")
    FLAGS += ["-DTC_DIAG_BUILD"]


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def headers() -> list[str]:
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs.append(os.path.join(ROOT, "include", "cycb200.h"))
    return hs


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    newest_dep = max([os.path.getmtime(src), os.path.getmtime(__file__)] + [os.path.getmtime(h) for h in headers()])
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-x", "cu" if src.endswith(".cu") else "c++", "-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, *FLAGS, "-x", "c++", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if "spill" in r.stderr and "0 bytes spill" not in r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def build_tools(force: bool = False) -> str:
    """tools/stream_bench: the C++ streaming driver bench.py uses for C1/C3."""
    lib = build(force)
    src = os.path.join(ROOT, "tools", "stream_bench.cpp")
    exe = os.path.join(ROOT, "tools", "stream_bench")
    if force or not os.path.exists(exe) or os.path.getmtime(exe) < max(os.path.getmtime(src), os.path.getmtime(lib)):
        cmd = [NVCC, "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-x", "c++", src, "-o", exe,
               f"-L{HERE}", "-lcycb200", "-Xlinker", f"-rpath,{HERE}"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"stream_bench build failed:\n{r.stdout}\n{r.stderr}")
    return exe


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
    if not EXTRA:
        print(build_tools())
