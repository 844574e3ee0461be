"""Build libpipo.so in-tree: nvcc for sm_100a (no fast-math: the quantizer's IEEE
division / RNE rounding is part of the bit-exact contract) + g++ for host C++.

    python -m paper_2504_03664_b200.build          # or __graft_entry__.build()
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libpipo.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
                     "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills", f"-I{ROOT}/include"]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-pthread", f"-I{ROOT}/include",
             "-I/usr/local/cuda/include", "-fno-fast-math", "-ffp-contract=off"]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers_digest():
    h = hashlib.sha256()
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".h", ".cuh")):
            h.update(open(os.path.join(CSRC, f), "rb").read())
    h.update(open(os.path.join(ROOT, "include", "pipo.h"), "rb").read())
    return h.hexdigest()[:16]


def _compile(src: str, digest: str, verbose: bool) -> str:
    path = os.path.join(CSRC, src)
    key = hashlib.sha256(open(path, "rb").read() + digest.encode()).hexdigest()[:16]
    obj = os.path.join(OBJ, f"{src}.{key}.o")
    if os.path.exists(obj):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC, *NVCC_FLAGS, "-c", path, "-o", obj]
    else:
        cmd = ["g++", *CXX_FLAGS, "-c", path, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    digest = _headers_digest()
    with ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1))) as ex:
        objs = list(ex.map(lambda s: _compile(s, digest, verbose), _sources()))
    stamp = hashlib.sha256("".join(objs).encode()).hexdigest()[:16]
    stamp_file = LIB + ".stamp"
    if os.path.exists(LIB) and os.path.exists(stamp_file) and open(stamp_file).read() == stamp:
        return LIB
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lpthread", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    open(stamp_file, "w").write(stamp)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
