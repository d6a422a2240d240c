"""Build libpint_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2110_10762_b200.build [--force]

The shared library lands next to this file, so it travels with the repo
snapshot to the GPU box (no JIT cache, no site-packages install).
"""
from __future__ import annotations

import argparse
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libpint_b200.so")
STAMP = LIB + ".srchash"

SOURCES = ["abi.cu", "tri1d.cu", "async_rt.cu", "correct.cu", "stencil.cu", "stencil_wave.cu", "stencil3d.cu", "cg.cu", "spectral.cu", "tc_xform.cu", "mailbox.cu"]
HEADERS = ["pint_internal.cuh", "tri1d_device.cuh", os.path.join("..", "..", "include", "pint_abi.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cand = os.path.join(cuda, "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _sources():
    return [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def source_hash() -> str:
    h = hashlib.sha256()
    for name in _sources() + HEADERS:
        path = os.path.join(CSRC, name)
        if os.path.exists(path):
            with open(path, "rb") as f:
                h.update(name.encode())
                h.update(f.read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def is_fresh() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return False
    with open(STAMP) as f:
        return f.read().strip() == source_hash()


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and is_fresh():
        return LIB
    objs = []
    jobs = []
    for src in _sources():
        obj = os.path.join(CSRC, "_build", src.replace(".cu", ".o"))
        os.makedirs(os.path.dirname(obj), exist_ok=True)
        cmd = [_nvcc()] + [f for f in NVCC_FLAGS if f != "-shared"] + [
            "-c", os.path.join(CSRC, src), "-o", obj]
        jobs.append((src, cmd))
        objs.append(obj)
    procs = [(src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
             for src, cmd in jobs]
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(out.decode(errors="replace"))
        elif verbose:
            print(f"[build] compiled {src}")
    if failed:
        raise RuntimeError("nvcc failed building libpint_b200")
    link = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC"] + objs + [
        "-o", LIB, "-lcudart"]
    subprocess.check_call(link)
    with open(STAMP, "w") as f:
        f.write(source_hash())
    if verbose:
        print(f"[build] linked {LIB}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    args = ap.parse_args()
    build(force=args.force)
