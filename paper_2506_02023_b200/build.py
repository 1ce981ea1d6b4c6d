"""Build the sm_100a shared library libgraphmd_b200.so in-tree with nvcc.

    python -m paper_2506_02023_b200.build        (or build() from Python)

Every translation unit is compiled for `-gencode arch=compute_100a,code=sm_100a`
with -lineinfo (ncu source view).  Host code is compiled with
-ffp-contract=off so the fp64 lattice algebra matches the reference's
unfused x86-64 arithmetic bit for bit.  The CUDA runtime is linked
statically so the library loads on the GPU box without extra paths.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgraphmd_b200.so")
OBJ = os.path.join(HERE, "build_obj")
SOURCES = ["gmd_scan.cu", "gmd_graph.cu", "gmd_partition.cu", "gmd_linegraph.cu",
           "gmd_model.cu", "gmd_generic.cu", "gmd_wide.cu", "gmd_comm.cu", "gmd_md.cu", "gmd_builders.cu",
           "gmd_api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
         "-Xptxas", "-O3", "--expt-relaxed-constexpr"]


def _deps_mtime():
    return max(os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC)) if os.path.isdir(CSRC) else 0


# Files whose backward computes the edge/reverse-edge products
# (m_u h_w + h_u m_w) that must round identically at both ends (exact
# Newton's third law, gmd_model.cu grad_add): ptxas contracts
# add.rn.f32x2(mul.rn.f32x2, mul.rn.f32x2) into an FFMA2 despite the explicit
# rounding (checked in the SASS), which makes the two ends differ by an ulp.
# Every intended fusion in these files is an explicit fmaf / __ffma2_rn.
NO_FMAD = {"gmd_model.cu", "gmd_wide.cu"}


def _compile(src: str) -> str:
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    extra = ["-fmad=false"] if src in NO_FMAD else []
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    hdr = os.path.join(os.path.dirname(HERE), "include", "graphmd_b200.h")
    newest = max(_deps_mtime(), os.path.getmtime(hdr), os.path.getmtime(__file__))
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static", "-lrt", "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
