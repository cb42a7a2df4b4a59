"""In-tree build of libskan.so for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2512_15742_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(CSRC, f) for f in ("skan_kernels.cu", "skan_head_b1.cu", "skan_api.cpp", "skan_format.cpp")]
HEADERS = [os.path.join(CSRC, "skan_internal.hpp"), os.path.join(CSRC, "skan_device.cuh"), os.path.join(ROOT, "include", "skan.h")]
OUT = os.path.join(HERE, "libskan.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-shared",
         "-I" + os.path.join(ROOT, "include")]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in SOURCES + HEADERS + [__file__])


def build_library(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    cmd = [NVCC, *ARCH, *FLAGS, "-o", OUT + ".tmp", *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
