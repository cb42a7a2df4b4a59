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
SOURCES = [os.path.join(CSRC, f) for f in ("skan_kernels.cu", "skan_head_b1.cu", "skan_gemm.cu", "skan_vq.cu", "skan_load.cu", "skan_api.cpp",
                                           "skan_format.cpp")]
HEADERS = [os.path.join(CSRC, f) for f in ("skan_internal.hpp", "skan_device.cuh", "skan_tc.cuh")] + [
    os.path.join(ROOT, "include", "skan.h")]
OUT = os.path.join(HERE, "libskan.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-shared",
         "-I" + os.path.join(ROOT, "include")]


OBJDIR = os.path.join(HERE, "build_obj")


def _obj(src: str) -> str:
    return os.path.join(OBJDIR, os.path.basename(src) + ".o")


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in SOURCES + HEADERS + [__file__])


def build_library(force: bool = False, verbose: bool = False) -> str:
    """Each translation unit compiles to its own object in parallel (only
    stale ones are rebuilt), then one nvcc link produces libskan.so."""
    if not force and up_to_date():
        return OUT
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJDIR, exist_ok=True)
    newest_hdr = max(os.path.getmtime(p) for p in HEADERS + [__file__])
    compile_flags = [f for f in FLAGS if f != "-shared"]

    def compile_one(src):
        obj = _obj(src)
        if (not force and os.path.exists(obj) and os.path.getmtime(obj) >= os.path.getmtime(src)
                and os.path.getmtime(obj) >= newest_hdr):
            return
        cmd = [NVCC, *ARCH, *compile_flags, "-c", "-o", obj + ".tmp", src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(obj + ".tmp", obj)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(compile_one, SOURCES))
    cmd = [NVCC, *ARCH, "-shared", "-Xlinker", "--no-undefined", "-o", OUT + ".tmp", *[_obj(s) for s in SOURCES]]
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT




REF_INCLUDE = "/root/reference/proj/include"
CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_lutham_b200.cpp")
CPP_TEST_BIN = os.path.join(ROOT, "tests", "cpp", "bin", "test_lutham_b200")


def build_cpp_tests(force: bool = False) -> str | None:
    """Compile the C++ drop-in parity test (tests/cpp) against the reference
    headers and the reference library in oracle/_ref (the checker).  Only
    possible where /root/reference exists; the binary travels to the GPU box
    with the snapshot.  Returns the binary path, or None if unbuildable here."""
    ref_so = os.path.join(ROOT, "oracle", "_ref", "libholoquant_ref.so")
    if not (os.path.isdir(REF_INCLUDE) and os.path.exists(ref_so)):
        return CPP_TEST_BIN if os.path.exists(CPP_TEST_BIN) else None
    deps = [CPP_TEST_SRC, os.path.join(ROOT, "include", "holoquant", "lutham_b200.hpp"),
            os.path.join(ROOT, "include", "skan.h"), OUT, ref_so]
    if (not force and os.path.exists(CPP_TEST_BIN)
            and all(os.path.getmtime(d) <= os.path.getmtime(CPP_TEST_BIN) for d in deps)):
        return CPP_TEST_BIN
    os.makedirs(os.path.dirname(CPP_TEST_BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I" + REF_INCLUDE, "-I" + os.path.join(ROOT, "include"),
           CPP_TEST_SRC, "-o", CPP_TEST_BIN,
           "-L" + os.path.dirname(ref_so), "-lholoquant_ref", "-L" + HERE, "-lskan",
           "-Wl,-rpath,$ORIGIN/../../../oracle/_ref", "-Wl,-rpath,$ORIGIN/../../../paper_2512_15742_b200",
           "-lpthread"]
    subprocess.run(cmd, check=True)
    return CPP_TEST_BIN


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
