"""Build the sm_100a shared library libhtrise_cuda.so in-tree with nvcc.

The library is the product: CUDA kernels (csrc/k_*.cu), the native runtime
(csrc/runtime.cu) and the C-ABI (csrc/capi.cu, include/htrise_cuda.h).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhtrise_cuda.so")
SOURCES = ["k_gemm.cu", "k_misc.cu", "k_eig.cu", "k_fused3.cu", "k_tail3.cu", "k_tail4.cu", "k_quad.cu", "k_decode.cu", "k_gram.cu", "k_tridiag.cu", "k_proj2.cu"]
HOST_SOURCES = ["runtime.cpp", "capi.cpp"]
CXX = os.environ.get("CXX", "g++")
CUDA_INC = "/usr/local/cuda/include"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _newest_input() -> float:
    paths = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    paths += [os.path.join(ROOT, "include", "htrise_cuda.h")]
    paths += [os.path.join(ROOT, "include", "htrise", f) for f in os.listdir(os.path.join(ROOT, "include", "htrise"))]
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_input():
        return LIB
    objdir = os.path.join(PKG, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for src in HOST_SOURCES:
        obj = os.path.join(objdir, src.replace(".cpp", ".o"))
        cmd = [CXX, "-O3", "-g", "-std=c++20", "-fPIC", "-fvisibility=hidden", "-Wall", "-Wno-unused-function",
               "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", CUDA_INC, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append(f"--- {src}\n{out}")
        elif verbose and out:
            print(out)
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl", "-Xlinker", "--exclude-libs,ALL"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


DROPIN_SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
DROPIN_BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_dropin")


def build_dropin_test() -> str:
    """Compile the C++ drop-in test program (reference-style tests written
    against include/htrise/*.hpp, linked to libhtrise_cuda.so)."""
    os.makedirs(os.path.dirname(DROPIN_BIN), exist_ok=True)
    cmd = [CXX, "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", CUDA_INC, DROPIN_SRC,
           "-L", PKG, "-lhtrise_cuda", "-Wl,-rpath,$ORIGIN/../../../paper_2412_16544_b200", "-o", DROPIN_BIN]
    subprocess.run(cmd, check=True)
    return DROPIN_BIN


IO_SRC = os.path.join(ROOT, "tests", "cpp", "test_io.cpp")
IO_BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_io")
PIN_SRC = os.path.join(ROOT, "tests", "cpp", "json_pin.cpp")
PIN_BIN = os.path.join(ROOT, "tests", "cpp", "build", "json_pin")
# the reference serialises container headers with nlohmann::json; the copy
# shipped in this image is the format checker of json_pin (test only)
NLOHMANN_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"


def build_io_test() -> str:
    """Compile the container test program (tests/cpp/test_io.cpp)."""
    os.makedirs(os.path.dirname(IO_BIN), exist_ok=True)
    cmd = [CXX, "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", CUDA_INC, IO_SRC,
           "-L", PKG, "-lhtrise_cuda", "-Wl,-rpath,$ORIGIN/../../../paper_2412_16544_b200", "-o", IO_BIN]
    subprocess.run(cmd, check=True)
    return IO_BIN


CLI_SRC = os.path.join(PKG, "cli", "htrise_cli.cpp")
CLI_BIN = os.path.join(PKG, "htrise")


def build_cli() -> str:
    """The `htrise` command-line tool (reference tools/main.cpp) over the
    drop-in headers, next to the library it links."""
    cmd = [CXX, "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", CUDA_INC, CLI_SRC,
           "-L", PKG, "-lhtrise_cuda", "-Wl,-rpath,$ORIGIN", "-o", CLI_BIN]
    subprocess.run(cmd, check=True)
    return CLI_BIN


def build_json_pin():
    """Compile json_pin against the image's nlohmann::json, if present."""
    if not os.path.exists(os.path.join(NLOHMANN_INC, "nlohmann", "json.hpp")):
        return None
    os.makedirs(os.path.dirname(PIN_BIN), exist_ok=True)
    subprocess.run([CXX, "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", NLOHMANN_INC, PIN_SRC,
                    "-o", PIN_BIN], check=True)
    return PIN_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    print(build_dropin_test())
    print(build_io_test())
    print(build_json_pin())
    print(build_cli())
