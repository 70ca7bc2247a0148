"""Build the two in-tree libraries (no JIT cache: the .so files travel to the GPU box).

libcwgpu.so         the server answer path: nvcc for sm_100a (api.cu + params.cpp), C ABI
                    include/cwgpu.h.
libcwgpu_client.so  the seeded client (keygen / query packing / decryption, include/cwgpu_client.h)
                    on the CPU, g++ only -- kept out of the product library so that harness code
                    which only needs keys and queries never maps the CUDA library.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libcwgpu.so")
CLIENT_LIB = os.path.join(HERE, "libcwgpu_client.so")
SOURCES = ["api.cu", "params.cpp"]
CLIENT_SOURCES = ["client.cpp", "params.cpp"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-shared",
]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-shared"]


def _inputs(exclude=("client.cpp",)):
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f not in exclude]  # every source and header
    files += [os.path.join(INC, f) for f in os.listdir(INC) if f != "cwgpu_client.h"]
    return files


def _stale(lib, inputs) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(f) > t for f in inputs)


def needs_build() -> bool:
    return _stale(LIB, _inputs()) or _stale(CLIENT_LIB, _client_inputs())


def _client_inputs():
    return [os.path.join(CSRC, f) for f in ("client.cpp", "params.cpp", "params.h")] + [
        os.path.join(INC, "cwgpu_client.h")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def build_client(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale(CLIENT_LIB, _client_inputs()):
        return CLIENT_LIB
    cmd = [os.environ.get("CXX", "g++"), *CXX_FLAGS, "-o", CLIENT_LIB + ".tmp",
           *[os.path.join(CSRC, f) for f in CLIENT_SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(CLIENT_LIB + ".tmp", CLIENT_LIB)
    return CLIENT_LIB


def build(force: bool = False, verbose: bool = False) -> str:
    build_client(force, verbose)
    if not force and not _stale(LIB, _inputs()):
        return LIB
    srcs = [os.path.join(CSRC, f) for f in SOURCES]
    cmd = [nvcc(), *NVCC_FLAGS, "-o", LIB + ".tmp", *srcs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
