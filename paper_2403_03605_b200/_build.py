"""In-tree build of libpmts.so for sm_100a (nvcc cross-compiles without a GPU).

Deterministic kernels (pd_det.cu) build with -fmad=false so their fp64
arithmetic rounds like the reference; the fast kernels keep FMA.
Host code builds with -ffp-contract=off for the bit-exact setup restatement.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib")
LIB = os.path.join(OUT, "libpmts.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

SOURCES = [
    # (file, extra nvcc flags)
    ("pd_det.cu", ["-fmad=false"]),
    ("pd_fast.cu", []),
    ("pd_stencil.cu", []),
    ("pd_tile9.cu", []),
    ("pd_lat3.cu", []),
    ("pd_setup.cu", ["-fmad=false"]),
    ("pmts_pd.cu", ["-fmad=false"]),
    ("pd_mts.cu", ["-fmad=false"]),
    ("pd_mts_lat.cu", ["-fmad=false"]),
    ("pmts_mts.cu", ["-fmad=false"]),
]
HOST_SOURCES = ["pmts_setup.cpp", "pmts_mts_setup.cpp"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(os.path.join(OUT, "obj"), exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(HERE, "..", "include", "pmts_capi.h"))
    objs = []
    jobs = []
    for src, extra in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT, "obj", src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + headers):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v",
                         "-Xcompiler", "-fPIC,-ffp-contract=off", *extra,
                         *os.environ.get("PMTS_NVCC_FLAGS", "").split(), "-c", s, "-o", o])
    for src in HOST_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT, "obj", src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + headers):
            jobs.append(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-c", s,
                         "-o", o])
    procs = [(j, subprocess.Popen(j, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                  text=True)) for j in jobs]
    for j, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError("build failed: " + " ".join(j))
        if verbose and out:
            sys.stderr.write(out)
    if force or jobs or not os.path.exists(LIB):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
