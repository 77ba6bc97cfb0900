"""Build libhplmm.so in-tree with nvcc for sm_100a (no JIT, no torch ext)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libhplmm.so")
SOURCES = ["host_setup.cpp", "supernodal_host.cpp", "fem.cu", "dense.cu", "coarse.cu", "krylov.cu",
           "supernodal.cu", "sn_setup.cu", "cholesky.cu", "ilu.cu", "api.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off",
         "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-lcudart"]


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "hplmm.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return OUT
    extra = os.environ.get("HPLMM_NVCC_EXTRA", "").split()   # e.g. -DHPLMM_SN_PROF=1
    cmd = [NVCC] + FLAGS + extra + [os.path.join(CSRC, s) for s in SOURCES] + ["-o", OUT + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(OUT + ".tmp", OUT)
    if verbose:
        print(r.stderr[-4000:])
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
