"""Build libhplmm.so in-tree with nvcc for sm_100a (no JIT, no torch ext)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libhplmm.so")
SOURCES = ["host_setup.cpp", "supernodal_host.cpp", "fem.cu", "dense.cu", "coarse.cu", "krylov.cu",
           "supernodal.cu", "sn_setup.cu", "cholesky.cu", "ilu.cu", "gmres.cu", "multirhs.cu", "api.cu"]
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
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f not in ("-shared", "-lcudart")]
    # one nvcc per translation unit, in parallel (each .cu holds its own kernels
    # and host launchers: no device linking), then one shared-library link
    jobs = [(s, [NVCC] + cflags + extra + ["-c", os.path.join(CSRC, s), "-o",
                                           os.path.join(objdir, s + ".o")]) for s in SOURCES]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
        res = list(ex.map(lambda j: (j, subprocess.run(j[1], capture_output=True, text=True)), jobs))
    link = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-lcudart"] + \
        [os.path.join(objdir, s + ".o") for s in SOURCES] + ["-o", OUT + ".tmp"]
    log = os.path.join(HERE, "build.log")
    ok = all(r.returncode == 0 for _, r in res)
    text = "".join(" ".join(j[1]) + "\n" + r.stdout + r.stderr for j, r in res)
    if ok:
        r = subprocess.run(link, capture_output=True, text=True)
        text += " ".join(link) + "\n" + r.stdout + r.stderr
        ok = r.returncode == 0
    with open(log, "w") as f:
        f.write(text)
    if not ok:
        sys.stderr.write(text[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(OUT + ".tmp", OUT)
    if verbose:
        print(text[-4000:])
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
