"""Build libduet.so in-tree (sm_100a).  ``python -m paper_2511_04791_b200.build``.

Host model code (predictor / optimizer) is compiled by g++ with -ffp-contract=off so its
doubles round exactly as written; CUDA sources by nvcc with
``-gencode arch=compute_100a,code=sm_100a`` (plain -arch=sm_100a would also embed
compute_100 PTX, which rejects tcgen05).
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(HERE, "libduet.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
GENCODE = "-gencode=arch=compute_100a,code=sm_100a"


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")
    return r.stdout + r.stderr


def _sources():
    cpp = sorted(glob.glob(os.path.join(CSRC, "*.cpp")))
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdr = sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                 glob.glob(os.path.join(CSRC, "kernels", "*.cuh")) + [os.path.join(ROOT, "include", "duet.h")])
    return cpp, cu, hdr


def _digest(files, extra=""):
    h = hashlib.sha256(extra.encode())
    for f in files:
        with open(f, "rb") as fh:
            h.update(f.encode())
            h.update(fh.read())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    cpp, cu, hdr = _sources()
    os.makedirs(BUILD, exist_ok=True)
    flags_cpp = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall",
                 f"-I{os.path.join(ROOT, 'include')}", f"-I{CUDA}/include"]
    flags_cu = ["-O3", "-std=c++17", GENCODE, "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off",
                "--expt-relaxed-constexpr", f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}",
                "-Xptxas", "-warn-spills"]
    stamp = os.path.join(BUILD, "libduet.stamp")
    flags_cu += os.environ.get("DUET_NVCC_EXTRA", "").split()   # A/B builds (e.g. -DDUET_NO_PDL_TRIGGER)
    dig = _digest(cpp + cu + hdr, " ".join(flags_cpp + flags_cu))
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == dig:
        return LIB
    objs = []
    for src in cpp:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        _run(["g++", *flags_cpp, "-c", src, "-o", obj])
        objs.append(obj)
    import concurrent.futures as cf
    def nv(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        out = _run([NVCC, *flags_cu, "-c", src, "-o", obj])
        if verbose and out.strip():
            print(out)
        return obj
    with cf.ThreadPoolExecutor(max_workers=max(1, min(8, len(cu)))) as ex:
        objs += list(ex.map(nv, cu))
    _run([NVCC, GENCODE, "-shared", "-cudart", "shared", "-o", LIB + ".tmp", *objs, f"-L{CUDA}/lib64"])
    os.replace(LIB + ".tmp", LIB)
    with open(stamp, "w") as fh:
        fh.write(dig)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
