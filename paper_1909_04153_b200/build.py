"""Build the sm_100a library in-tree: paper_1909_04153_b200/lib/libbsq.so.

    python -m paper_1909_04153_b200.build

nvcc cross-compiles without a GPU.  Flags that matter for parity:
--fmad=false (no contracted multiply-adds anywhere: the reference's numba
kernels emit none) and the default IEEE division / square root
(-prec-div=true -prec-sqrt=true); host code is built with
-ffp-contract=off for the same reason.

Every kernel source is compiled twice: once for the fp64 kernels with the
flags above (-DBSQ_TU_F64), once for the fp32 kernels (-DBSQ_TU_F32
-DBSQ_FAST_F32) with approximate single-precision square root and plain
division, flush-to-zero and (except where fp64 controller arithmetic shares
the file) contracted multiply-adds: the fp32 mode's contract is a tolerance,
not bits.  Its Markstein quotients stay correctly rounded (accuracy).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(OUT_DIR, "libbsq.so")
KERNEL_SOURCES = ["bsq_ghost.cu", "bsq_stage.cu", "bsq_stage_tiled.cu", "bsq_solve.cu", "bsq_cr.cu",
                  "bsq_spike.cu", "bsq_correct.cu", "bsq_final.cu", "bsq_check.cu"]
HOST_SOURCES = ["bsq_api.cu", "bsq_io.cpp"]
SOURCES = KERNEL_SOURCES + HOST_SOURCES
# fp32 objects keep --fmad=false where the file also runs fp64 scalar code that
# must match the host bit for bit (k_final's device controller) or is trivial
F32_NO_CONTRACT = {"bsq_final.cu", "bsq_ghost.cu"}
HEADERS = ["bsq_device.cuh", "bsq_launch.h", "bsq_tma.cuh"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
    "-ccbin", "/usr/bin/g++",
]


def flags_for(src: str, prec: str) -> list:
    """nvcc flags of one object: prec is "f64", "f32" or "" (host sources)."""
    if prec == "f64":
        return [*FLAGS, "-DBSQ_TU_F64"]
    if prec == "f32":
        fl = [f for f in FLAGS if f not in ("--fmad=false", "-prec-div=true", "-prec-sqrt=true")]
        fl += ["-prec-div=false", "-prec-sqrt=false", "-ftz=true",
               "--fmad=false" if src in F32_NO_CONTRACT else "--fmad=true",
               "-DBSQ_TU_F32", "-DBSQ_FAST_F32"]
        return fl + os.environ.get("BSQ_F32_EXTRA", "").split()  # A/B builds only
    return list(FLAGS)


def jobs(out_dir: str = None) -> list:
    """(source, object, precision) for every object of the library."""
    out_dir = out_dir or OUT_DIR
    res = []
    for src in KERNEL_SOURCES:
        stem = os.path.splitext(src)[0]
        res.append((src, os.path.join(out_dir, stem + ".o"), "f64"))
        res.append((src, os.path.join(out_dir, stem + "_f32.o"), "f32"))
    for src in HOST_SOURCES:
        res.append((src, os.path.join(out_dir, os.path.splitext(src)[0] + ".o"), ""))
    return res


def compile_jobs(todo: list, extra: list = (), verbose: bool = False) -> list:
    """Compile (source, object, precision) jobs in parallel; returns stderr texts."""
    from concurrent.futures import ThreadPoolExecutor

    def one(job):
        src, obj, prec = job
        cmd = [nvcc(), *flags_for(src, prec), *extra, "-c", os.path.join(SRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed on {src} ({prec or 'host'})")
        return f"{src} [{prec or 'host'}]\n" + res.stderr

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        logs = list(ex.map(one, todo))
    if verbose:
        for lg in logs:
            sys.stderr.write(lg)
    return logs


def link(objs: list, out: str) -> None:
    tmp = out + ".tmp"
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           "-ccbin", "/usr/bin/g++", "-lcudart", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, out)


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(SRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(PKG), "include", "bsq.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    todo = jobs()
    compile_jobs(todo, verbose=verbose)
    link([o for _, o, _ in todo], LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
