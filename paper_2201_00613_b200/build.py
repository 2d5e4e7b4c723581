"""Builds libsqueeze.so (the C-ABI library of include/squeeze.h) in-tree for sm_100a.

    python -m paper_2201_00613_b200.build        # or __graft_entry__.build()

nvcc cross-compiles without a GPU.  The .so lands next to this file so that it travels
to the GPU box with the repository snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsqueeze.so")
SOURCES = ["sqz_api.cu", "sqz_kernels.cu", "sqz_tile.cu", "sqz_stream.cu", "sqz_packed.cu", "sqz_engines.cu", "sqz_bb.cu", "sqz_heat.cu", "sqz_mma.cu", "sqz_host.cpp"]
HEADERS = ["sqz_common.h", "sqz_host.h", "sqz_kernels.cuh", "sqz_device.cuh", "sqz_bits.cuh", "sqz_heat.cuh"]

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-O3,-Wall",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_rebuild() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "squeeze.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compiles every source to an object in parallel (one nvcc per translation unit), then
    links the shared library."""
    if not force and not needs_rebuild():
        return LIB
    import concurrent.futures as cf
    import tempfile

    nvcc = nvcc_path()
    with tempfile.TemporaryDirectory(prefix="sqz_build_") as tmpd:
        def compile_one(src):
            obj = os.path.join(tmpd, src + ".o")
            cmd = [nvcc, *NVCC_FLAGS, "-c", "-o", obj, os.path.join(CSRC, src)]
            proc = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
            return obj, " ".join(cmd) + "\n" + proc.stdout + proc.stderr, proc.returncode

        with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
            results = list(ex.map(compile_one, SOURCES))
        log = "".join(r[1] for r in results)
        rc = max(r[2] for r in results)
        tmp = LIB + ".tmp"
        if rc == 0:
            cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp,
                   *[r[0] for r in results], "-lpthread"]
            proc = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
            log += " ".join(cmd) + "\n" + proc.stdout + proc.stderr
            rc = proc.returncode
    with open(os.path.join(HERE, "build.log"), "w") as fh:
        fh.write(log)
    if rc != 0:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed (see paper_2201_00613_b200/build.log)")
    if verbose:
        sys.stdout.write(log)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
