"""In-tree build of libcomoe_b200.so (sm_100a) with nvcc.

The shared library is the product's compute path; Python loads it with
ctypes (see _lib.py). Objects go to build/, the .so next to this file so it
travels with the repository snapshot to the GPU box.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "csrc"
LIB = PKG / "libcomoe_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr",
              "-Xcompiler", "-fPIC",
              "-I", str(ROOT / "include")]

SOURCES = ["capi.cu", "gate.cu", "permute.cu", "ffn.cu", "merge.cu",
           "similarity.cu", "predictor.cu", "peer.cu"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"),
                 "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA extension cannot be built")


def _needs(obj: Path, deps: list) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, ptxas_info: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    exe = nvcc()
    jobs = []
    for src in SOURCES:
        s = CSRC / src
        o = BUILD / (s.stem + ".o")
        if force or _needs(o, [s] + headers):
            cmd = [exe, *ARCH, *NVCC_FLAGS, "-c", str(s), "-o", str(o)]
            if ptxas_info:
                cmd += ["-Xptxas", "-v"]
            jobs.append((cmd, o))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for (cmd, o), res in zip(jobs, ex.map(
                lambda j: subprocess.run(j[0], capture_output=True, text=True), jobs)):
            if verbose or res.returncode != 0 or ptxas_info:
                sys.stderr.write(res.stdout + res.stderr)
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed for {o.name}")
    objs = [str(BUILD / (Path(s).stem + ".o")) for s in SOURCES]
    if force or jobs or not LIB.exists():
        cmd = [exe, *ARCH, "-shared", "-o", str(LIB), *objs]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link of libcomoe_b200.so failed")
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, ptxas_info="--ptxas" in sys.argv,
          force="--force" in sys.argv)
    print(LIB)
