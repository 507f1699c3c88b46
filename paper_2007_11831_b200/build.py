"""Build libdbs_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2007_11831_b200.build [--force] [--jobs N]

Each csrc/*.cu is compiled to an object (controller.cu with -fmad=false so the
fp64 controller never contracts into FMA), then linked into
paper_2007_11831_b200/libdbs_b200.so.  The CUDA runtime is linked statically;
driver entry points (TMA descriptor encoding, IPC) are resolved at run time
through cudaGetDriverEntryPoint, so no libcuda stub is needed at build time.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libdbs_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-Xptxas", "-warn-spills", f"-I{ROOT / 'include'}"]
PER_FILE = {
    "controller.cu": ["-fmad=false"],
    "problems.cu": ["-fmad=false"],
    "theory.cu": ["-fmad=false"],
}
# measurement builds only: DBS_GEMM_ATTRIB=1 compiles gemm.cu's DBS_GEMM_DBG attribution
# switches in (they cost the production kernels registers; rebuild with force after toggling)
if os.environ.get("DBS_GEMM_ATTRIB") == "1":
    PER_FILE["gemm.cu"] = ["-DDBS_GEMM_ATTRIB"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(CSRC.glob("*.cu"))


def _deps(src: Path):
    return [src, *CSRC.glob("*.cuh"), ROOT / "include" / "dbs_b200.h"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def compile_one(src: Path, force: bool, verbose: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    if not force and not _stale(obj, _deps(src)):
        return obj
    cmd = [nvcc(), *ARCH, *COMMON, *PER_FILE.get(src.name, []), "-c", str(src), "-o", str(obj)]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed on {src.name}")
    if verbose and r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    srcs = sources()
    with ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: compile_one(s, force, verbose), srcs))
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lpthread", "-ldl", "-lrt"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.jobs, a.verbose))


if __name__ == "__main__":
    main()
