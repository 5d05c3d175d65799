"""Build libtetri.so (sm_100a) in-tree with nvcc.

    python -m paper_2401_11181_b200.build

The library lands in paper_2401_11181_b200/lib/ so it travels with the repo
snapshot to the GPU box.  Objects are rebuilt only when a source or header is
newer than the library.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libtetri.so"
INCLUDE = PKG.parent / "include"
SOURCES = ["gemm.cu", "kernels.cu", "attention_tc.cu", "runtime.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         f"-I{INCLUDE}", f"-I{CSRC}"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    built = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > built for p in deps)


def build(force: bool = False, verbose: bool = False, experiments: bool = False) -> Path:
    """experiments=True (or TK_BUILD_EXPERIMENTS=1) builds lib/libtetri_exp.so with the
    GEMM experiment hooks (TK_GEMM_TRACE / _EXP / _WAIT / _PF ...); scripts load it via
    TK_LIB.  The product library never contains them."""
    experiments = experiments or bool(os.environ.get("TK_BUILD_EXPERIMENTS"))
    if experiments:
        return _build_into(LIB_DIR / "libtetri_exp.so", LIB_DIR / "obj_exp", ["-DTK_GEMM_EXPERIMENTS"],
                           verbose)
    if not force and not _stale():
        return LIB
    return _build_into(LIB, LIB_DIR / "obj", [], verbose)


def _build_into(LIB: Path, obj_dir: Path, extra: list, verbose: bool) -> Path:
    LIB_DIR.mkdir(exist_ok=True)
    obj_dir.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objs = []
    procs = []
    for src in SOURCES:
        obj = obj_dir / (Path(src).stem + ".o")
        objs.append(obj)
        cmd = [nvcc, *ARCH, *FLAGS, *extra, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{out.decode()}")
        if verbose and out:
            print(out.decode())
    tmp = LIB.with_suffix(".so.tmp")
    # cudart is linked as a shared library: a statically linked runtime inside
    # a dlopen()ed library hides its launches from Nsight Compute.
    link = [nvcc, *ARCH, "-shared", "-cudart", os.environ.get("TK_CUDART", "shared"), "-o",
            str(tmp), *map(str, objs), "-Xlinker", "-rpath,$ORIGIN"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(link)}\n{r.stdout}{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
