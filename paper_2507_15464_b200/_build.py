"""Build the in-tree C-ABI library ``libtidas_b200.so`` with nvcc for sm_100a.

``python -m paper_2507_15464_b200._build`` (or ``__graft_entry__.build()``).
The .so lands next to this file so it travels with the repo snapshot to the GPU
box; it is git-ignored.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libtidas_b200.so"
SOURCES = ["api.cu", "analytic.cu", "das.cu", "rowconv.cu", "rowconv_tc1.cu", "rowkernels.cu", "tidas_ops.cu", "simulate.cu", "sweep.cu", "metrics.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# K1's packed complex arithmetic folds +-i into FADD2 operand modifiers only
# without flush-to-zero (common.cuh)
NO_FTZ = {"analytic.cu"}
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-ftz=true",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "tidas_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every translation unit in parallel (one nvcc per .cu), then link."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    objdir = PKG.parent / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    compile_flags = [f for f in FLAGS if f != "-shared"]

    def compile_one(src: str):
        obj = objdir / (Path(src).stem + ".o")
        flags = [f for f in compile_flags if not (src in NO_FTZ and f.startswith("-ftz"))]
        cmd = [nvcc(), *ARCH, *flags, "-c", str(CSRC / src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, res, obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    link = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", *[str(r[2]) for r in results], "-o", str(tmp)]
    lres = subprocess.run(link, capture_output=True, text=True) if all(r[1].returncode == 0 for r in results) else None
    log = PKG / "build.log"
    log.write_text("".join(" ".join(c) + "\n" + r.stdout + r.stderr for c, r, _ in results)
                   + (" ".join(link) + "\n" + lres.stdout + lres.stderr if lres else ""))
    failed = [r for _, r, _ in results if r.returncode != 0] + ([lres] if lres and lres.returncode != 0 else [])
    if failed:
        sys.stderr.write(failed[0].stderr[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write("".join(r.stderr for _, r, _ in results))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
