"""Build ``libfastbcc_b200.so`` in-tree for sm_100a (nvcc, no JIT cache).

    python -m paper_2301_01356_b200.build [--force]

Each ``csrc/*.cu`` compiles to an object with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and the objects
link into one shared library exporting the C ABI of
``include/fastbcc_b200.h``.  The .so is git-ignored but travels to the GPU
box with the repo snapshot.
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libfastbcc_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-v"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [PKG.parent / "include" / "fastbcc_b200.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, extra=(), out: Path | None = None) -> Path:
    """extra / out: experiment builds (tools/build_variant.py) -- extra nvcc
    flags, a separate object directory and library path."""
    lib = out or LIB
    bdir = BUILD if out is None else BUILD.parent / "_build_variants" / lib.stem
    if out is None and not force and not _stale():
        return LIB
    nvcc = _nvcc()
    bdir.mkdir(parents=True, exist_ok=True)

    def compile_one(src):
        obj = bdir / (src.stem + ".o")
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stderr}")
        (bdir / (src.stem + ".ptxas.txt")).write_text(r.stderr)
        if verbose:
            sys.stderr.write(r.stderr)
        return str(obj)

    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:  # one nvcc per translation unit
        objs = list(ex.map(compile_one, sources()))
    lib.parent.mkdir(parents=True, exist_ok=True)
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
