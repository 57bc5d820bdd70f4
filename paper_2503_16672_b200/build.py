"""Build libs24.so in-tree (sm_100a) with plain nvcc.

The library has no torch dependency: it is a C-ABI shared object (see
include/s24.h) that the Python package loads with ctypes. Rebuilt only when a
source is newer than the library unless ``force``.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB = PKG_DIR / "libs24.so"
SOURCES = ["gemm_capi.cu", "sparse_capi.cu", "fp8.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [REPO / "include" / "s24.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps if p.is_file())


def build(force: bool = False, verbose: bool = False, defines: list[str] | None = None,
          out: Path | None = None) -> Path:
    """Compile libs24.so. `defines`/`out` build an experimental variant
    (e.g. a different tile configuration) next to the product library."""
    lib = Path(out) if out else LIB
    if not force and not defines and lib == LIB and not _stale():
        return LIB
    nvcc = _nvcc()
    objs = []
    tmp = PKG_DIR / "_build" / (lib.stem if lib != LIB else "")
    tmp.mkdir(parents=True, exist_ok=True)
    flags = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", *ARCH, "-I", str(REPO / "include")]
    flags += [f"-D{d}" for d in (defines or [])]
    procs = []
    for src in SOURCES:
        obj = tmp / (Path(src).stem + ".o")
        objs.append(obj)
        cmd = [nvcc, *flags, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{out}")
    link = [nvcc, "-shared", *ARCH, "-o", str(lib) + ".tmp", *map(str, objs), "-lcudart_static"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(link)}\n{r.stdout}{r.stderr}")
    os.replace(str(lib) + ".tmp", lib)
    return lib


if __name__ == "__main__":
    argv = sys.argv[1:]
    defs = [argv[i + 1] for i, a in enumerate(argv) if a == "-D"]
    out = next((argv[i + 1] for i, a in enumerate(argv) if a == "--out"), None)
    print(build(force="--force" in argv, verbose=True, defines=defs, out=out))
