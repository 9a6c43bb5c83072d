"""Build libptycho_b200.so in-tree with nvcc for sm_100a (no torch extension
machinery: the library is a plain C-ABI shared object loaded with ctypes)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = Path(os.environ["PTY_LIB_OUT"]).resolve() if os.environ.get("PTY_LIB_OUT") else PKG / "libptycho_b200.so"
SOURCES = sorted(CSRC.glob("*.cu"))
DEPS = sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "ptycho_b200.h"] + SOURCES
OBJDIR = PKG / "build" if LIB.parent == PKG and LIB.name == "libptycho_b200.so" else LIB.parent / f"build_{LIB.stem}"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# experiment builds: PTY_NVCC_DEFS="-DX -DY" and PTY_LIB_OUT=<path> build a variant
# library beside the default one (loaded with PTY_LIB=<path>)
EXTRA = os.environ.get("PTY_NVCC_DEFS", "").split()
FLAGS = ["-O3", "-lineinfo", "--std=c++17", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-I", str(ROOT / "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def _compile(src: Path, verbose: bool):
    obj = OBJDIR / (src.stem + ".o")
    cmd = [nvcc(), *ARCH, *FLAGS, *EXTRA, *(["-Xptxas", "-v"] if verbose else []), "-c", "-o", str(obj), str(src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return src, obj, res


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> Path:
    """Compile every csrc/*.cu for sm_100a in parallel and link the C-ABI library."""
    from concurrent.futures import ThreadPoolExecutor
    if not force and not needs_build():
        return LIB
    OBJDIR.mkdir(exist_ok=True)
    jobs = jobs or max(1, min(len(SOURCES), os.cpu_count() or 1))
    with ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    failed = [r for r in results if r[2].returncode != 0]
    for src, _, res in results:
        if verbose or res.returncode != 0:
            sys.stderr.write(f"== {src.name}\n" + res.stdout + res.stderr)
    if failed:
        raise RuntimeError(f"nvcc failed for {[f[0].name for f in failed]}")
    tmp = LIB.with_suffix(".so.tmp")
    link = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *[str(r[1]) for r in results]]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
