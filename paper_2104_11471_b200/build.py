"""Build the sm_100a extension in-tree: paper_2104_11471_b200/libtcfft_b200.so.

nvcc cross-compiles for sm_100a without a GPU.  ``-gencode
arch=compute_100a,code=sm_100a`` is required: plain ``-arch=sm_100a`` also
embeds compute_100 PTX, which ptxas rejects for tcgen05 instructions.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libtcfft_b200.so"
SOURCES = [CSRC / "tcfft_api.cu", CSRC / "plan.cpp"]
# every source and header the library is built from (a stale .so must never load)
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.hpp")) + sorted((ROOT / "include").glob("*.h"))


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (Path(c).exists() or c == "nvcc"):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: Path | None = None) -> Path:
    out = Path(out) if out else LIB
    if out == LIB and not force and not needs_build():
        return LIB
    cmd = [
        nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
        "-shared", "-Xcompiler", "-fPIC", "-cudart", "static", "-I", str(ROOT / "include"),
        "-Xptxas", "-v" if verbose else "-O3",
        *[f"-D{d}" for d in os.environ.get("TCFFT_DEFINES", "").split(",") if d],
        "-o", str(out) + ".tmp", *map(str, SOURCES),
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libtcfft_b200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(str(out) + ".tmp", out)
    return out


if __name__ == "__main__":
    o = None
    if "-o" in sys.argv:
        o = sys.argv[sys.argv.index("-o") + 1]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=o))
