"""Build the sm_100a C-ABI library ``libsun_b200.so`` in-tree with nvcc.

The library is the only compute path of the package (no Triton, no CPU
fallback). It is built here (CPU container, nvcc cross-compiles sm_100a) and
travels to the GPU box inside the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libsun_b200.so"
SOURCES = [CSRC / "sun_capi.cu"]
DEPS = SOURCES + sorted(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "sun_b200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-cudart", "static",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v,-warn-spills",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the SUN B200 kernels cannot be built")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not needs_build():
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    extra = os.environ.get("SUN_NVCC_EXTRA", "").split()  # experiments only (e.g. -DSUN_W4_CONV_WARPS=16)
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", str(tmp), *map(str, SOURCES)]
    proc = subprocess.run(cmd, cwd=str(CSRC), capture_output=True, text=True)
    log = proc.stdout + proc.stderr
    (PKG / "build.log").write_text(" ".join(cmd) + "\n" + log)
    if proc.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed ({proc.returncode}); see {PKG / 'build.log'}")
    if verbose:
        sys.stdout.write(log)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
