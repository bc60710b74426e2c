"""Build the sm_100a shared library in-tree with nvcc (no torch extension,
no JIT cache): paper_2507_01021_b200/_lib/libdictamux_b200.so.

The library exports only the C ABI declared in include/dictamux_b200.h.
"""

from __future__ import annotations

import hashlib
import os
import shlex
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libdictamux_b200.so"
SOURCES = ["engine.cu", "gemm.cu", "attention.cu", "logmel.cu", "decode.cu", "ctc.cu", "vad.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-Xptxas", "-v"]
# experiment builds only (e.g. -DDM_ATTN_TRACE, -DDM_XA_KEYS=128): scripts/build_variant.sh
FLAGS += shlex.split(os.environ.get("DM_NVCC_EXTRA", ""))


def _fingerprint() -> str:
    h = hashlib.sha256()
    for f in sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh"))
                    + [ROOT / "include" / "dictamux_b200.h", Path(__file__)]):
        h.update(f.name.encode())
        h.update(f.read_bytes())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> Path:
    LIBDIR.mkdir(exist_ok=True)
    stamp = LIBDIR / "build.sha256"
    fp = _fingerprint()
    if LIB.exists() and stamp.exists() and stamp.read_text() == fp and not force:
        return LIB
    objs = []
    for src in SOURCES:
        obj = LIBDIR / (Path(src).stem + ".o")
        cmd = [NVCC, *FLAGS, "-I", str(ROOT / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = LIBDIR / (Path(src).stem + ".ptxas.log")
        log.write_text(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
        if verbose:
            print(r.stderr, file=sys.stderr)
        objs.append(str(obj))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(LIB),
           *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    stamp.write_text(fp)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
