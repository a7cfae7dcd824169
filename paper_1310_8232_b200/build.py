"""Build the in-tree C-ABI shared library ``librtm_b200.so`` for sm_100a with nvcc.

    python paper_1310_8232_b200/build.py [--verbose]   (standalone: does not import the package)

Kernels (csrc/rtm_kernels.cu) and the host library (csrc/rtm_host.cpp) are compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and linked against the NCCL 2.28
shipped in the venv (rpath'd), with cudart static.  nvcc cross-compiles without a GPU.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "librtm_b200.so"
SOURCES = [CSRC / "rtm_kernels.cu", CSRC / "rtm_tb.cu", CSRC / "rtm_resident.cu", CSRC / "rtm_stream2.cu",
           CSRC / "rtm_host.cpp"]
HEADERS = [CSRC / "rtm_internal.h", CSRC / "rtm_device.cuh", ROOT / "include" / "rtm.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl  # the venv's NCCL 2.28 (also what torch loads)
    base = Path(list(nvidia.nccl.__path__)[0])
    return base / "include", base / "lib"


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or Path(c).exists()):
            return c
    return "nvcc"


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    inc, lib = nccl_dirs()
    common = ["-std=c++17", "-O3", *ARCH, "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC",
              "-I", str(ROOT / "include"), "-I", str(inc)]
    if verbose:
        common += ["-Xptxas", "-v"]
    objs = []
    cmds = []
    for src in SOURCES:
        obj = PKG / "build" / (src.stem + ".o")
        obj.parent.mkdir(exist_ok=True)
        objs.append(obj)
        cmds.append([nvcc(), *common, "-c", str(src), "-o", str(obj)])
    with ThreadPoolExecutor(len(cmds)) as ex:
        for r in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds):
            if verbose or r.returncode:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode:
                raise RuntimeError(f"nvcc failed: {' '.join(r.args)}")
    tmp = LIB.with_suffix(f".so.tmp{os.getpid()}")
    link = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-L", str(lib),
            "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}", "-lcudart_static"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="--verbose" in sys.argv)
    print(LIB)
