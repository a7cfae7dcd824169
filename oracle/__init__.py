"""ORACLE — test infrastructure only (see oracle/rtm_oracle.cpp header).

Plain ctypes wrappers around the unblocked C++ CPU reference of the RTM 3D-model step
(§2, Algorithm 1).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` leg may import this package.
The product package ``paper_1310_8232_b200`` never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "rtm_oracle.cpp"
_LIB = _HERE / "liboracle.so"
_lib = None

CXXFLAGS = ["-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c++17", "-march=x86-64-v2"]


def build(force: bool = False) -> Path:
    """Compile oracle/rtm_oracle.cpp -> oracle/liboracle.so (g++, -ffp-contract=off)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["g++", *CXXFLAGS, str(_SRC), "-o", str(tmp)])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB))
        P = ctypes.c_void_p
        I = ctypes.c_int
        F = ctypes.c_float
        D = ctypes.c_double
        L.oracle_run_f32.argtypes = [I, I, I, F, F, P, P, P, P, I, P, P, P, I, P, P, I]
        L.oracle_run_f64.argtypes = [I, I, I, D, D, P, P, P, P, I, P, P, P, I, P, P, I]
        L.oracle_points_f32.argtypes = [I, I, I, F, F, P, P, P, P, ctypes.c_long, P, P]
        L.oracle_slab_step_f32.argtypes = [I, I, I, P, P, P, P, I]
        L.oracle_cfield_f32.argtypes = [ctypes.c_long, F, F, P, P]
        L.oracle_last_loop_seconds.argtypes = []
        L.oracle_last_loop_seconds.restype = D
        for f in ("oracle_run_f32", "oracle_run_f64", "oracle_points_f32",
                  "oracle_slab_step_f32", "oracle_cfield_f32", "oracle_max_threads"):
            getattr(L, f).restype = I
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _sources(sources, dtype):
    """sources: list of (x, y, z, samples) -> (xyz int32, concatenated samples, lengths)."""
    if not sources:
        return 0, np.zeros(3, np.int32), np.zeros(1, dtype), np.zeros(1, np.int32)
    xyz = np.array([[s[0], s[1], s[2]] for s in sources], dtype=np.int32).ravel()
    smp = [np.ascontiguousarray(s[3], dtype=dtype) for s in sources]
    lens = np.array([len(s) for s in smp], dtype=np.int32)
    cat = np.concatenate(smp) if lens.sum() else np.zeros(1, dtype)
    return len(sources), xyz, cat, lens


def run(v, dx, dt, coeffs, steps, u0=None, up0=None, sources=(), dtype=np.float32,
        nthreads=0, return_prev=False):
    """Run the oracle for ``steps`` steps.  ``v`` is (nz, ny, nx); returns u^steps
    (and u^(steps-1) if return_prev) as arrays of shape (nz, ny, nx) in ``dtype``."""
    dtype = np.dtype(dtype)
    nz, ny, nx = v.shape
    v = np.ascontiguousarray(v, dtype=dtype)
    c = np.ascontiguousarray(coeffs, dtype=dtype)
    u0 = None if u0 is None else np.ascontiguousarray(u0, dtype=dtype)
    up0 = None if up0 is None else np.ascontiguousarray(up0, dtype=dtype)
    ns, xyz, cat, lens = _sources(list(sources), dtype)
    out = np.empty((nz, ny, nx), dtype)
    prev = np.empty((nz, ny, nx), dtype) if return_prev else None
    f = lib().oracle_run_f32 if dtype == np.float32 else lib().oracle_run_f64
    rc = f(nx, ny, nz, dx, dt, _ptr(c), _ptr(v), _ptr(u0), _ptr(up0), ns, _ptr(xyz), _ptr(cat),
           _ptr(lens), int(steps), _ptr(out), _ptr(prev), int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_run failed rc={rc}")
    return (out, prev) if return_prev else out


def points_f32(v, dx, dt, coeffs, u, up, pts):
    """One fp32 step evaluated at points pts (k, 3) int (x, y, z); no source term."""
    nz, ny, nx = v.shape
    pts = np.ascontiguousarray(pts, dtype=np.int32)
    out = np.empty(len(pts), np.float32)
    c = np.ascontiguousarray(coeffs, dtype=np.float32)
    rc = lib().oracle_points_f32(nx, ny, nz, float(dx), float(dt), _ptr(c),
                                 _ptr(np.ascontiguousarray(v, np.float32)),
                                 _ptr(np.ascontiguousarray(u, np.float32)),
                                 _ptr(np.ascontiguousarray(up, np.float32)), len(pts), _ptr(pts),
                                 _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle_points failed rc={rc}")
    return out


def cfield_f32(v, dx, dt):
    v = np.ascontiguousarray(v, np.float32)
    C = np.empty_like(v)
    lib().oracle_cfield_f32(v.size, float(dx), float(dt), _ptr(v), _ptr(C))
    return C


def slab_step_f32(coeffs, C, U, P, nthreads=0):
    """In-place slab step: U, P are (nzl+10, ny, nx) float32 with explicit z-halo planes."""
    nzp, ny, nx = U.shape
    nzl = nzp - 10
    assert C.shape == (nzl, ny, nx) and P.shape == U.shape
    assert U.flags.c_contiguous and P.flags.c_contiguous and C.flags.c_contiguous
    c = np.ascontiguousarray(coeffs, dtype=np.float32)
    rc = lib().oracle_slab_step_f32(nx, ny, nzl, _ptr(c), _ptr(C), _ptr(U), _ptr(P), int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_slab_step failed rc={rc}")


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def last_loop_seconds() -> float:
    """Wall time of the step loop of the last ``run`` (allocation, C(p) and copies excluded)."""
    return float(lib().oracle_last_loop_seconds())
