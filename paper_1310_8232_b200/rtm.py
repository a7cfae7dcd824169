"""Thin ctypes binding of the C ABI in include/rtm.h (argument marshalling only).

Every function here has the name of the C entry point it calls.  Arrays are numpy
float32, C-contiguous, shape (nz, ny, nx) (x fastest), or raw device pointers (ints, e.g.
``tensor.data_ptr()``) for the ``*_device`` calls.  Errors raise :class:`RtmError` with
the library's rtm_last_error() message.  There is no fallback: if ``librtm_b200.so`` is
missing or cannot be loaded, importing this module fails.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "librtm_b200.so"

RTM_OK, RTM_EINVAL, RTM_ECFL, RTM_ENOMEM, RTM_ECUDA, RTM_ENCCL, RTM_ESTATE = 0, -1, -2, -3, -4, -5, -6
RTM_EUNSTABLE = -7
RTM_MAX_SOURCES = 64
RTM_OPT_ZCHUNK, RTM_OPT_CACHE_MODE, RTM_OPT_GRAPHS, RTM_OPT_SHOT_ORDER, RTM_OPT_HALO_MODE = 1, 2, 3, 4, 5
RTM_OPT_CHECK_EVERY = 6
RTM_OPT_TB_CTAS = 7
RTM_OPT_PDL = 8
RTM_OPT_HOST_ORDERED = 9
RTM_OPT_ZDIR = 10
RTM_OPT_SLAB_SHARE = 11
RTM_IPC_RECORD_BYTES = 512
_NAMES = {0: "RTM_OK", -1: "RTM_EINVAL", -2: "RTM_ECFL", -3: "RTM_ENOMEM", -4: "RTM_ECUDA",
          -5: "RTM_ENCCL", -6: "RTM_ESTATE", -7: "RTM_EUNSTABLE"}


class RtmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


if not _LIB_PATH.exists():
    raise ImportError(f"{_LIB_PATH} not built; run python paper_1310_8232_b200/build.py "
                      "(the product has no CPU fallback)")
lib = ctypes.CDLL(str(_LIB_PATH))

_P, _I, _F, _D, _LL = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_double, ctypes.c_longlong


class rtm_tune_result(ctypes.Structure):
    _fields_ = [("best_tile", ctypes.c_int), ("best_zchunk", ctypes.c_int),
                ("ncandidates", ctypes.c_int), ("min_time_ms", ctypes.c_double),
                ("actual_time_ms", ctypes.c_double), ("quality_pct", ctypes.c_double)]
_SIGS = {
    "rtm_create": (_P, [_I, _I, _I, _F, _F, _P]),
    "rtm_set_velocity": (_I, [_P, _P]),
    "rtm_inject_source": (_I, [_P, _I, _I, _I, _P, _I]),
    "rtm_step": (_I, [_P, _I]),
    "rtm_read_field": (_I, [_P, _P]),
    "rtm_destroy": (None, [_P]),
    "rtm_last_error": (ctypes.c_char_p, []),
    "rtm_set_fields": (_I, [_P, _P, _P]),
    "rtm_read_fields": (_I, [_P, _P, _P]),
    "rtm_reset": (_I, [_P]),
    "rtm_step_count": (_LL, [_P]),
    "rtm_get_dims": (_I, [_P, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_I),
                         ctypes.POINTER(_I)]),
    "rtm_set_step_count": (_I, [_P, _LL]),
    "rtm_field_stats": (_I, [_P, ctypes.POINTER(_D), ctypes.POINTER(_LL)]),
    "rtm_set_velocity_device": (_I, [_P, _P]),
    "rtm_read_field_device": (_I, [_P, _P]),
    "rtm_set_tile": (_I, [_P, _I]),
    "rtm_get_tile": (_I, [_P]),
    "rtm_num_tiles": (_I, []),
    "rtm_set_zchunk": (_I, [_P, _I]),
    "rtm_set_option": (_I, [_P, _I, _LL]),
    "rtm_get_option": (_LL, [_P, _I]),
    "rtm_tile_name": (ctypes.c_char_p, [_I]),
    "rtm_set_stream": (_I, [_P, _P]),
    "rtm_last_elapsed_ms": (_F, [_P]),
    "rtm_set_profiling": (_I, [_P, _I]),
    "rtm_kernel_stats": (_I, [_P, ctypes.POINTER(_LL), ctypes.POINTER(_D)]),
    "rtm_launch_count": (_LL, [_P]),
    "rtm_create_multi": (_P, [_I, _I, _I, _F, _F, _P, _I, _P]),
    "rtm_create_batch": (_P, [_I, _I, _I, _F, _F, _P, _I]),
    "rtm_num_shots": (_I, [_P]),
    "rtm_inject_source_shot": (_I, [_P, _I, _I, _I, _I, _P, _I]),
    "rtm_get_unique_id": (_I, [_P]),
    "rtm_create_dist": (_P, [_I, _I, _I, _F, _F, _P, _I, _I, _P, _I]),
    "rtm_slab_range": (_I, [_I, _I, _I, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "rtm_halo_plan": (_I, [_I, _I, _I, _I, _I, ctypes.POINTER(_LL), ctypes.POINTER(_LL)]),
    "rtm_nu_crit": (_D, [_P]),
    "rtm_autotune": (_I, [_P, _I, _P, _P, _I, ctypes.POINTER(rtm_tune_result), _P]),
    "rtm_select_mwmb": (_I, [_P, _I, _I]),
    "rtm_blocksize_lattice": (_I, [_I, _I, _P]),
    "rtm_set_velocity_async": (_I, [_P, _P]),
    "rtm_step_async": (_I, [_P, _I]),
    "rtm_read_field_async": (_I, [_P, _P]),
    "rtm_sync": (_I, [_P]),
    "rtm_create_peer": (_P, [_I, _I, _I, _F, _F, _P, _I, _I, _I]),
    "rtm_ipc_export": (_I, [_P, _P]),
    "rtm_ipc_import": (_I, [_P, _P, _P]),
    "rtm_set_host_barrier": (_I, [_P, _P, _P]),
    "rtm_last_enqueue_ms": (_D, [_P]),
}
BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)
_barriers: dict = {}  # handle -> the ctypes callback object (kept alive while installed)
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def _err() -> str:
    m = lib.rtm_last_error()
    return m.decode() if m else ""


def _check(rc: int) -> int:
    if rc != RTM_OK:
        raise RtmError(rc, _err())
    return rc


def _f32(a, n=None, name="array"):
    a = np.ascontiguousarray(a, dtype=np.float32)
    if n is not None and a.size != n:
        raise ValueError(f"{name} has {a.size} elements, expected {n}")
    return a


def rtm_get_dims(h):
    """(nx, ny, nzl, nshots) of the host arrays the context reads and writes."""
    nx, ny, nzl, ns = _I(0), _I(0), _I(0), _I(0)
    _check(lib.rtm_get_dims(h, ctypes.byref(nx), ctypes.byref(ny), ctypes.byref(nzl),
                            ctypes.byref(ns)))
    return int(nx.value), int(ny.value), int(nzl.value), int(ns.value)


def _n_velocity(h):
    nx, ny, nzl, _ = rtm_get_dims(h)
    return nx * ny * nzl


def _n_field(h):
    nx, ny, nzl, ns = rtm_get_dims(h)
    return nx * ny * nzl * ns


def _out_buf(a, h, name):
    """A host output array the library writes the context's field into: it must be exactly
    that (float32, C-contiguous, writeable, nshots*nzl*ny*nx elements)."""
    if not isinstance(a, np.ndarray):
        raise ValueError(f"{name} must be a numpy array")
    if a.dtype != np.float32 or not a.flags.c_contiguous or not a.flags.writeable:
        raise ValueError(f"{name} must be a writeable C-contiguous float32 array")
    n = _n_field(h)
    if a.size != n:
        raise ValueError(f"{name} has {a.size} elements, expected {n}")
    return _ptr(a)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _coeffs(c):
    c = np.ascontiguousarray(c, dtype=np.float32)
    if c.size != 6:
        raise ValueError("coeffs must have 6 entries c0..c5")
    return c


# ---- north-star entry points ------------------------------------------------------------
def rtm_create(nx, ny, nz, dx, dt, coeffs):
    c = _coeffs(coeffs)
    h = lib.rtm_create(int(nx), int(ny), int(nz), float(dx), float(dt), _ptr(c))
    if not h:
        raise RtmError(RTM_EINVAL if "CUDA" not in _err() else RTM_ECUDA, _err())
    return h


def rtm_set_velocity(h, v):
    v = _f32(v, _n_velocity(h), "v")
    return _check(lib.rtm_set_velocity(h, _ptr(v)))


def rtm_inject_source(h, ix, iy, iz, samples):
    s = _f32(samples)
    return _check(lib.rtm_inject_source(h, int(ix), int(iy), int(iz), _ptr(s) if s.size else None,
                                        int(s.size)))


def rtm_step(h, nsteps):
    return _check(lib.rtm_step(h, int(nsteps)))


def rtm_read_field(h, out):
    return _check(lib.rtm_read_field(h, _out_buf(out, h, "out")))


def rtm_destroy(h):
    if h:
        lib.rtm_destroy(h)
        _barriers.pop(h, None)


def rtm_last_error() -> str:
    return _err()


# ---- extensions --------------------------------------------------------------------------
def rtm_set_fields(h, u=None, u_prev=None):
    n = _n_field(h)
    u = None if u is None else _f32(u, n, "u")
    up = None if u_prev is None else _f32(u_prev, n, "u_prev")
    return _check(lib.rtm_set_fields(h, _ptr(u), _ptr(up)))


def rtm_read_fields(h, u=None, u_prev=None):
    pu = None if u is None else _out_buf(u, h, "u")
    pp = None if u_prev is None else _out_buf(u_prev, h, "u_prev")
    return _check(lib.rtm_read_fields(h, pu, pp))


def rtm_reset(h):
    return _check(lib.rtm_reset(h))


def rtm_step_count(h) -> int:
    return int(lib.rtm_step_count(h))


def rtm_set_step_count(h, n):
    return _check(lib.rtm_set_step_count(h, int(n)))


def rtm_field_stats(h):
    m, bad = _D(0), _LL(0)
    _check(lib.rtm_field_stats(h, ctypes.byref(m), ctypes.byref(bad)))
    return float(m.value), int(bad.value)


def _async_buf(a, name, h, nfn, write=False):
    # no implicit conversion copy: the library reads/writes the caller's memory after return
    if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous
            and (a.flags.writeable or not write)):
        raise ValueError(f"{name} must be a C-contiguous float32 array"
                         + (" (writeable)" if write else ""))
    n = nfn(h)  # the context's extents (raises RtmError for a NULL context)
    if a.size != n:
        raise ValueError(f"{name} has {a.size} elements, expected {n}")
    return _ptr(a)


def rtm_blocksize_lattice(S, P) -> list[int]:
    """PAPER.md:296-301 candidate values for one dimension of size S divided in P parts."""
    out = (_I * max(int(P), 1))()
    n = lib.rtm_blocksize_lattice(int(S), int(P), out)
    if n < 0:
        raise RtmError(n, _err())
    return [int(out[k]) for k in range(n)]


def rtm_set_velocity_async(h, v):
    """v must stay alive and unmodified until rtm_sync (keep a reference)."""
    return _check(lib.rtm_set_velocity_async(h, _async_buf(v, "v", h, _n_velocity)))


def rtm_step_async(h, nsteps):
    return _check(lib.rtm_step_async(h, int(nsteps)))


def rtm_read_field_async(h, out):
    """out: a C-contiguous float32 array, filled once rtm_sync returns."""
    return _check(lib.rtm_read_field_async(h, _async_buf(out, "out", h, _n_field, write=True)))


def rtm_sync(h):
    return _check(lib.rtm_sync(h))


def rtm_set_velocity_device(h, dptr: int):
    return _check(lib.rtm_set_velocity_device(h, _P(int(dptr))))


def rtm_read_field_device(h, dptr: int):
    return _check(lib.rtm_read_field_device(h, _P(int(dptr))))


def rtm_set_tile(h, tile_id):
    return _check(lib.rtm_set_tile(h, int(tile_id)))


def rtm_get_tile(h) -> int:
    return int(lib.rtm_get_tile(h))


def rtm_num_tiles() -> int:
    return int(lib.rtm_num_tiles())


def rtm_tile_name(tile_id) -> str | None:
    n = lib.rtm_tile_name(int(tile_id))
    return n.decode() if n else None


def rtm_set_zchunk(h, planes):
    return _check(lib.rtm_set_zchunk(h, int(planes)))


def rtm_set_option(h, key, value):
    return _check(lib.rtm_set_option(h, int(key), int(value)))


def rtm_get_option(h, key) -> int:
    return int(lib.rtm_get_option(h, int(key)))


def rtm_set_stream(h, stream_handle):
    return _check(lib.rtm_set_stream(h, _P(int(stream_handle)) if stream_handle else None))


def rtm_last_elapsed_ms(h) -> float:
    return float(lib.rtm_last_elapsed_ms(h))


def rtm_set_profiling(h, on):
    return _check(lib.rtm_set_profiling(h, int(bool(on))))


def rtm_kernel_stats(h):
    n, ms = _LL(0), _D(0)
    _check(lib.rtm_kernel_stats(h, ctypes.byref(n), ctypes.byref(ms)))
    return int(n.value), float(ms.value)


def rtm_launch_count(h) -> int:
    return int(lib.rtm_launch_count(h))


def rtm_create_multi(nx, ny, nz, dx, dt, coeffs, devices):
    c = _coeffs(coeffs)
    d = np.ascontiguousarray(devices, dtype=np.int32)
    h = lib.rtm_create_multi(int(nx), int(ny), int(nz), float(dx), float(dt), _ptr(c), int(d.size),
                             _ptr(d))
    if not h:
        raise RtmError(RTM_EINVAL, _err())
    return h


def rtm_create_batch(nx, ny, nz, dx, dt, coeffs, nshots):
    c = _coeffs(coeffs)
    h = lib.rtm_create_batch(int(nx), int(ny), int(nz), float(dx), float(dt), _ptr(c), int(nshots))
    if not h:
        raise RtmError(RTM_EINVAL if "CUDA" not in _err() else RTM_ECUDA, _err())
    return h


def rtm_num_shots(h) -> int:
    return int(lib.rtm_num_shots(h))


def rtm_inject_source_shot(h, shot, ix, iy, iz, samples):
    s = _f32(samples)
    return _check(lib.rtm_inject_source_shot(h, int(shot), int(ix), int(iy), int(iz),
                                             _ptr(s) if s.size else None, int(s.size)))


def rtm_get_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(lib.rtm_get_unique_id(ctypes.cast(buf, _P)))
    return bytes(buf)


def rtm_create_dist(nx, ny, nz_global, dx, dt, coeffs, rank, world, uid: bytes, device):
    c = _coeffs(coeffs)
    if len(uid) != 128:
        raise ValueError("unique id must be 128 bytes")
    buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
    h = lib.rtm_create_dist(int(nx), int(ny), int(nz_global), float(dx), float(dt), _ptr(c),
                            int(rank), int(world), ctypes.cast(buf, _P), int(device))
    if not h:
        raise RtmError(RTM_ENCCL if "NCCL" in _err() else RTM_EINVAL, _err())
    return h


def rtm_slab_range(nz_global, world, rank):
    z0, nzl = _I(0), _I(0)
    _check(lib.rtm_slab_range(int(nz_global), int(world), int(rank), ctypes.byref(z0),
                              ctypes.byref(nzl)))
    return int(z0.value), int(nzl.value)


def rtm_halo_plan(nx, ny, nzl, rank, world):
    offs = (_LL * 4)()
    cnt = _LL(0)
    _check(lib.rtm_halo_plan(int(nx), int(ny), int(nzl), int(rank), int(world), offs,
                             ctypes.byref(cnt)))
    return [int(o) for o in offs], int(cnt.value)


def rtm_nu_crit(coeffs) -> float:
    return float(lib.rtm_nu_crit(_ptr(_coeffs(coeffs))))


def rtm_autotune(h, nI, tiles=None, zchunks=None):
    """Two-phase selection/verification tuner.  Returns (result dict,
    per-candidate selection times in ms)."""
    res = rtm_tune_result()
    if tiles is not None:
        t = np.ascontiguousarray(tiles, dtype=np.int32)
        z = np.ascontiguousarray(zchunks if zchunks is not None else np.zeros(len(t)), dtype=np.int32)
        n = len(t)
    else:
        t = z = None
        n = rtm_num_tiles()
    times = np.full(n, np.nan)
    _check(lib.rtm_autotune(h, int(nI), _ptr(t), _ptr(z), int(n if t is not None else 0),
                            ctypes.byref(res), _ptr(times)))
    d = {f: getattr(res, f) for f, _ in rtm_tune_result._fields_}
    return d, times[: res.ncandidates]


def rtm_select_mwmb(times) -> int:
    t = np.ascontiguousarray(times, dtype=np.float64)
    if t.ndim != 2:
        raise ValueError("times must be (nranks, ncand)")
    return int(lib.rtm_select_mwmb(_ptr(t), int(t.shape[0]), int(t.shape[1])))


# ---- peer contexts: CUDA-IPC data plane without NCCL -----------------------------------
def rtm_create_peer(nx, ny, nz_global, dx, dt, coeffs, rank, world, device):
    c = _coeffs(coeffs)
    h = lib.rtm_create_peer(int(nx), int(ny), int(nz_global), float(dx), float(dt), _ptr(c),
                            int(rank), int(world), int(device))
    if not h:
        raise RtmError(RTM_ECUDA if "CUDA" in _err() else RTM_EINVAL, _err())
    return h


def rtm_ipc_export(h) -> bytes:
    buf = (ctypes.c_ubyte * RTM_IPC_RECORD_BYTES)()
    _check(lib.rtm_ipc_export(h, ctypes.cast(buf, _P)))
    return bytes(buf)


def rtm_ipc_import(h, lo: bytes | None, hi: bytes | None):
    def arg(r, name):
        if r is None:
            return None, None
        if len(r) != RTM_IPC_RECORD_BYTES:
            raise ValueError(f"{name} record must be {RTM_IPC_RECORD_BYTES} bytes")
        b = (ctypes.c_ubyte * RTM_IPC_RECORD_BYTES).from_buffer_copy(r)
        return b, ctypes.cast(b, _P)
    bl, pl = arg(lo, "lo")
    bh, ph = arg(hi, "hi")
    return _check(lib.rtm_ipc_import(h, pl, ph))


def rtm_set_host_barrier(h, fn):
    """fn() -> None: returns once every rank called it (e.g. a gloo-group barrier); an
    exception inside it makes the calling library operation fail with RTM_ESTATE."""
    if fn is None:
        _barriers.pop(h, None)
        return _check(lib.rtm_set_host_barrier(h, None, None))

    def tramp(_user):
        try:
            fn()
            return 0
        except Exception:  # noqa: BLE001  (reported to the caller as RTM_ESTATE)
            return 1
    cb = BARRIER_FN(tramp)
    _barriers[h] = cb
    return _check(lib.rtm_set_host_barrier(h, ctypes.cast(cb, _P), None))


def rtm_last_enqueue_ms(h) -> float:
    return float(lib.rtm_last_enqueue_ms(h))
