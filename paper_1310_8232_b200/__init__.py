"""B200-native RTM 3D-model time step (arxiv 1310.8232, §2).

The product is the C-ABI library ``librtm_b200.so`` (include/rtm.h): sm_100a kernels for the
radius-5 31-point star + leapfrog + fused source injection, z-slab decomposition with
NCCL halo exchange.  ``paper_1310_8232_b200.rtm`` is the ctypes binding (same names as the
C entry points); :class:`Simulation` is a small convenience wrapper over those calls.
"""
from __future__ import annotations

import numpy as np

from . import rtm as _r
from .rtm import *  # noqa: F401,F403  (the binding: rtm_* functions, RtmError, RTM_* codes)
from .rtm import RtmError

__all__ = ["Simulation", "RtmError"] + [n for n in dir(_r) if n.startswith(("rtm_", "RTM_"))]


class Simulation:
    """Owns one rtm_ctx.  Arrays are float32 (nz, ny, nx)."""

    def __init__(self, nx, ny, nz, dx, dt, coeffs, *, devices=None, dist=None, shots=1):
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.dist = dist
        self.shots = int(shots)
        if self.shots > 1:  # batched independent wavefields on one velocity model
            self.h = _r.rtm_create_batch(nx, ny, nz, dx, dt, coeffs, self.shots)
            self.z0, self.nzl = 0, self.nz
        elif dist is not None:  # (rank, world, uid, device)
            rank, world, uid, device = dist
            self.h = _r.rtm_create_dist(nx, ny, nz, dx, dt, coeffs, rank, world, uid, device)
            self.z0, self.nzl = _r.rtm_slab_range(nz, world, rank)
        elif devices is not None and len(devices) > 1:
            self.h = _r.rtm_create_multi(nx, ny, nz, dx, dt, coeffs, devices)
            self.z0, self.nzl = 0, self.nz
        else:
            self.h = _r.rtm_create(nx, ny, nz, dx, dt, coeffs)
            self.z0, self.nzl = 0, self.nz

    @property
    def local_shape(self):
        if self.shots > 1:
            return (self.shots, self.nzl, self.ny, self.nx)
        return (self.nzl, self.ny, self.nx)

    def set_velocity(self, v):
        _r.rtm_set_velocity(self.h, v)

    def inject_source(self, ix, iy, iz, samples, shot=0):
        _r.rtm_inject_source_shot(self.h, shot, ix, iy, iz, samples)

    def set_fields(self, u=None, u_prev=None):
        _r.rtm_set_fields(self.h, u, u_prev)

    def step(self, n=1):
        _r.rtm_step(self.h, n)

    def read_field(self):
        out = np.empty(self.local_shape, np.float32)
        _r.rtm_read_field(self.h, out)
        return out

    def read_fields(self):
        u = np.empty(self.local_shape, np.float32)
        up = np.empty(self.local_shape, np.float32)
        _r.rtm_read_fields(self.h, u, up)
        return u, up

    def reset(self):
        _r.rtm_reset(self.h)

    def set_tile(self, tile_id):
        _r.rtm_set_tile(self.h, tile_id)

    @property
    def tile(self):
        return _r.rtm_get_tile(self.h)

    @property
    def steps_taken(self):
        return _r.rtm_step_count(self.h)

    @property
    def last_elapsed_ms(self):
        return _r.rtm_last_elapsed_ms(self.h)

    def close(self):
        if getattr(self, "h", None):
            _r.rtm_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
