"""Seeded synthetic inputs for the RTM 3D-model step — shared by tests, smoke and bench.

This module holds NO arithmetic of the method (no stencil, no C(p), no update, no
injection).  It only produces the *inputs* both sides consume: the FD coefficients
(BASELINE.json configs[0]), velocity models, source positions and source sample tables
(Ricker wavelets, pre-scaled on the host as DESIGN.md reading R4 states), and random
initial conditions.  Recipes are the readings R5, R8, R10-R12 of DESIGN.md.

The paper's own workloads are private per-process RTM grids (PAPER.md:186, PAPER.md:480,
200x200x800 .. 250x250x1500, 448 steps) with a Petrobras velocity model we do not have;
the five configs of BASELINE.json stand in for them (synthetic, seeded).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

# ---------------------------------------------------------------------------------------
# FD coefficients: standard 10th-order central 2nd-derivative weights (BASELINE.json
# configs[0]; "design decisions"; the paper is silent, R1).
COEFFS_EXACT = (Fraction(-5269, 1800), Fraction(5, 3), Fraction(-5, 21), Fraction(5, 126),
                Fraction(-5, 1008), Fraction(1, 3150))


def _nearest_f32(q: Fraction) -> np.float32:
    f = np.float32(float(q))
    cands = [np.nextafter(f, np.float32(-np.inf)), f, np.nextafter(f, np.float32(np.inf))]
    return min(cands, key=lambda c: abs(Fraction(float(c)) - q))


COEFFS_F32 = np.array([_nearest_f32(c) for c in COEFFS_EXACT], dtype=np.float32)
COEFFS_F64 = np.array([float(c) for c in COEFFS_EXACT], dtype=np.float64)

# Stability bound of the 3D leapfrog with these coefficients, nu_crit = 5/sqrt(128)
# (R8).  Used by the generators only to draw CFL-safe layers.
NU_CRIT = 5.0 / math.sqrt(128.0)

SEED_BASE = 13108232  # numpy.random.default_rng([SEED_BASE, k]) for config k


def rng_for(k: int, *extra: int) -> np.random.Generator:
    return np.random.default_rng([SEED_BASE, int(k), *[int(e) for e in extra]])


# ---------------------------------------------------------------------------------------
def ricker(t: np.ndarray, f0: float, t0: float | None = None) -> np.ndarray:
    """Ricker wavelet (1 - 2a) e^{-a}, a = (pi f0 (t - t0))^2, t0 = 1/f0 (R5)."""
    if t0 is None:
        t0 = 1.0 / f0
    a = (math.pi * f0 * (np.asarray(t, np.float64) - t0)) ** 2
    return (1.0 - 2.0 * a) * np.exp(-a)


def source_samples(v_s: float, dt: float, f0: float, nsteps: int) -> np.ndarray:
    """w[n] = fp32((v_s dt)^2 ricker(n dt)), computed in fp64 (R4).  Both the library and
    the oracle add these fp32 samples as-is after step n."""
    n = np.arange(nsteps, dtype=np.float64)
    return ((float(v_s) * float(dt)) ** 2 * ricker(n * float(dt), f0)).astype(np.float32)


def random_fields(shape, seed: int = 0, scale: float = 1.0):
    """Seeded U[-scale, scale] initial conditions (u, u_prev), fp32."""
    g = np.random.default_rng([SEED_BASE, 1000, int(seed)])
    out = []
    for _ in range(2):  # float32 draws (no float64 temporaries at 1024^3)
        a = g.random(size=shape, dtype=np.float32)
        a *= np.float32(2 * scale)
        a -= np.float32(scale)
        out.append(a)
    return out[0], out[1]


# ---------------------------------------------------------------------------------------
# Velocity models (R10, R11).  All return float32 arrays of shape (nz, ny, nx).
def layered_velocity(shape, layers: np.ndarray) -> np.ndarray:
    """6 equal horizontal layers along z: layer(z) = floor(6 z / nz) (R10)."""
    nz, ny, nx = shape
    nl = len(layers)
    z = np.arange(nz)
    lz = (nl * z) // nz
    col = np.asarray(layers, np.float32)[lz]
    return np.broadcast_to(col[:, None, None], shape).astype(np.float32)


def draw_layers(rng: np.random.Generator, dx: float, dt: float, n: int = 6):
    """Draw n layer velocities U[1500, 4500]; redraw the whole vector until
    max v <= 0.98 * nu_crit * dx / dt (R8).  Returns (layers, draws)."""
    vlim = 0.98 * NU_CRIT * dx / dt
    draws = 0
    while True:
        draws += 1
        lay = rng.uniform(1500.0, 4500.0, n)
        if lay.max() <= vlim:
            return lay.astype(np.float32), draws


def gaussian_filter_fine(a: np.ndarray, sigma: float = 8.0, truncate: float = 4.0) -> np.ndarray:
    """The config text's ``gaussian_filter(noise, sigma=8, mode='reflect', truncate=4.0)`` on
    the fine grid (R11): a separable Gaussian of radius int(truncate*sigma + 0.5) = 32 cells
    along axes 0, 1, 2 in turn, each output the weighted sum of the 65 reflected neighbours
    (scipy's 'reflect' = symmetric extension, repeated for axes shorter than the radius).
    Evaluated with torch shifted multiply-adds in fp32 — on the GPU when one is present (a
    2e9-point C5 field in about a second), else on the CPU (test-sized grids).  Input
    generation only: no arithmetic of the method."""
    import torch
    dev = torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")
    r = int(truncate * float(sigma) + 0.5)
    x = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (x / float(sigma)) ** 2)
    w /= w.sum()
    t = torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev)
    for axis in range(t.ndim):
        n = t.shape[axis]
        i = np.arange(-r, n + r)
        j = np.mod(i, 2 * n)
        j = np.where(j >= n, 2 * n - 1 - j, j)
        p = torch.index_select(t, axis, torch.from_numpy(j).to(dev))
        del t
        out = torch.zeros_like(p.narrow(axis, 0, n))
        for k in range(2 * r + 1):
            out.add_(p.narrow(axis, k, n), alpha=float(w[k]))
        del p
        t = out
    res = t.cpu().numpy()
    del t
    if dev.type == "cuda":
        torch.cuda.empty_cache()
    return res


def smooth_noise(rng: np.random.Generator, shape, sigma: int = 8) -> np.ndarray:
    """R11: seeded i.i.d. N(0, 1) fp32 noise on the fine grid, Gaussian-filtered (sigma cells)."""
    return gaussian_filter_fine(rng.standard_normal(shape, dtype=np.float32), sigma=sigma)


def smooth_velocity(rng, shape, vmin=1500.0, vmax=4500.0, sigma=8, nz_generate=None):
    """C3/C5: smooth random field scaled affinely to [vmin, vmax] (R11).  For C5 the field
    is defined on the G=8 grid (nz_generate planes) and the first shape[0] planes are kept;
    min/max are taken over the full generated field."""
    nz, ny, nx = shape
    nzg = nz if nz_generate is None else nz_generate
    s = smooth_noise(rng, (nzg, ny, nx), sigma)
    lo, hi = float(s.min()), float(s.max())
    out = np.ascontiguousarray(s[:nz])
    del s
    scale = np.float32((vmax - vmin) / (hi - lo))
    out -= np.float32(lo)
    out *= scale
    out += np.float32(vmin)
    np.clip(out, vmin, vmax, out=out)
    return out


def layered_smooth_velocity(rng, shape, dx, dt, sigma=8, amp=300.0):
    """C4: clip(layered(z) + amp * s / std(s), 1500, 4500) (R11)."""
    layers, _ = draw_layers(rng, dx, dt)
    nz, ny, nx = shape
    s = smooth_noise(rng, shape, sigma)
    s1 = s2 = 0.0
    for q in s.reshape(nz, -1):  # std over the whole field in fp64 (two moments, per plane)
        s1 += float(q.sum(dtype=np.float64))
        s2 += float(np.dot(q.astype(np.float64), q.astype(np.float64)))
    n = float(nz) * ny * nx
    std = math.sqrt(max(s2 / n - (s1 / n) ** 2, 1e-30))
    s *= np.float32(amp / std)
    lz = (len(layers) * np.arange(nz)) // nz
    s += layers[lz][:, None, None]
    np.clip(s, 1500.0, 4500.0, out=s)
    return s


# ---------------------------------------------------------------------------------------
@dataclass
class Config:
    """One BASELINE.json config (possibly resized for tests)."""
    k: int
    nx: int
    ny: int
    nz: int
    dx: float
    dt: float
    f0: float
    steps: int
    G: int = 1
    sources_xyz: list = field(default_factory=list)   # global (x, y, z) interior coords
    notes: str = ""
    _v: np.ndarray | None = None
    _vfn: object = None

    @property
    def shape(self):
        return (self.nz, self.ny, self.nx)

    @property
    def points(self) -> int:
        return self.nx * self.ny * self.nz

    def velocity(self) -> np.ndarray:
        if self._v is None:
            self._v = self._vfn()
        return self._v

    def sources(self, v: np.ndarray | None = None):
        """[(x, y, z, samples fp32[steps])] with per-source (v_s dt)^2 scaling (R4, R12)."""
        v = self.velocity() if v is None else v
        return [(x, y, z, source_samples(float(v[z, y, x]), self.dt, self.f0, self.steps))
                for (x, y, z) in self.sources_xyz]

    def describe(self) -> dict:
        return {"config": f"C{self.k}", "grid": [self.nx, self.ny, self.nz], "G": self.G,
                "dx": self.dx, "dt": self.dt, "f0": self.f0, "steps": self.steps,
                "sources": len(self.sources_xyz), "notes": self.notes}


def make_config(k: int, G: int = 1, shape=None, steps=None) -> Config:
    """BASELINE.json configs[k-1] (k = 1..5).  ``shape`` = (nz, ny, nx) resizes the grid for
    small tests while keeping the recipe (source positions are scaled proportionally)."""
    dx = 10.0
    if k == 1:
        n = (64, 64, 64)
        dt, f0, st = 1e-3, 15.0, 100
    elif k == 2:
        n = (256, 256, 256)
        dt, f0, st = 1e-3, 15.0, 500
    elif k == 3:
        n = (512, 512, 512)
        dt, f0, st = 0.8e-3, 20.0, 200
    elif k == 4:
        n = (1024, 1024, 1024)
        dt, f0, st = 0.8e-3, 15.0, 100
    elif k == 5:
        n = (256 * G, 1024, 1024)
        dt, f0, st = 0.8e-3, 15.0, 100
    else:
        raise ValueError(f"unknown config {k}")
    full = n
    if shape is not None:
        n = tuple(int(s) for s in shape)
    nz, ny, nx = n
    steps = st if steps is None else int(steps)
    sx = lambda a, ax: int(round(a * n[ax] / full[ax]))  # noqa: E731
    rng = rng_for(k)
    if k == 1:
        srcs = [(nx // 2, ny // 2, nz // 2)]                               # R9
        vfn = lambda: np.full(n, 2000.0, np.float32)                       # noqa: E731
        notes = "constant 2000 m/s"
    elif k == 2:
        layers, draws = draw_layers(rng, dx, dt)
        srcs = [(nx // 2, ny // 2, min(nz - 1, sx(20, 0)))]                # depth 20 cells (R12)
        vfn = lambda: layered_velocity(n, layers)                          # noqa: E731
        notes = f"6 layers {np.round(layers, 1).tolist()} ({draws} draws)"
    elif k == 3:
        srcs = [(nx // 2, ny // 2, nz // 2)]
        vfn = lambda: smooth_velocity(rng_for(3, 1), n)                    # noqa: E731
        notes = "smooth random: N(0,1) noise, Gaussian sigma=8 cells, scaled to [1500, 4500]"
    elif k == 4:
        jr = rng_for(4, 2)
        srcs = []
        for j in range(4):
            for i in range(4):
                jx, jy = (int(t) for t in jr.integers(-32, 33, 2))
                x = min(nx - 1, max(0, (2 * i + 1) * nx // 8 + sx(jx, 2)))
                y = min(ny - 1, max(0, (2 * j + 1) * ny // 8 + sx(jy, 1)))
                srcs.append((x, y, min(nz - 1, sx(10, 0))))
        vfn = lambda: layered_smooth_velocity(rng_for(4, 1), n, dx, dt)   # noqa: E731
        notes = "layered + smooth noise, 16 shots at z=10"
    else:
        srcs = [(nx // 2, ny // 2, min(nz - 1, sx(20, 0)))]
        nzg = (n[0] // G) * 8 if shape is None else None
        vfn = lambda: smooth_velocity(rng_for(5, 1), n, nz_generate=nzg)  # noqa: E731
        notes = "weak scaling, smooth random defined on the G=8 grid"
    return Config(k=k, nx=nx, ny=ny, nz=nz, dx=dx, dt=dt, f0=f0, steps=steps, G=G,
                  sources_xyz=srcs, notes=notes, _vfn=vfn)
