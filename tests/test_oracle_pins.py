"""Pins for the CPU oracle (oracle/rtm_oracle.cpp) against things OTHER than itself:
exact rational arithmetic, closed forms, invariants and brute force (SURVEY.md §8(c)
P1-P13; DESIGN.md §"Oracle pins").  No GPU needed.

The paper (§2, Algorithm 1) prints no wavefield values, so the
wavefield is pinned by the mathematics of the scheme it names: a 10th-order central
second difference per axis (exact on polynomials of degree <= 11), 2nd-order leapfrog in
time (exact discrete dispersion relation, time reversibility, a conserved discrete energy).
Each test is chosen so a plausible mistake (dropped term, wrong sign, wrong index or
stride, transposed axes, wrong coefficient) fails at least one of them.
"""
from __future__ import annotations

import math
from fractions import Fraction as Fr
from pathlib import Path

import numpy as np
import pytest

import oracle
import rtm_inputs as ri

C_EX = ri.COEFFS_EXACT
C32 = ri.COEFFS_F32
C64 = ri.COEFFS_F64
DX, DT = 10.0, 1e-3


def v_for_nu(nu, shape, dtype=np.float64):
    """Velocity giving Courant number nu = v dt / dx at DX, DT."""
    return np.full(shape, nu * DX / DT, dtype)


# ---------------------------------------------------------------- P1 coefficients
def test_p1_coefficient_moments_exact():
    """sum_k c_k k^{2m}: 1 for m = 1, 0 for m = 2..5, and c0 + 2 sum c_k = 0 (exactness of
    the 10th-order central 2nd difference on polynomials of degree <= 11)."""
    c = C_EX
    assert c[0] + 2 * sum(c[1:]) == 0
    for m in range(1, 6):
        mom = sum(c[k] * Fr(k) ** (2 * m) for k in range(1, 6))
        assert mom == (1 if m == 1 else 0), m
    assert sum(c[k] * Fr(k) ** 12 for k in range(1, 6)) != 0  # degree 12 is not exact


def test_p1_f32_coefficients_are_nearest_rounding():
    assert C32.view(np.uint32)[0] == 0xC03B579C  # c0 = -2.9272223
    for q, f in zip(C_EX, C32):
        fr = Fr(float(f))
        for nb in (np.nextafter(f, np.float32(-1e30)), np.nextafter(f, np.float32(1e30))):
            assert abs(fr - q) <= abs(Fr(float(nb)) - q)


# ---------------------------------------------------------------- P12 zero fixed point
def test_p12_zero_fixed_point():
    v = v_for_nu(0.3, (12, 14, 16), np.float32)
    src = [(3, 4, 5, np.zeros(5, np.float32))]
    u = oracle.run(v, DX, DT, C32, 5, sources=src)
    assert not np.any(u)


# ---------------------------------------------------------------- P2 polynomial exactness
def _laplacian_through_step(u, dtype=np.float64):
    """u_prev = 2u and C = 1 give u^1 = 2u - 2u + 1 * L(u) = L(u) exactly."""
    nz, ny, nx = u.shape
    v = np.full(u.shape, DX / DT, dtype)  # nu = 1 -> C = 1 exactly
    return oracle.run(v, DX, DT, C64 if dtype == np.float64 else C32, 1,
                      u0=u.astype(dtype), up0=(2 * u).astype(dtype), dtype=dtype)


@pytest.mark.parametrize("deg", [(7, 0, 0), (0, 9, 0), (0, 0, 10), (2, 3, 4), (11, 1, 0)])
def test_p2_polynomial_exactness(deg):
    """L(xi^a eta^b zeta^c) equals the analytic Laplacian (in grid units) at every point
    >= 5 cells from the boundary, for per-axis degrees <= 11.  Non-cubic grid and distinct
    degrees per axis, so a swapped stride or axis fails."""
    nz, ny, nx = 18, 20, 24
    h = 8.0
    a, b, c = deg  # powers of x, y, z
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    xi, eta, ze = (x - 11.3) / h, (y - 9.6) / h, (z - 8.2) / h
    u = xi**a * eta**b * ze**c
    d2 = lambda t, p: p * (p - 1) * t ** max(p - 2, 0) / h**2 if p >= 2 else 0 * t  # noqa: E731
    lap = d2(xi, a) * eta**b * ze**c + xi**a * d2(eta, b) * ze**c + xi**a * eta**b * d2(ze, c)
    L = _laplacian_through_step(u)
    s = (slice(5, -5),) * 3
    err = np.abs(L[s] - lap[s]).max()
    scale = max(np.abs(lap[s]).max(), np.abs(u[s]).max() / h**2)
    assert err <= 1e-11 * scale, (err, scale)


def test_p2_degree12_is_not_exact():
    """Sensitivity check: xi^12 at xi = 0 gives 2 sum_k c_k k^12 / h^12, not 0."""
    n = 24
    h = 2.0
    x = np.arange(n, dtype=np.float64)
    u = np.broadcast_to(((x - 12) / h) ** 12, (n, n, n)).copy()
    L = _laplacian_through_step(u)
    expect = float(2 * sum(C_EX[k] * Fr(k) ** 12 for k in range(1, 6))) / h**12
    assert L[12, 12, 12] == pytest.approx(expect, rel=1e-9)
    assert expect != 0


# ---------------------------------------------------------------- P3 null space
def test_p3_constant_and_linear_fields_fp64():
    nz, ny, nx = 16, 18, 20
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    for u in (np.full((nz, ny, nx), 3.7), 0.5 + 0.1 * x - 0.2 * y + 0.3 * z):
        v = v_for_nu(0.4, u.shape)
        out = oracle.run(v, DX, DT, C64, 1, u0=u, up0=u, dtype=np.float64)
        s = (slice(5, -5),) * 3
        assert np.abs(out[s] - u[s]).max() <= 1e-13 * np.abs(u).max()
        # ... while next to the boundary the zero halo must show (sign: L < 0 for u > 0)
        if np.all(u > 0):
            assert np.all(out[0] < u[0])


def test_p3_constant_field_fp32_spec_example():
    """a constant field is invariant >= 5 cells from the boundary.  In fp32 the
    rounded coefficients leave c0 + 2 sum c_k ~ -1e-7 per axis, so tolerance 1e-6 |u|."""
    u = np.full((16, 16, 16), 2.5, np.float32)
    out = oracle.run(v_for_nu(1.0, u.shape, np.float32), DX, DT, C32, 1, u0=u, up0=u)
    s = (slice(5, -5),) * 3
    assert np.abs(out[s] - 2.5).max() <= 1e-6 * 2.5


# ---------------------------------------------------------------- P4 brute force
def _star_kernel(c):
    K = np.zeros((11, 11, 11))
    for o in range(-5, 6):
        K[5 + o, 5, 5] += float(c[abs(o)])
        K[5, 5 + o, 5] += float(c[abs(o)])
        K[5, 5, 5 + o] += float(c[abs(o)])
    return K


def brute_force_run(v, dx, dt, u0, up0, sources, steps):
    """Independent fp64 reference: dense 11x11x11 convolution (star embedded, centre 3 c0)
    over a zero-padded copy, written as a plain loop over the 1331 kernel taps."""
    K = _star_kernel(C_EX)
    Cf = (v.astype(np.float64) * dt / dx) ** 2
    u, up = u0.astype(np.float64).copy(), up0.astype(np.float64).copy()
    nz, ny, nx = u.shape
    for n in range(steps):
        pad = np.zeros((nz + 10, ny + 10, nx + 10))
        pad[5:-5, 5:-5, 5:-5] = u
        acc = np.zeros_like(u)
        for a in range(11):
            for b in range(11):
                for c in range(11):
                    if K[a, b, c] != 0.0:
                        acc += K[a, b, c] * pad[a:a + nz, b:b + ny, c:c + nx]
        nxt = 2 * u - up + Cf * acc
        for (x, y, z, w) in sources:
            if n < len(w):
                nxt[z, y, x] += float(w[n])
        up, u = u, nxt
    return u


def test_p4_brute_force_fp64_and_fp32():
    nz, ny, nx = 12, 14, 16
    rng = np.random.default_rng(4)
    u0 = rng.uniform(-1, 1, (nz, ny, nx))
    up0 = rng.uniform(-1, 1, (nz, ny, nx))
    v = rng.uniform(1500, 4400, (nz, ny, nx))
    w = rng.uniform(-1, 1, 4)
    src = [(3, 7, 9, w), (10, 2, 1, -w)]
    ref = brute_force_run(v, DX, DT, u0, up0, src, 4)
    got64 = oracle.run(v, DX, DT, C64, 4, u0=u0, up0=up0, sources=src, dtype=np.float64)
    assert np.abs(got64 - ref).max() <= 1e-12 * np.abs(ref).max()
    got32 = oracle.run(v.astype(np.float32), DX, DT, C32, 4, u0=u0.astype(np.float32),
                       up0=up0.astype(np.float32),
                       sources=[(x, y, z, ww.astype(np.float32)) for x, y, z, ww in src])
    assert np.abs(got32 - ref).max() <= 1e-5 * np.abs(ref).max()


def test_p4_spec_delta_on_32cube():
    """a centred delta on 32^3, one step, equals the direct summation."""
    n = 32
    u0 = np.zeros((n, n, n))
    u0[16, 16, 16] = 1.0
    v = v_for_nu(0.2, u0.shape)
    ref = brute_force_run(v, DX, DT, u0, np.zeros_like(u0), [], 1)
    got = oracle.run(v, DX, DT, C64, 1, u0=u0, dtype=np.float64)
    assert np.abs(got - ref).max() <= 1e-15


# ---------------------------------------------------------------- P13 exact delta response
def _golden_delta():
    path = Path(__file__).parent / "golden" / "delta_response_c1.txt"
    rows = []
    for line in path.read_text().splitlines():
        if line.startswith("#"):
            continue
        n, dz, dy, dx, num, den, _ = line.split()
        rows.append((int(n), int(dz), int(dy), int(dx), Fr(int(num), int(den))))
    return rows


def test_p13_golden_file_is_reproducible():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "mk", Path(__file__).parent / "golden" / "make_delta_response.py")
    mk = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mk)
    hist = mk.evolve(3)
    assert [len(h) for h in hist] == [31, 361, 1991]
    for n, dz, dy, dx, val in _golden_delta():
        assert hist[n - 1].get((dz, dy, dx), Fr(0)) == val


def test_p13_closed_form_first_step():
    """u^1 = 2 delta + nu^2 L delta: centre 2 + 3 c0 / 25, axis offsets c_m / 25."""
    g = {(n, dz, dy, dx): v for n, dz, dy, dx, v in _golden_delta()}
    assert g[(1, 0, 0, 0)] == 2 + 3 * C_EX[0] / 25 == Fr(24731, 15000)
    assert g[(1, 1, 0, 0)] == C_EX[1] / 25
    assert g[(1, 5, 0, 0)] == C_EX[5] / 25
    assert g[(1, 6, 0, 0)] == 0 and g[(1, 1, 1, 0)] == 0


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-14), (np.float32, 3e-7)])
def test_p13_oracle_matches_exact_delta_response(dtype, tol):
    n = 64  # C1's grid; delta at index 32 (R9), C = (2000*1e-3/10)^2 = 1/25
    u0 = np.zeros((n, n, n), dtype)
    u0[32, 32, 32] = 1
    v = np.full((n, n, n), 2000.0, dtype)
    c = C64 if dtype == np.float64 else C32
    for steps in (1, 2, 3):
        out = oracle.run(v, DX, DT, c, steps, u0=u0, dtype=dtype, nthreads=4)
        for st, dz, dy, dx, val in _golden_delta():
            if st == steps:
                assert abs(float(out[32 + dz, 32 + dy, 32 + dx]) - float(val)) <= tol, (st, dz, dy, dx)
        assert np.count_nonzero(out) <= [31, 361, 1991][steps - 1]


# ---------------------------------------------------------------- P5 plane-wave dispersion
def symbol_S(theta):
    """S(theta) = -(c0 + 2 sum_m c_m cos(m theta)) (Fourier symbol of -L per axis)."""
    return -(C64[0] + 2 * sum(C64[m] * math.cos(m * theta) for m in range(1, 6)))


def omega_dt(nu, thetas):
    """Discrete leapfrog dispersion: sin^2(w dt / 2) = nu^2/4 * sum_a S(theta_a)."""
    return 2 * math.asin(math.sqrt(nu**2 / 4 * sum(symbol_S(t) for t in thetas)))


def test_p5_dispersion_formula_references():
    # SURVEY.md §8(c) P5 cross-check values, and the continuum limit w = nu |theta|
    assert omega_dt(0.3, (0.7, 0.5, 0.3)) == pytest.approx(0.274170802, abs=1e-9)
    assert omega_dt(0.2, (math.pi / 4, 0, 0)) == pytest.approx(0.157241223, abs=1e-9)
    th = (0.02, 0.013, 0.007)
    cont = 0.25 * math.sqrt(sum(t * t for t in th))
    assert omega_dt(0.25, th) == pytest.approx(cont, rel=1e-5)
    assert symbol_S(math.pi) == pytest.approx(512 / 75, rel=1e-14)  # Nyquist symbol


@pytest.mark.parametrize("nu,th", [(0.3, (0.7, 0.5, 0.3)), (0.2, (math.pi / 4, 0.0, 0.0)),
                                   (0.43, (0.2, 1.1, 2.4))])
def test_p5_plane_wave_is_exact(nu, th):
    """u^0 = cos(theta.p), u^-1 = cos(theta.p + W) -> u^n = cos(theta.p - n W) exactly at
    points >= 5 n cells from the boundary (domain of dependence avoids the halo)."""
    nz, ny, nx = 36, 38, 40
    steps = 3
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ph = th[0] * x + th[1] * y + th[2] * z
    W = omega_dt(nu, th)
    u0, um1 = np.cos(ph), np.cos(ph + W)
    out = oracle.run(v_for_nu(nu, u0.shape), DX, DT, C64, steps, u0=u0, up0=um1,
                     dtype=np.float64)
    s = (slice(5 * steps, -5 * steps),) * 3
    assert np.abs(out[s] - np.cos(ph - steps * W)[s]).max() <= 1e-12
    # a wrong frequency (continuum instead of discrete) is detectably different
    Wc = nu * math.sqrt(sum(t * t for t in th))
    assert np.abs(out[s] - np.cos(ph - steps * Wc)[s]).max() > 1e-6


# ---------------------------------------------------------------- P6 symmetry
def test_p6_mirror_and_permutation_symmetry_fp64():
    n = 65
    v = v_for_nu(0.2, (n, n, n))
    w = ri.source_samples(2000.0, DT, 15.0, 40).astype(np.float64)
    out = oracle.run(v, DX, DT, C64, 40, sources=[(32, 32, 32, w)], dtype=np.float64)
    m = np.abs(out).max()
    assert m > 0
    for ax in range(3):
        assert np.abs(out - np.flip(out, axis=ax)).max() <= 1e-12 * m
    assert np.abs(out - out.transpose(1, 0, 2)).max() <= 1e-12 * m
    assert np.abs(out - out.transpose(2, 1, 0)).max() <= 1e-12 * m


def test_p6_off_centre_source_breaks_symmetry():
    """Sensitivity: on a non-cubic grid an off-centre source is not mirror-symmetric, and
    its field is centred on the source (peak |u| adjacent to it)."""
    v = v_for_nu(0.2, (20, 24, 28))
    w = np.ones(3)
    out = oracle.run(v, DX, DT, C64, 3, sources=[(9, 11, 7, w)], dtype=np.float64)
    assert np.unravel_index(np.abs(out).argmax(), out.shape) == (7, 11, 9)
    assert np.abs(out - np.flip(out, axis=2)).max() > 1e-3


# ---------------------------------------------------------------- P7 energy
def _L_np(u):
    nz, ny, nx = u.shape
    pad = np.zeros((nz + 10, ny + 10, nx + 10))
    pad[5:-5, 5:-5, 5:-5] = u
    acc = np.zeros_like(u)
    for o in range(-5, 6):
        c = C64[abs(o)]
        acc += c * pad[5 + o:5 + o + nz, 5:5 + ny, 5:5 + nx]
        acc += c * pad[5:5 + nz, 5 + o:5 + o + ny, 5:5 + nx]
        acc += c * pad[5:5 + nz, 5:5 + ny, 5 + o:5 + o + nx]
    return acc


def test_p7_discrete_energy_conserved_fp64():
    """E^{n+1/2} = sum (u^{n+1}-u^n)^2 / C - sum u^{n+1} L u^n is invariant (L symmetric
    with the zero halo, leapfrog), with variable C and no source."""
    shape = (14, 16, 18)
    rng = np.random.default_rng(7)
    v = rng.uniform(1500, 4300, shape)
    Cf = (v * DT / DX) ** 2
    u, up = rng.uniform(-1, 1, shape), rng.uniform(-1, 1, shape)
    E = []
    for _ in range(60):
        nxt = oracle.run(v, DX, DT, C64, 1, u0=u, up0=up, dtype=np.float64)
        E.append(np.sum((nxt - u) ** 2 / Cf) - np.sum(nxt * _L_np(u)))
        up, u = u, nxt
    E = np.array(E)
    assert E[0] > 0
    assert np.abs(E - E[0]).max() <= 1e-10 * E[0]


# ---------------------------------------------------------------- P8 reversibility
def test_p8_time_reversibility_fp64():
    shape = (16, 14, 18)
    rng = np.random.default_rng(8)
    v = rng.uniform(1500, 4300, shape)
    u0, up0 = rng.uniform(-1, 1, shape), rng.uniform(-1, 1, shape)
    uN, uNm1 = oracle.run(v, DX, DT, C64, 30, u0=u0, up0=up0, dtype=np.float64, return_prev=True)
    back, back_prev = oracle.run(v, DX, DT, C64, 30, u0=uNm1, up0=uN, dtype=np.float64,
                                 return_prev=True)
    assert np.abs(back - up0).max() <= 1e-10
    assert np.abs(back_prev - u0).max() <= 1e-10


# ---------------------------------------------------------------- P9 linearity
def test_p9_linearity_and_superposition():
    shape = (20, 22, 24)
    v = np.full(shape, 3000.0, np.float32)
    w = ri.source_samples(3000.0, DT, 15.0, 30)
    s1, s2 = (5, 6, 7), (15, 14, 12)
    a = oracle.run(v, DX, DT, C32, 30, sources=[(*s1, w)])
    a2 = oracle.run(v, DX, DT, C32, 30, sources=[(*s1, 2 * w)])
    assert np.array_equal(a2, 2 * a)  # scaling by 2 is exact in binary floating point
    b = oracle.run(v, DX, DT, C32, 30, sources=[(*s2, -0.5 * w)])
    ab = oracle.run(v, DX, DT, C32, 30, sources=[(*s1, w), (*s2, -0.5 * w)])
    assert np.abs(ab - (a + b)).max() <= 1e-5 * np.abs(ab).max()


def test_p9_sources_at_same_point_add_in_order():
    shape = (12, 12, 12)
    v = np.full(shape, 2000.0, np.float32)
    w = ri.source_samples(2000.0, DT, 15.0, 10)
    a = oracle.run(v, DX, DT, C32, 10, sources=[(5, 5, 5, w), (5, 5, 5, w)])
    b = oracle.run(v, DX, DT, C32, 10, sources=[(5, 5, 5, 2 * w)])
    assert np.abs(a - b).max() <= 1e-6 * np.abs(b).max()
    # sample n is injected after step n: one step from rest gives exactly w[0] at the source
    c1 = oracle.run(v, DX, DT, C32, 1, sources=[(5, 5, 5, w)])
    assert c1[5, 5, 5] == w[0] and np.count_nonzero(c1) == 1


# ---------------------------------------------------------------- P10 CFL
@pytest.mark.parametrize("factor,explodes", [(1.02, True), (0.99, False)])
def test_p10_cfl_bound(factor, explodes):
    shape = (32, 32, 32)
    rng = np.random.default_rng(10)
    u0, up0 = rng.uniform(-1, 1, shape), rng.uniform(-1, 1, shape)
    v = v_for_nu(factor * ri.NU_CRIT, shape)
    out = oracle.run(v, DX, DT, C64, 120, u0=u0, up0=up0, dtype=np.float64)
    if explodes:
        assert np.abs(out).max() > 1e6
    else:
        assert np.abs(out).max() < 20


# ---------------------------------------------------------------- P11 traversal invariance
def test_p11_thread_count_invariance_bitwise():
    cfg = ri.make_config(2, shape=(40, 36, 32), steps=25)
    v = cfg.velocity()
    u0, up0 = ri.random_fields(v.shape, seed=11)
    a = oracle.run(v, cfg.dx, cfg.dt, C32, 25, u0=u0, up0=up0, sources=cfg.sources(), nthreads=1)
    b = oracle.run(v, cfg.dx, cfg.dt, C32, 25, u0=u0, up0=up0, sources=cfg.sources(), nthreads=5)
    assert np.array_equal(a, b)


def test_p11_slab_simulator_equals_unsplit_bitwise():
    """CPU slab simulator: G z-slabs with explicit 5-plane halo copies equal
    the unsplit oracle bitwise (same per-point expression, exact copies)."""
    cfg = ri.make_config(3, shape=(30, 20, 24), steps=12)
    v = cfg.velocity()
    nz, ny, nx = v.shape
    u0, up0 = ri.random_fields(v.shape, seed=12)
    srcs = cfg.sources() + [(3, 4, 9, cfg.sources()[0][3])]  # one source right at a slab edge
    ref = oracle.run(v, cfg.dx, cfg.dt, C32, 12, u0=u0, up0=up0, sources=srcs)
    G = 3
    bounds = [(r * nz // G, (r + 1) * nz // G) for r in range(G)]
    slabs = []
    for z0, z1 in bounds:
        nzl = z1 - z0
        U = np.zeros((nzl + 10, ny, nx), np.float32)
        P = np.zeros_like(U)
        U[5:5 + nzl] = u0[z0:z1]
        P[5:5 + nzl] = up0[z0:z1]
        slabs.append([U, P, oracle.cfield_f32(v[z0:z1], cfg.dx, cfg.dt), z0, nzl])

    def exchange():
        for r in range(G):
            U, _, _, _, nzl = slabs[r]
            if r > 0:
                U[0:5] = slabs[r - 1][0][slabs[r - 1][4]:slabs[r - 1][4] + 5]
            if r < G - 1:
                U[nzl + 5:nzl + 10] = slabs[r + 1][0][5:10]

    exchange()
    for n in range(12):
        for s in slabs:
            U, P, C, z0, nzl = s
            oracle.slab_step_f32(C32, C, U, P)
            for (x, y, z, w) in srcs:
                if z0 <= z < z0 + nzl and n < len(w):
                    P[z - z0 + 5, y, x] = np.float32(P[z - z0 + 5, y, x] + w[n])
            s[0], s[1] = P, U
        exchange()
    got = np.concatenate([s[0][5:5 + s[4]] for s in slabs])
    assert np.array_equal(got, ref)


def test_points_function_matches_run():
    cfg = ri.make_config(4, shape=(24, 28, 32), steps=1)
    v = cfg.velocity()
    u0, up0 = ri.random_fields(v.shape, seed=13)
    ref = oracle.run(v, cfg.dx, cfg.dt, C32, 1, u0=u0, up0=up0)
    rng = np.random.default_rng(0)
    pts = np.stack([rng.integers(0, 32, 500), rng.integers(0, 28, 500), rng.integers(0, 24, 500)], 1)
    pts[:4] = [[0, 0, 0], [31, 27, 23], [0, 27, 0], [31, 0, 23]]
    got = oracle.points_f32(v, cfg.dx, cfg.dt, C32, u0, up0, pts)
    assert np.array_equal(got, ref[pts[:, 2], pts[:, 1], pts[:, 0]])
