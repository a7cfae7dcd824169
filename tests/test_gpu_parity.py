"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element, on
the same seeded inputs (BASELINE.json north_star tolerances: max|d| <= 1e-5 max|u| after one
step, <= 1e-4 max|u| after the config's full step count).  Plus bitwise identity across all
kernel variants and slab decompositions, ABI properties and errors."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import rtm_inputs as ri

pytestmark = pytest.mark.gpu

TOL_1 = 1e-5
TOL_FULL = 1e-4
C32 = ri.COEFFS_F32


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from conftest import build_library
    build_library()
    import paper_1310_8232_b200 as P
    return P


def relerr(a, b):
    m = float(np.abs(b).max())
    return float(np.abs(a.astype(np.float64) - b).max()) / (m if m > 0 else 1.0)


def gpu_run(P, v, dx, dt, steps, u0=None, up0=None, sources=(), tile=-1, devices=None):
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, dx, dt, C32, devices=devices) as sim:
        if tile != -1:
            sim.set_tile(tile)
        sim.set_velocity(v)
        for (x, y, z, w) in sources:
            sim.inject_source(x, y, z, w)
        if u0 is not None or up0 is not None:
            sim.set_fields(u0, up0)
        sim.step(steps)
        assert sim.steps_taken == steps
        return sim.read_field()


# ----------------------------------------------------------------------------- configs
def test_c1_full_run_vs_oracle(P):
    cfg = ri.make_config(1)
    v = cfg.velocity()
    src = cfg.sources()
    ref = oracle.run(v, cfg.dx, cfg.dt, C32, cfg.steps, sources=src)
    got = gpu_run(P, v, cfg.dx, cfg.dt, cfg.steps, sources=src)
    assert relerr(got, ref) <= TOL_FULL
    assert np.abs(ref).max() > 0


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_one_step_random_ics_small_grids(P, k):
    """1 step from seeded U[-1,1] ICs on each config's velocity recipe, at a size the oracle
    finishes in well under a second, spanning several tiles with ragged x/y/z tails."""
    cfg = ri.make_config(k, shape=(45, 70, 136), steps=1)
    v = cfg.velocity()
    u0, up0 = ri.random_fields(v.shape, seed=k)
    src = cfg.sources()
    ref = oracle.run(v, cfg.dx, cfg.dt, C32, 1, u0=u0, up0=up0, sources=src)
    got = gpu_run(P, v, cfg.dx, cfg.dt, 1, u0=u0, up0=up0, sources=src)
    assert relerr(got, ref) <= TOL_1


def test_c2_full_run_vs_oracle(P):
    cfg = ri.make_config(2)
    v = cfg.velocity()
    src = cfg.sources()
    ref = oracle.run(v, cfg.dx, cfg.dt, C32, cfg.steps, sources=src)
    got = gpu_run(P, v, cfg.dx, cfg.dt, cfg.steps, sources=src)
    assert relerr(got, ref) <= TOL_FULL


def test_c2_one_step_random_ics(P):
    cfg = ri.make_config(2)
    v = cfg.velocity()
    u0, up0 = ri.random_fields(v.shape, seed=22)
    ref = oracle.run(v, cfg.dx, cfg.dt, C32, 1, u0=u0, up0=up0, sources=cfg.sources())
    got = gpu_run(P, v, cfg.dx, cfg.dt, 1, u0=u0, up0=up0, sources=cfg.sources())
    assert relerr(got, ref) <= TOL_1


def test_c3_full_grid_20_steps_vs_oracle(P):
    cfg = ri.make_config(3, steps=20)
    v = cfg.velocity()
    u0, up0 = ri.random_fields(v.shape, seed=33)
    src = cfg.sources()
    ref = oracle.run(v, cfg.dx, cfg.dt, C32, 20, u0=u0, up0=up0, sources=src)
    got = gpu_run(P, v, cfg.dx, cfg.dt, 20, u0=u0, up0=up0, sources=src)
    assert relerr(got, ref) <= TOL_FULL


@pytest.mark.parametrize("k", [3, 5, 4])
def test_full_size_full_step_count_vs_oracle(P, k):
    """BASELINE.json north_star: "<= 1e-4 max|u| after the config's full step count" — the
    config's own recipe (zero ICs, its velocity model and Ricker sources) at full size and full
    step count: C3 512^3 x 200, C5 (G=1) 1024x1024x256 x 100, C4 1024^3 x 100 (16 shots'
    sources), every point against the fp32 oracle on all host cores (C4: ~2-3 min of CPU)."""
    cfg = ri.make_config(k)
    v = cfg.velocity()
    src = cfg.sources()
    got = gpu_run(P, v, cfg.dx, cfg.dt, cfg.steps, sources=src)
    ref = oracle.run(v, cfg.dx, cfg.dt, C32, cfg.steps, sources=src)
    assert np.abs(ref).max() > 0
    e = relerr(got, ref)
    print(f"C{k} {v.shape} {cfg.steps} steps: max|d|/max|u| = {e:.3e}")
    assert e <= TOL_FULL


@pytest.mark.parametrize("k", [4, 5])
def test_full_size_one_step_sampled(P, k):
    """Full BASELINE sizes (C4 1024^3, C5 1024x1024x256), in the bench's launch config:
    one step from random ICs, 200k sampled points + all of a few boundary lines checked
    one by one against the oracle's point evaluator."""
    cfg = ri.make_config(k)
    v = cfg.velocity()
    u0, up0 = ri.random_fields(v.shape, seed=40 + k)
    got = gpu_run(P, v, cfg.dx, cfg.dt, 1, u0=u0, up0=up0)
    nz, ny, nx = v.shape
    rng = np.random.default_rng(k)
    pts = np.stack([rng.integers(0, nx, 200_000), rng.integers(0, ny, 200_000),
                    rng.integers(0, nz, 200_000)], 1)
    edges = []
    for z in (0, 1, 4, 5, nz // 2, nz - 5, nz - 1):
        for y in (0, 4, ny - 1):
            edges.append(np.stack([np.arange(nx), np.full(nx, y), np.full(nx, z)], 1))
    pts = np.concatenate([pts] + edges).astype(np.int32)
    ref = oracle.points_f32(v, cfg.dx, cfg.dt, C32, u0, up0, pts)
    g = got[pts[:, 2], pts[:, 1], pts[:, 0]]
    assert relerr(g, ref) <= TOL_1


# ----------------------------------------------------------------------------- variants
def test_all_variants_bitwise_identical_and_match_oracle(P):
    """Every tile variant (and the naive kernel) computes the same bits: one per-point
    expression (SPEC.md:83 tiling transparency).  Ragged in x, y and z."""
    nz, ny, nx = 29, 37, 100
    rng = np.random.default_rng(5)
    v = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=5)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 7)
    src = [(3, 4, 5, w), (99, 36, 28, -w), (0, 0, 0, w), (50, 20, 14, 0.5 * w), (50, 20, 14, w)]
    ref = oracle.run(v, 10.0, 1e-3, C32, 7, u0=u0, up0=up0, sources=src)
    outs = [gpu_run(P, v, 10.0, 1e-3, 7, u0=u0, up0=up0, sources=src, tile=t)
            for t in range(P.rtm_num_tiles())]
    for t, o in enumerate(outs):
        assert np.array_equal(o, outs[0]), P.rtm_tile_name(t)
    assert relerr(outs[0], ref) <= TOL_1 * 10


@pytest.mark.parametrize("zchunk", [1, 3, 8, 64])
def test_zchunking_bitwise(P, zchunk):
    nz, ny, nx = 40, 24, 64
    v = np.full((nz, ny, nx), 2500.0, np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=9)
    base = gpu_run(P, v, 10.0, 1e-3, 5, u0=u0, up0=up0, tile=1)
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
        sim.set_tile(1)
        P.rtm_set_zchunk(sim.h, zchunk)
        sim.set_velocity(v)
        sim.set_fields(u0, up0)
        sim.step(5)
        assert np.array_equal(sim.read_field(), base)


def test_graph_and_direct_launch_paths_agree(P):
    """rtm_step uses CUDA graphs for runs of >= 16 steps from an even step; stepping one at a
    time (no graph) must give the same bits, including the source sample index."""
    cfg = ri.make_config(1, steps=40)
    v = cfg.velocity()
    src = cfg.sources()
    a = gpu_run(P, v, cfg.dx, cfg.dt, 40, sources=src)
    with P.Simulation(64, 64, 64, cfg.dx, cfg.dt, C32) as sim:
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        for _ in range(3):
            sim.step(1)           # odd start -> direct launches
        sim.step(33)              # direct, then graph
        sim.step(4)
        assert np.array_equal(sim.read_field(), a)


# ----------------------------------------------------------------------------- slabs
@pytest.mark.parametrize("G,halo", [(2, 0), (3, 0), (4, 0), (2, 1), (3, 1), (4, 1), (2, 2), (3, 2),
                                    (4, 2)])
def test_multislab_on_one_gpu_bitwise_equals_single(P, G, halo):
    """z-slab decomposition on one GPU gives exactly the G=1 field (R14): halo mode 0
    (boundary planes first, halo copies, interior), 1 (fused push, event ordered), 2 (fused
    push, flag protocol: stream waits on flag words + system-scope release kernels — the
    protocol the distributed context uses across processes)."""
    nz, ny, nx = 47, 33, 72
    rng = np.random.default_rng(G)
    v = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=100 + G)
    w = ri.source_samples(2500.0, 1e-3, 15.0, 9)
    bounds = [P.rtm_slab_range(nz, G, r)[0] for r in range(1, G)]
    src = [(5, 6, b, w) for b in bounds] + [(7, 8, b - 1, -w) for b in bounds] + [(1, 1, 0, w)]
    ref = gpu_run(P, v, 10.0, 1e-3, 9, u0=u0, up0=up0, sources=src)
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=[0] * G) as sim:
        P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
        assert P.rtm_get_option(sim.h, P.RTM_OPT_HALO_MODE) == halo
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        sim.step(4)
        sim.step(5)
        got = sim.read_field()
    assert np.array_equal(got, ref)
    orc = oracle.run(v, 10.0, 1e-3, C32, 9, u0=u0, up0=up0, sources=src)
    assert relerr(got, orc) <= TOL_1 * 10


@pytest.mark.parametrize("halo", [0, 2, 3])
def test_dist_world1_equals_single(P, halo):
    """The NCCL-communicator context at world 1; halo mode 2 runs its collective set-up (IPC
    handle export + NCCL all-gather) and the flag-protocol step path."""
    nz, ny, nx = 20, 16, 32
    v = np.full((nz, ny, nx), 2000.0, np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=3)
    ref = gpu_run(P, v, 10.0, 1e-3, 6, u0=u0, up0=up0)
    uid = P.rtm_get_unique_id()
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, dist=(0, 1, uid, 0)) as sim:
        P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
        sim.set_velocity(v)
        sim.set_fields(u0, up0)
        sim.step(6)
        assert np.array_equal(sim.read_field(), ref)
        P.rtm_set_step_count(sim.h, 3)  # collective barrier + flag generation restart
        sim.set_fields(u0, up0)
        sim.step(2)


@pytest.mark.parametrize("halo", [1, 2])
def test_multislab_fused_resume_and_reset(P, halo):
    """Flag generations: reset / set_fields / rtm_set_step_count restart the protocol (stale
    flags never satisfy a wait), including a parity swap of the time levels."""
    cfg = ri.make_config(2, shape=(40, 24, 64), steps=20)
    v = cfg.velocity()
    src = cfg.sources()
    ref = gpu_run(P, v, cfg.dx, cfg.dt, 20, sources=src)
    with P.Simulation(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, C32, devices=[0, 0, 0]) as sim:
        P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.step(9)
        u, up = sim.read_fields()
        sim.reset()
        sim.step(3)
        sim.set_fields(u, up)
        P.rtm_set_step_count(sim.h, 9)
        sim.step(11)
        assert np.array_equal(sim.read_field(), ref)


# ----------------------------------------------------------------------------- properties
def test_zero_fixed_point(P):
    v = np.full((16, 12, 20), 3000.0, np.float32)
    out = gpu_run(P, v, 10.0, 1e-3, 10, sources=[(3, 3, 3, np.zeros(10, np.float32))])
    assert not np.any(out)


def test_source_sample_timing(P):
    """sample n is added right after the stencil of step n (R4)."""
    v = np.full((12, 12, 12), 2000.0, np.float32)
    w = np.array([0.5, 0.25, 2.0], np.float32)
    out = gpu_run(P, v, 10.0, 1e-3, 1, sources=[(5, 6, 7, w)])
    assert out[7, 6, 5] == w[0] and np.count_nonzero(out) == 1


def test_mirror_symmetry_c1(P):
    """Centred source on 64^3: u(32+k) = u(32-k) per axis for k <= 31 (the boundary-induced
    asymmetry is ~1e-11 max|u| in fp64 over C1's 100 steps)."""
    cfg = ri.make_config(1)
    out = gpu_run(P, cfg.velocity(), cfg.dx, cfg.dt, cfg.steps, sources=cfg.sources())
    m = np.abs(out).max()
    s = out[1:, 1:, 1:]
    for ax in range(3):
        assert np.abs(s - np.flip(s, axis=ax)).max() <= 1e-6 * m


def test_polynomial_laplacian_through_abi(P):
    """u_prev = 2u trick: u^1 = C * L(u); for u = (x-xc)^a (y-yc)^b /h^(a+b) of per-axis
    degree <= 10 the result is C * analytic Laplacian away from the boundary."""
    nz, ny, nx = 24, 28, 32
    h = 6.0
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    xi, eta, ze = (x - 15.5) / h, (y - 13.5) / h, (z - 11.5) / h
    u = (xi**4 * eta**3 + ze**5).astype(np.float64)
    lap = (12 * xi**2 * eta**3 + 6 * xi**4 * eta + 20 * ze**3) / h**2
    nu = 0.4
    v = np.full(u.shape, nu * 10.0 / 1e-3, np.float32)
    out = gpu_run(P, v, 10.0, 1e-3, 1, u0=u.astype(np.float32), up0=(2 * u).astype(np.float32))
    Cf = np.float32(np.float64(v[0, 0, 0]) * 1e-3 / 10.0) ** 2
    s = (slice(5, -5),) * 3
    err = np.abs(out[s] - Cf * lap[s]).max()
    assert err <= 2e-5 * np.abs(u[s]).max() * 8 * Cf


def test_time_reversibility_fp32(P):
    nz, ny, nx = 24, 20, 32
    rng = np.random.default_rng(1)
    v = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=77)
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
        sim.set_velocity(v)
        sim.set_fields(u0, up0)
        sim.step(20)
        uN, uNm1 = sim.read_fields()
        sim.set_fields(uNm1, uN)
        sim.step(20)
        back, back_prev = sim.read_fields()
    assert np.abs(back - up0).max() <= 1e-4
    assert np.abs(back_prev - u0).max() <= 1e-4


# ----------------------------------------------------------------------------- edges
@pytest.mark.parametrize("shape", [(1, 1, 4), (1, 9, 8), (11, 1, 12), (3, 5, 7), (2, 3, 1), (13, 17, 20)])
def test_degenerate_and_tiny_grids(P, shape):
    v = np.full(shape, 3000.0, np.float32)
    u0, up0 = ri.random_fields(shape, seed=sum(shape))
    src = [(0, 0, 0, np.ones(4, np.float32))]
    ref = oracle.run(v, 10.0, 1e-3, C32, 4, u0=u0, up0=up0, sources=src)
    got = gpu_run(P, v, 10.0, 1e-3, 4, u0=u0, up0=up0, sources=src)
    assert relerr(got, ref) <= TOL_1 * 10


def test_zero_steps_and_reset(P):
    v = np.full((8, 8, 8), 3000.0, np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=2)
    with P.Simulation(8, 8, 8, 10.0, 1e-3, C32) as sim:
        sim.set_velocity(v)
        sim.set_fields(u0, up0)
        sim.step(0)
        assert np.array_equal(sim.read_field(), u0)
        sim.step(3)
        sim.reset()
        assert sim.steps_taken == 0 and not np.any(sim.read_field())


def test_max_sources_same_point(P):
    v = np.full((10, 10, 12), 2000.0, np.float32)
    w = np.linspace(-1, 1, 5).astype(np.float32)
    src = [(4, 5, 6, w * (k + 1) / 7) for k in range(P.RTM_MAX_SOURCES)]
    ref = oracle.run(v, 10.0, 1e-3, C32, 5, sources=src)
    got = gpu_run(P, v, 10.0, 1e-3, 5, sources=src)
    assert relerr(got, ref) <= 1e-6
    with P.Simulation(12, 10, 10, 10.0, 1e-3, C32) as sim:
        for s in src:
            sim.inject_source(*s)
        with pytest.raises(P.RtmError):
            sim.inject_source(1, 1, 1, w)


def test_errors_are_reported(P):
    with P.Simulation(8, 8, 8, 10.0, 1e-3, C32) as sim:
        with pytest.raises(P.RtmError) as e:
            sim.step(1)
        assert e.value.code == P.RTM_ESTATE
        vlim = ri.NU_CRIT * 10.0 / 1e-3
        with pytest.raises(P.RtmError) as e:
            sim.set_velocity(np.full((8, 8, 8), vlim * 1.001, np.float32))
        assert e.value.code == P.RTM_ECFL and "CFL" in str(e.value)
        sim.set_velocity(np.full((8, 8, 8), vlim * 0.999, np.float32))
        bad = np.full((8, 8, 8), 2000.0, np.float32)
        bad[3, 3, 3] = np.nan
        with pytest.raises(P.RtmError) as e:
            sim.set_velocity(bad)
        assert e.value.code == P.RTM_EINVAL
        with pytest.raises(P.RtmError) as e:
            sim.step(1)  # failed set_velocity leaves no velocity installed
        assert e.value.code == P.RTM_ESTATE
        with pytest.raises(P.RtmError):
            sim.inject_source(8, 0, 0, np.ones(2, np.float32))
        with pytest.raises(P.RtmError):
            sim.set_tile(P.rtm_num_tiles())
    with P.Simulation(6, 8, 8, 10.0, 1e-3, C32) as sim:  # nx % 4 != 0: pitched rows, all variants
        assert sim.tile == 35
        sim.set_tile(1)


def test_cfl_growth_at_1_02_nu_crit_is_rejected_and_0_99_is_bounded(P):
    shape = (32, 32, 32)
    vlim = ri.NU_CRIT * 10.0 / 1e-3
    with P.Simulation(32, 32, 32, 10.0, 1e-3, C32) as sim:
        with pytest.raises(P.RtmError):
            sim.set_velocity(np.full(shape, 1.02 * vlim, np.float32))
        sim.set_velocity(np.full(shape, 0.99 * vlim, np.float32))
        u0, up0 = ri.random_fields(shape, seed=8)
        sim.set_fields(u0, up0)
        sim.step(200)
        assert np.abs(sim.read_field()).max() < 20


# ----------------------------------------------------------------------------- torch plumbing
def test_device_pointer_variants_and_user_stream(P):
    import torch
    cfg = ri.make_config(2, shape=(40, 48, 64), steps=30)
    v = cfg.velocity()
    src = cfg.sources()
    ref = gpu_run(P, v, cfg.dx, cfg.dt, 30, sources=src)
    dv = torch.from_numpy(v).cuda()
    dout = torch.empty_like(dv)
    s = torch.cuda.Stream()
    with P.Simulation(64, 48, 40, cfg.dx, cfg.dt, C32) as sim:
        for x in src:
            sim.inject_source(*x)
        P.rtm_set_stream(sim.h, s.cuda_stream)
        with torch.cuda.stream(s):
            P.rtm_set_velocity_device(sim.h, dv.data_ptr())
            P.rtm_reset(sim.h)
            P.rtm_step(sim.h, 30)
            P.rtm_read_field_device(sim.h, dout.data_ptr())
        s.synchronize()
        assert np.array_equal(dout.cpu().numpy(), ref)
        P.rtm_set_profiling(sim.h, 1)
        P.rtm_step(sim.h, 5)
        n, ms = P.rtm_kernel_stats(sim.h)
        assert n == 5 and ms > 0
        P.rtm_set_stream(sim.h, 0)


# ----------------------------------------------------------------------------- tuner (f2)
def test_autotune_preserves_state_and_installs_winner(P):
    cfg = ri.make_config(2, shape=(96, 128, 128), steps=30)
    v = cfg.velocity()
    src = cfg.sources()
    ref = gpu_run(P, v, cfg.dx, cfg.dt, 30, sources=src)
    with P.Simulation(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, C32) as sim:
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.step(11)
        res, times = P.rtm_autotune(sim.h, 4)
        assert res["ncandidates"] == P.rtm_num_tiles() - 1 and len(times) == res["ncandidates"]
        assert np.all(np.isfinite(times)) and np.all(times > 0)
        assert res["min_time_ms"] == pytest.approx(times.min())
        assert res["quality_pct"] == pytest.approx(
            100 * (res["actual_time_ms"] - res["min_time_ms"]) / res["min_time_ms"])
        assert sim.tile == res["best_tile"] and sim.steps_taken == 11
        sim.step(19)
        assert np.array_equal(sim.read_field(), ref)
        res2, t2 = P.rtm_autotune(sim.h, 2, tiles=[1, 1, 2], zchunks=[0, 7, 0])
        assert res2["ncandidates"] == 3 and res2["best_tile"] in (1, 2)


def test_autotune_multislab(P):
    nz, ny, nx = 60, 40, 64
    v = np.full((nz, ny, nx), 2500.0, np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=4)
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=[0, 0]) as sim:
        sim.set_velocity(v)
        sim.set_fields(u0, up0)
        res, times = P.rtm_autotune(sim.h, 2, tiles=[1, 5, 0])
        assert res["best_tile"] == [1, 5, 0][int(np.argmin(times))]
        sim.step(4)
        got = sim.read_field()
    assert np.array_equal(got, gpu_run(P, v, 10.0, 1e-3, 4, u0=u0, up0=up0))


# ----------------------------------------------------------------------------- batched shots (f3)
@pytest.mark.parametrize("tile,order", [(-1, 0), (0, 0), (5, 1), (9, 2), (-1, 1), (-1, 2), (14, 1), (14, 2)])
def test_batched_shots_equal_independent_runs(P, tile, order):
    """A batch of shots on one velocity model = each shot run alone, bitwise; and each
    matches the oracle.  Shots differ in ICs and sources (one shot has none)."""
    nz, ny, nx = 23, 41, 68
    rng = np.random.default_rng(3)
    v = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
    S = 3
    ics = [ri.random_fields(v.shape, seed=200 + k) for k in range(S)]
    w = ri.source_samples(3000.0, 1e-3, 15.0, 6)
    srcs = {0: [(5, 6, 7, w)], 1: [], 2: [(60, 40, 22, -w), (0, 0, 0, 0.5 * w)]}
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, shots=S) as sim:
        if tile != -1:
            sim.set_tile(tile)
        P.rtm_set_option(sim.h, P.RTM_OPT_SHOT_ORDER, order)
        sim.set_velocity(v)
        for k in range(S):
            for s in srcs[k]:
                sim.inject_source(*s, shot=k)
        sim.set_fields(np.stack([a for a, _ in ics]), np.stack([b for _, b in ics]))
        sim.step(6)
        got = sim.read_field()
        assert got.shape == (S, nz, ny, nx)
    for k in range(S):
        alone = gpu_run(P, v, 10.0, 1e-3, 6, u0=ics[k][0], up0=ics[k][1], sources=srcs[k],
                        tile=tile)
        assert np.array_equal(got[k], alone), k
        orc = oracle.run(v, 10.0, 1e-3, C32, 6, u0=ics[k][0], up0=ics[k][1], sources=srcs[k])
        assert relerr(got[k], orc) <= TOL_1 * 10


def test_batch_errors(P):
    with pytest.raises(P.RtmError):
        P.rtm_create_batch(8, 8, 8, 10.0, 1e-3, C32, 0)
    h = P.rtm_create_batch(8, 8, 8, 10.0, 1e-3, C32, 2)
    try:
        assert P.rtm_num_shots(h) == 2
        with pytest.raises(P.RtmError):
            P.rtm_inject_source_shot(h, 2, 1, 1, 1, np.ones(3, np.float32))
    finally:
        P.rtm_destroy(h)


def test_fused_halo_mode_rejected_without_slabs(P):
    with P.Simulation(16, 16, 16, 10.0, 1e-3, C32) as sim:
        for mode in (1, 2, 3, -1):
            with pytest.raises(P.RtmError):
                P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, mode)
        assert P.rtm_get_option(sim.h, P.RTM_OPT_HALO_MODE) == 0


# ----------------------------------------------------------------------------- full-size properties
def _star_L_f64(u):
    """L(u) in fp64 with the zero halo (independent numpy evaluation, plane-chunked)."""
    nz, ny, nx = u.shape
    c = ri.COEFFS_F64
    out = np.zeros(u.shape, np.float64)
    out += 3 * c[0] * u
    for m in range(1, 6):
        out[m:] += c[m] * u[:-m]
        out[:-m] += c[m] * u[m:]
        out[:, m:] += c[m] * u[:, :-m]
        out[:, :-m] += c[m] * u[:, m:]
        out[:, :, m:] += c[m] * u[:, :, :-m]
        out[:, :, :-m] += c[m] * u[:, :, m:]
    return out


def _energy(u1, u0, Cf):
    """E^{n+1/2} = sum (u^{n+1}-u^n)^2 / C - sum u^{n+1} L u^n."""
    d = u1.astype(np.float64) - u0
    return float(np.sum(d * d / Cf) - np.sum(u1.astype(np.float64) * _star_L_f64(u0.astype(np.float64))))


def test_full_size_c3_energy_conserved_over_200_steps(P):
    """C3 at full size (512^3) for its full 200 steps from random ICs without sources: the
    discrete energy of the scheme (conserved exactly in real arithmetic for symmetric L and
    any C > 0) drifts only by fp32 rounding.  A dropped/extra term, a wrong index in any
    kernel path or a mis-staged tile breaks conservation at O(1)."""
    cfg = ri.make_config(3)
    v = cfg.velocity()
    Cf = (v.astype(np.float64) * cfg.dt / cfg.dx) ** 2
    u0, up0 = ri.random_fields(v.shape, seed=303, scale=1e-2)
    with P.Simulation(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, C32) as sim:
        sim.set_velocity(v)
        sim.set_fields(u0, up0)
        sim.step(1)
        a1, a0 = sim.read_fields()
        e_start = _energy(a1, a0, Cf)
        sim.step(cfg.steps - 1)
        b1, b0 = sim.read_fields()
        e_end = _energy(b1, b0, Cf)
    assert e_start > 0
    assert abs(e_end - e_start) <= 1e-4 * e_start, (e_start, e_end)


def test_full_size_c4_autotuned_variant_one_step_sampled(P):
    """The launch configuration bench.py times: rtm_autotune over the stream variants on the
    full C4 grid, then one step from random ICs with the selected variant, sampled against
    the oracle point evaluator."""
    cfg = ri.make_config(4)
    v = cfg.velocity()
    u0, up0 = ri.random_fields(v.shape, seed=44)
    with P.Simulation(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, C32) as sim:
        sim.set_velocity(v)
        cands = [t for t in range(P.rtm_num_tiles()) if P.rtm_tile_name(t).startswith("stream")]
        res, _ = P.rtm_autotune(sim.h, 2, tiles=cands)
        assert sim.tile == res["best_tile"]
        sim.set_fields(u0, up0)
        sim.step(1)
        got = sim.read_field()
    rng = np.random.default_rng(404)
    nz, ny, nx = v.shape
    pts = np.stack([rng.integers(0, nx, 100_000), rng.integers(0, ny, 100_000),
                    rng.integers(0, nz, 100_000)], 1).astype(np.int32)
    ref = oracle.points_f32(v, cfg.dx, cfg.dt, C32, u0, up0, pts)
    assert relerr(got[pts[:, 2], pts[:, 1], pts[:, 0]], ref) <= TOL_1


# ----------------------------------------------------------------------------- resume / failure detection
@pytest.mark.parametrize("n0", [30, 31])
def test_checkpoint_resume_bitwise(P, n0):
    cfg = ri.make_config(2, shape=(40, 36, 64), steps=50)
    v = cfg.velocity()
    src = cfg.sources()
    ref = gpu_run(P, v, cfg.dx, cfg.dt, 50, sources=src)
    with P.Simulation(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, C32) as sim:
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.step(n0)
        u, up = sim.read_fields()
    with P.Simulation(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, C32) as sim:
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u, up)
        P.rtm_set_step_count(sim.h, n0)
        assert sim.steps_taken == n0
        sim.step(50 - n0)
        assert np.array_equal(sim.read_field(), ref)


def test_field_stats_and_instability_detection(P):
    shape = (20, 24, 32)
    v = np.full(shape, 3000.0, np.float32)
    u0, up0 = ri.random_fields(shape, seed=6)
    with P.Simulation(32, 24, 20, 10.0, 1e-3, C32) as sim:
        sim.set_velocity(v)
        sim.set_fields(u0, up0)
        m, bad = P.rtm_field_stats(sim.h)
        assert bad == 0 and m == pytest.approx(float(np.abs(u0).max()))
        P.rtm_set_option(sim.h, P.RTM_OPT_CHECK_EVERY, 3)
        sim.step(7)  # finite: no error
        u0[10, 12, 16] = np.inf
        sim.set_fields(u0, up0)
        with pytest.raises(P.RtmError) as e:
            sim.step(5)
        assert e.value.code == P.RTM_EUNSTABLE
        assert sim.steps_taken == 3  # stopped at the first check


# ----------------------------------------------------------------------------- two-step passes (f4)
def _tb_ids(P):
    return [t for t in range(P.rtm_num_tiles()) if P.rtm_tile_name(t).startswith("tb2")]


def _tb_reps(P):
    """The two-step variants exercised by the slower cases: the first and the last."""
    ids = _tb_ids(P)
    return [ids[0], ids[-1]]


def _run_opts(P, v, steps, u0, up0, src, tile, tb_ctas=0, graphs=1, chunks=None):
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
        sim.set_tile(tile)
        P.rtm_set_option(sim.h, P.RTM_OPT_TB_CTAS, tb_ctas)
        P.rtm_set_option(sim.h, P.RTM_OPT_GRAPHS, graphs)
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        for k in (chunks or [steps]):
            sim.step(k)
        return sim.read_fields()


@pytest.mark.parametrize("tb_ctas", [0, 12, 24])
def test_tb2_bitwise_equals_single_step(P, tb_ctas):
    """Two steps per pass (k_tb2s) give exactly the bits of two single steps (k_stream): same
    per-point expression, u^{n+1} handed between CTAs through L2.  tb_ctas = 12 / 24 force
    multi-band plans (redundant A rows at every band edge) on a ragged 200 x 150 plane;
    sources sit on band edges, on the z ends and in the ragged x tail."""
    nz, ny, nx = 23, 150, 200
    rng = np.random.default_rng(77)
    v = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=77)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 9)
    src = [(5, 0, 0, w), (199, 149, 22, -w), (130, 36, 11, w), (64, 37, 3, 0.5 * w),
           (63, 38, 19, w), (100, 75, 12, w), (196, 112, 7, -w), (17, 113, 7, w)]
    ref_u, ref_up = _run_opts(P, v, 9, u0, up0, src, 35)
    for t in _tb_ids(P):
        u, up = _run_opts(P, v, 9, u0, up0, src, t, tb_ctas=tb_ctas)
        assert np.array_equal(u, ref_u), P.rtm_tile_name(t)
        assert np.array_equal(up, ref_up), P.rtm_tile_name(t)


def test_tb2_graphs_odd_starts_and_short_z(P):
    """Graph replays of 16 passes (from both parities and both buffer banks), odd remainders
    and direct passes all agree bitwise with single steps; nz smaller than the lag."""
    for shape in [(70, 40, 64), (3, 33, 48), (1, 20, 32)]:
        nz, ny, nx = shape
        rng = np.random.default_rng(nz)
        v = rng.uniform(1500, 4300, shape).astype(np.float32)
        u0, up0 = ri.random_fields(shape, seed=nz)
        w = ri.source_samples(3000.0, 1e-3, 15.0, 80)
        src = [(nx // 2, ny // 2, nz // 2, w)]
        ref_u, _ = _run_opts(P, v, 75, u0, up0, src, 35, chunks=[75])
        for tb in _tb_reps(P):
            for chunks in ([75], [1, 33, 1, 40], [2, 2, 32, 39]):
                u, _ = _run_opts(P, v, 75, u0, up0, src, tb, chunks=chunks)
                assert np.array_equal(u, ref_u), (shape, chunks, P.rtm_tile_name(tb))
            u, _ = _run_opts(P, v, 75, u0, up0, src, tb, graphs=0, tb_ctas=6)
            assert np.array_equal(u, ref_u), (shape, P.rtm_tile_name(tb))


def test_tb2_c1_c2_full_runs_vs_oracle(P):
    """The configs' full step counts through the two-step path vs the fp32 oracle
    (north_star tolerance 1e-4 max|u|)."""
    for k in (1, 2):
        cfg = ri.make_config(k)
        v = cfg.velocity()
        src = cfg.sources()
        ref = oracle.run(v, cfg.dx, cfg.dt, C32, cfg.steps, sources=src)
        for tb in _tb_reps(P):
            got = gpu_run(P, v, cfg.dx, cfg.dt, cfg.steps, sources=src, tile=tb)
            assert relerr(got, ref) <= TOL_FULL, (k, P.rtm_tile_name(tb))


def test_full_size_c4_tb2_sampled(P):
    """C4 (1024^3, 8 y-bands) two steps through k_tb2s from random ICs: bitwise equal to two
    single steps of k_stream (itself sampled against the oracle at this size), and u^1 —
    produced by stage A and consumed by stage B through L2 — sampled against the oracle."""
    cfg = ri.make_config(4)
    v = cfg.velocity()
    u0, up0 = ri.random_fields(v.shape, seed=45)
    tb = _tb_reps(P)[0]
    outs = {}
    for t in (35, tb):
        with P.Simulation(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, C32) as sim:
            sim.set_tile(t)
            sim.set_velocity(v)
            sim.set_fields(u0, up0)
            sim.step(2)
            outs[t] = sim.read_fields()
    assert np.array_equal(outs[tb][0], outs[35][0])
    assert np.array_equal(outs[tb][1], outs[35][1])
    u1 = outs[tb][1]  # u^1
    rng = np.random.default_rng(405)
    nz, ny, nx = v.shape
    pts = np.stack([rng.integers(0, nx, 50_000), rng.integers(0, ny, 50_000),
                    rng.integers(0, nz, 50_000)], 1).astype(np.int32)
    ref1 = oracle.points_f32(v, cfg.dx, cfg.dt, C32, u0, up0, pts)
    assert relerr(u1[pts[:, 2], pts[:, 1], pts[:, 0]], ref1) <= TOL_1


# ----------------------------------------------------------------------------- asynchronous pipeline
def test_async_pipeline_equals_sync_calls(P):
    """rtm_set_velocity_async / rtm_step_async / rtm_read_field_async pipelined over several
    velocity models (H2D of the next model and D2H of the previous result overlap the steps)
    give bitwise the results of the synchronous calls; mixing in a synchronous call works."""
    nz, ny, nx = 30, 40, 64
    rng = np.random.default_rng(12)
    models = [rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32) for _ in range(3)]
    w = ri.source_samples(3000.0, 1e-3, 15.0, 20)
    src = [(30, 20, 15, w)]
    refs = [gpu_run(P, v, 10.0, 1e-3, 17, sources=src) for v in models]
    outs = [np.empty((nz, ny, nx), np.float32) for _ in models]
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
        for s in src:
            sim.inject_source(*s)
        for v, o in zip(models, outs):
            P.rtm_set_velocity_async(sim.h, v)
            P.rtm_reset(sim.h)
            P.rtm_step_async(sim.h, 17)
            P.rtm_read_field_async(sim.h, o)
        P.rtm_sync(sim.h)
        for o, r in zip(outs, refs):
            assert np.array_equal(o, r)
        sim.set_velocity(models[1])           # synchronous call after asynchronous ones
        sim.reset()
        P.rtm_step_async(sim.h, 17)
        assert np.array_equal(sim.read_field(), refs[1])
        with pytest.raises(ValueError):
            P.rtm_read_field_async(sim.h, np.empty((nz, ny, nx), np.float64))


def test_async_velocity_verdict_is_deferred(P):
    nz, ny, nx = 12, 16, 32
    good = np.full((nz, ny, nx), 2000.0, np.float32)
    bad = np.full((nz, ny, nx), 4600.0, np.float32)  # nu = 0.46 > nu_crit = 0.4419 at dt = 1 ms
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
        P.rtm_set_velocity_async(sim.h, good)
        P.rtm_step_async(sim.h, 2)
        P.rtm_sync(sim.h)
        P.rtm_set_velocity_async(sim.h, bad)
        P.rtm_step_async(sim.h, 2)
        with pytest.raises(P.RtmError) as e:
            P.rtm_sync(sim.h)
        assert e.value.code == P.RTM_ECFL
        with pytest.raises(P.RtmError) as e:
            P.rtm_step_async(sim.h, 1)       # the velocity is unset after the verdict
        assert e.value.code == P.RTM_ESTATE
        nan = good.copy()
        nan[3, 4, 5] = np.nan
        P.rtm_set_velocity_async(sim.h, nan)
        with pytest.raises(P.RtmError) as e:
            sim.set_velocity(good)             # a synchronising call returns the pending verdict
        assert e.value.code == P.RTM_EINVAL
        sim.set_velocity(good)
        sim.step(1)


def test_async_pipeline_batched_shots_and_dist_world1(P):
    """The asynchronous calls on a batched (2-shot) context and on a distributed context at
    world 1: same bits as the synchronous path."""
    nz, ny, nx = 20, 24, 32
    rng = np.random.default_rng(21)
    v = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 12)
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, shots=2) as sim:
        P.rtm_inject_source_shot(sim.h, 0, 5, 6, 7, w)
        P.rtm_inject_source_shot(sim.h, 1, 20, 12, 9, -w)
        sim.set_velocity(v)
        sim.step(11)
        ref = sim.read_field()
        out = np.empty_like(ref)
        P.rtm_set_velocity_async(sim.h, v)
        P.rtm_reset(sim.h)
        P.rtm_step_async(sim.h, 11)
        P.rtm_read_field_async(sim.h, out)
        P.rtm_sync(sim.h)
        assert np.array_equal(out, ref)
    ref1 = gpu_run(P, v, 10.0, 1e-3, 11, sources=[(5, 6, 7, w)])
    uid = P.rtm_get_unique_id()
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, dist=(0, 1, uid, 0)) as sim:
        sim.inject_source(5, 6, 7, w)
        out = np.empty((nz, ny, nx), np.float32)
        P.rtm_set_velocity_async(sim.h, v)
        P.rtm_step_async(sim.h, 11)
        P.rtm_read_field_async(sim.h, out)
        P.rtm_sync(sim.h)
        assert np.array_equal(out, ref1)


# ----------------------------------------------------------------------------- resident multi-step kernel
def test_resident_kernel_c1_and_batched_bitwise(P):
    """k_resident (many steps per cooperative launch, grid barrier between steps) gives the
    bits of per-step k_stream launches: C1's full run with its source, odd starts and
    multi-launch runs, and a 3-shot batch; and stays within the oracle tolerance."""
    ids = [t for t in range(P.rtm_num_tiles()) if P.rtm_tile_name(t).startswith("resident")]
    assert ids
    cfg = ri.make_config(1)
    v = cfg.velocity()
    src = cfg.sources()
    ref = gpu_run(P, v, cfg.dx, cfg.dt, cfg.steps, sources=src, tile=35)
    orc = oracle.run(v, cfg.dx, cfg.dt, C32, cfg.steps, sources=src)
    for t in ids:
        with P.Simulation(64, 64, 64, cfg.dx, cfg.dt, C32) as sim:
            sim.set_tile(t)
            sim.set_velocity(v)
            for s in src:
                sim.inject_source(*s)
            for k in (1, 40, 3, 56):   # odd start, several launches
                sim.step(k)
            got = sim.read_field()
        assert np.array_equal(got, ref), P.rtm_tile_name(t)
    assert relerr(got, orc) <= TOL_FULL
    nz, ny, nx = 18, 22, 36
    rng = np.random.default_rng(5)
    vb = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
    u0, up0 = ri.random_fields((3, nz, ny, nx), seed=6)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 9)
    outs = []
    for t in (35, ids[0]):
        with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, shots=3) as sim:
            sim.set_tile(t)
            sim.set_velocity(vb)
            P.rtm_inject_source_shot(sim.h, 2, 35, 21, 17, w)
            P.rtm_inject_source_shot(sim.h, 0, 0, 0, 0, -w)
            sim.set_fields(u0, up0)
            sim.step(9)
            outs.append(sim.read_fields())
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_pdl_launches_bitwise(P):
    """Programmatic dependent launch of consecutive k_stream steps (graph and direct paths,
    multi-slab fused mode) gives the same bits as plain launches."""
    cfg = ri.make_config(2, shape=(48, 40, 64), steps=37)
    v = cfg.velocity()
    src = cfg.sources()
    ref = gpu_run(P, v, cfg.dx, cfg.dt, 37, sources=src, tile=35)
    for devices, halo in ((None, 0), ([0, 0, 0], 2), ([0, 0], 1)):
        with P.Simulation(64, 40, 48, cfg.dx, cfg.dt, C32, devices=devices) as sim:
            P.rtm_set_option(sim.h, P.RTM_OPT_PDL, 1)
            assert P.rtm_get_option(sim.h, P.RTM_OPT_PDL) == 1
            if halo:
                P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
            sim.set_tile(35)
            sim.set_velocity(v)
            for s in src:
                sim.inject_source(*s)
            sim.step(3)
            sim.step(34)
            assert np.array_equal(sim.read_field(), ref), (devices, halo)


def test_new_paths_edge_cases(P):
    """Asynchronous calls refuse multi-slab contexts; the two-step and resident variants run
    under the field check and under per-launch profiling; option ranges are validated."""
    nz, ny, nx = 24, 30, 64
    v = np.full((nz, ny, nx), 2500.0, np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=31)
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=[0, 0]) as sim:
        sim.set_velocity(v)
        for call in (lambda: P.rtm_set_velocity_async(sim.h, v), lambda: P.rtm_step_async(sim.h, 1),
                     lambda: P.rtm_read_field_async(sim.h, np.empty(v.shape, np.float32))):
            with pytest.raises(P.RtmError) as e:
                call()
            assert e.value.code == P.RTM_EINVAL
    ref = gpu_run(P, v, 10.0, 1e-3, 12, u0=u0, up0=up0, tile=35)
    names = {P.rtm_tile_name(t): t for t in range(P.rtm_num_tiles())}
    for name in [n for n in names if n.startswith(("tb2s_", "resident"))][:2] + ["resident256x2"]:
        for mode in ("check", "profile"):
            with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
                sim.set_tile(names[name])
                sim.set_velocity(v)
                sim.set_fields(u0, up0)
                if mode == "check":
                    P.rtm_set_option(sim.h, P.RTM_OPT_CHECK_EVERY, 5)
                else:
                    P.rtm_set_profiling(sim.h, 1)
                sim.step(7)
                sim.step(5)
                if mode == "profile":
                    launches, ms = P.rtm_kernel_stats(sim.h)
                    assert launches >= 1 and ms > 0
                assert np.array_equal(sim.read_field(), ref), (name, mode)
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
        for key, bad in ((P.RTM_OPT_PDL, 2), (P.RTM_OPT_TB_CTAS, -1), (P.RTM_OPT_HALO_MODE, 3)):
            with pytest.raises(P.RtmError):
                P.rtm_set_option(sim.h, key, bad)


def test_autotune_over_paper_lattice_is_exhaustive_argmin(P):
    """Selection phase over {2 tiles} x the P-parts z-chunk lattice: the
    installed candidate is the argmin of the per-candidate times (the exhaustive-lattice
    ranking, MWMB at one rank), the verification time is reported, the wavefield is kept."""
    nz, ny, nx = 40, 48, 64
    v = np.full((nz, ny, nx), 2500.0, np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=8)
    lat = P.rtm_blocksize_lattice(nz, 4)
    assert lat == [1, 14, 27, 40]
    tiles = [1, 35]
    cands = [t for t in tiles for _ in lat]
    zcs = [z for _ in tiles for z in lat]
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
        sim.set_velocity(v)
        sim.set_fields(u0, up0)
        res, times = P.rtm_autotune(sim.h, 3, tiles=cands, zchunks=zcs)
        k = int(np.argmin(times))
        assert len(times) == len(cands) and np.all(times > 0)
        assert (res["best_tile"], res["best_zchunk"]) == (cands[k], zcs[k])
        assert res["actual_time_ms"] > 0
        assert sim.tile == cands[k] and P.rtm_get_option(sim.h, P.RTM_OPT_ZCHUNK) == zcs[k]
        u, up = sim.read_fields()
        assert np.array_equal(u, u0) and np.array_equal(up, up0)


def test_beyond_2pow32_points_one_step_sampled(P):
    """A 2048 x 2048 x 1024 grid (4.3e9 points > 2^32, 52 GB of fields on the device): every
    offset is 64-bit.  One step from random ICs with the default (autotune-free) variant,
    sampled against the oracle point evaluator, with samples forced into the last planes,
    rows and columns."""
    nz, ny, nx = 1024, 2048, 2048
    v = ri.layered_velocity((nz, ny, nx), np.array([1800, 2600, 3200, 3900, 4200, 2900], np.float32))
    u0, up0 = ri.random_fields(v.shape, seed=4242)
    with P.Simulation(nx, ny, nz, 10.0, 0.8e-3, C32) as sim:
        sim.set_velocity(v)
        sim.set_fields(u0, up0)
        sim.step(1)
        got = sim.read_field()
    rng = np.random.default_rng(4243)
    m = 60_000
    pts = np.stack([rng.integers(0, nx, m), rng.integers(0, ny, m), rng.integers(0, nz, m)], 1)
    tail = np.stack([rng.integers(0, nx, 4000), rng.integers(ny - 8, ny, 4000),
                     rng.integers(nz - 8, nz, 4000)], 1)
    edge = np.array([[nx - 1, ny - 1, nz - 1], [0, 0, 0], [nx - 1, 0, nz - 1], [0, ny - 1, nz - 2]])
    pts = np.concatenate([pts, tail, edge]).astype(np.int32)
    ref = oracle.points_f32(v, 10.0, 0.8e-3, C32, u0, up0, pts)
    assert relerr(got[pts[:, 2], pts[:, 1], pts[:, 0]], ref) <= TOL_1


# ----------------------------------------------------------------------------- pitched rows (nx % 4 != 0)
@pytest.mark.parametrize("nx", [5, 66, 131])
def test_ragged_nx_all_variants_bitwise_and_vs_oracle(P, nx):
    """Rows are pitched to a multiple of 4 floats and the padding columns stay zero, so every
    variant (TMA stream/tiled kernels, two-step, resident) runs any nx and matches the naive
    kernel bitwise; sources on the last column (inside the padded group) and the first."""
    nz, ny = 19, 23
    rng = np.random.default_rng(nx)
    v = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=nx)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 7)
    src = [(nx - 1, ny // 2, nz // 2, w), (0, 0, 3, -w), (nx // 2, ny - 1, nz - 1, w)]
    ref = oracle.run(v, 10.0, 1e-3, C32, 7, u0=u0, up0=up0, sources=src)
    outs = {}
    for t in range(P.rtm_num_tiles()):
        outs[t] = gpu_run(P, v, 10.0, 1e-3, 7, u0=u0, up0=up0, sources=src, tile=t)
        assert np.array_equal(outs[t], outs[0]), P.rtm_tile_name(t)
    assert relerr(outs[0], ref) <= TOL_1 * 10


def test_ragged_nx_slabs_async_dist_and_device_velocity(P):
    """Pitched layout through every copy path: multi-slab (halo modes 0/1/2), the asynchronous
    pipeline, the distributed context at world 1 and the device-pointer velocity/readback."""
    import torch
    nz, ny, nx = 36, 21, 66
    rng = np.random.default_rng(66)
    v = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
    u0, up0 = ri.random_fields(v.shape, seed=67)
    ref = gpu_run(P, v, 10.0, 1e-3, 9, u0=u0, up0=up0, tile=0)
    for halo in (0, 1, 2):
        with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=[0, 0, 0]) as sim:
            P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
            sim.set_velocity(v)
            sim.set_fields(u0, up0)
            sim.step(9)
            assert np.array_equal(sim.read_field(), ref), halo
    uid = P.rtm_get_unique_id()
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, dist=(0, 1, uid, 0)) as sim:
        sim.set_velocity(v)
        sim.set_fields(u0, up0)
        sim.step(9)
        assert np.array_equal(sim.read_field(), ref)
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
        d_v = torch.from_numpy(v).cuda()
        d_out = torch.empty_like(d_v)
        P.rtm_set_velocity_device(sim.h, d_v.data_ptr())
        sim.set_fields(u0, up0)
        sim.step(9)
        P.rtm_read_field_device(sim.h, d_out.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(d_out.cpu().numpy(), ref)
        out = np.empty_like(v)
        P.rtm_set_velocity_async(sim.h, v)
        sim.set_fields(u0, up0)
        P.rtm_step_async(sim.h, 9)
        P.rtm_read_field_async(sim.h, out)
        P.rtm_sync(sim.h)
        assert np.array_equal(out, ref)


def test_bench_line_contract_and_consistency(P):
    """bench.py (C1, 3 steps) prints one JSON line with the driver's keys, and its roofline
    fields are self-consistent: achieved = alg bytes per launch / average launch time,
    frac = achieved / peak; e2e counts its H2D / D2H bytes; launches are counted."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--config", "1", "--steps", "3",
                        "--warmup", "3", "--no-cpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0 and d["gpu_launches"] > 0
    rf = d["roofline"]
    achieved = rf["alg_bytes_per_launch"] / (rf["avg_launch_ms"] / 1e3) / 1e9
    assert abs(achieved - rf["achieved"]) <= 0.01 * rf["achieved"] + 1.0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) <= 1e-3
    nbytes = 64 ** 3 * 4
    assert d["e2e"]["h2d_bytes_per_step"] == nbytes and d["e2e"]["d2h_bytes_per_step"] == nbytes
    assert d["e2e"]["value"] > 0 and d["e2e"]["matches_device_result"] is True
    assert d["config"]["workload"] == "C1" and d["clocks"]["sm_max_mhz"]
    # the tuner refinement installed its pick: the timed kernel is the refined selection
    ref = d["autotune"]["refine"]
    assert ref["selected"] == d["autotune"]["selected"]
    if ref["finalists"] > 1:
        assert len(ref["mean_ms_per_step"]) == ref["finalists"]
        assert d["kernel_variant"] == ref["selected"] or ref["selected"] in rf["kernel"]


def test_randomized_parity_fuzz_slice(P):
    """40 cases of tests/fuzz_parity.py (random ragged shapes, velocities, ICs, sources, step
    counts): every variant bitwise equal to the naive kernel, slab modes bitwise equal to the
    single slab, the naive kernel within tolerance of the oracle."""
    import importlib.util
    import sys
    from pathlib import Path
    path = Path(__file__).resolve().parent.parent / "tests" / "fuzz_parity.py"
    spec = importlib.util.spec_from_file_location("fuzz_parity", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    argv = sys.argv
    try:
        sys.argv = ["fuzz_parity.py", "40", "99", "1.0"]
        assert mod.main() == 0
    finally:
        sys.argv = argv
