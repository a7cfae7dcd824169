"""GPU regression tests of round 2: state restarts of the fused-halo flag protocol and the
two-step flag numbering, the field check's own reduction buffer, and host-array validation in
the binding.  Each compares against the G = 1 single-step kernel bitwise (R14, SURVEY.md §8(c)
P11) or checks an error contract of include/rtm.h."""
from __future__ import annotations

import os

import numpy as np
import pytest

import rtm_inputs as ri

os.environ.setdefault("RTM_DEBUG", "1")  # the library reports a refused graph capture on stderr

pytestmark = pytest.mark.gpu
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


def _single(P, v, steps, u0, up0, src, tile=35):
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
        sim.set_tile(tile)
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        sim.step(steps)
        return sim.read_fields()


def _case(seed, shape=(47, 33, 72)):
    rng = np.random.default_rng(seed)
    v = rng.uniform(1500, 4300, shape).astype(np.float32)
    u0, up0 = ri.random_fields(shape, seed=seed + 1)
    w = ri.source_samples(2500.0, 1e-3, 15.0, 40)
    nz = shape[0]
    src = [(5, 6, nz // 3, w), (7, 8, 2 * nz // 3 - 1, -w), (1, 1, 0, w)]
    return v, u0, up0, src


@pytest.mark.parametrize("G", [2, 3])
def test_autotune_then_step_in_halo_mode_2_is_bitwise(P, G):
    """rtm_autotune rewinds the step counter; the flag words then hold
    generation|steps-reached-while-tuning.  The tuner now starts a new flag generation (after a
    rank barrier in distributed contexts), so the slabs stay ordered after tuning."""
    v, u0, up0, src = _case(10 + G)
    ref_u, ref_up = _single(P, v, 17, u0, up0, src)
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=[0] * G) as sim:
        P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, 2)
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        sim.step(5)
        res, _ = P.rtm_autotune(sim.h, 6, tiles=[1, 35, 8], zchunks=[0, 0, 9])
        assert sim.steps_taken == 5
        sim.step(12)
        u, up = sim.read_fields()
    assert np.array_equal(u, ref_u) and np.array_equal(up, ref_up)


def test_field_stats_keeps_the_pending_async_velocity_verdict(P):
    """rtm_field_stats between rtm_set_velocity_async and rtm_sync must not
    overwrite the deferred CFL verdict (it now reduces into its own buffer)."""
    shape = (20, 24, 32)
    good = np.full(shape, 2000.0, np.float32)
    bad = np.full(shape, 2000.0, np.float32)
    bad[3, 4, 5] = 9000.0  # nu = 0.9 > nu_crit
    with P.Simulation(shape[2], shape[1], shape[0], 10.0, 1e-3, C32) as sim:
        sim.set_velocity(good)
        sim.set_fields(*ri.random_fields(shape, seed=5))
        P.rtm_set_velocity_async(sim.h, bad)
        m, nbad = P.rtm_field_stats(sim.h)
        assert m > 0 and nbad == 0
        with pytest.raises(P.RtmError) as e:
            P.rtm_sync(sim.h)
        assert e.value.code == P.RTM_ECFL
        # the verdict marked the velocity unset
        with pytest.raises(P.RtmError) as e:
            sim.step(1)
        assert e.value.code == P.RTM_ESTATE


def test_two_step_plan_change_on_a_running_context_is_bitwise(P):
    """the two-step flag epoch (epoch*nbands + band + 1) only grows while
    the band count is fixed.  Raising RTM_OPT_TB_CTAS on a context that already ran passes
    lowers the band count; the flags are now cleared when the plan changes."""
    shape = (23, 150, 200)
    v, u0, up0, src = _case(77, shape)
    ref_u, ref_up = _single(P, v, 30, u0, up0, src)
    tb = [t for t in range(P.rtm_num_tiles()) if (P.rtm_tile_name(t) or "").startswith("tb2")]
    nz, ny, nx = shape
    for t in (tb[0], tb[-1]):
        with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
            sim.set_tile(t)
            sim.set_velocity(v)
            for s in src:
                sim.inject_source(*s)
            sim.set_fields(u0, up0)
            P.rtm_set_option(sim.h, P.RTM_OPT_GRAPHS, 0)
            P.rtm_set_option(sim.h, P.RTM_OPT_TB_CTAS, 12)   # many narrow bands
            sim.step(10)
            P.rtm_set_option(sim.h, P.RTM_OPT_TB_CTAS, 0)    # one band per SM set: fewer bands
            sim.step(10)
            P.rtm_set_option(sim.h, P.RTM_OPT_TB_CTAS, 24)
            P.rtm_set_option(sim.h, P.RTM_OPT_GRAPHS, 1)
            sim.step(10)
            u, up = sim.read_fields()
        assert np.array_equal(u, ref_u), P.rtm_tile_name(t)
        assert np.array_equal(up, ref_up), P.rtm_tile_name(t)


def test_binding_validates_host_arrays(P):
    """every host-array entry point checks dtype, contiguity and element count
    against the context's extents (rtm_get_dims) and raises ValueError before the library
    touches memory."""
    shape = (12, 10, 16)
    v = np.full(shape, 2000.0, np.float32)
    with P.Simulation(shape[2], shape[1], shape[0], 10.0, 1e-3, C32) as sim:
        assert P.rtm_get_dims(sim.h) == (16, 10, 12, 1)
        with pytest.raises(ValueError):
            P.rtm_set_velocity(sim.h, v[:-1])
        sim.set_velocity(v)
        with pytest.raises(ValueError):
            P.rtm_set_fields(sim.h, np.zeros(5, np.float32))
        with pytest.raises(ValueError):
            P.rtm_read_field(sim.h, np.empty(shape[0] * shape[1] * shape[2] - 1, np.float32))
        with pytest.raises(ValueError):
            P.rtm_read_field(sim.h, np.empty(shape, np.float64))
        with pytest.raises(ValueError):
            P.rtm_read_field(sim.h, np.empty((shape[0], shape[1], 2 * shape[2]), np.float32)[:, :, ::2])
        with pytest.raises(ValueError):
            P.rtm_read_fields(sim.h, None, np.empty(7, np.float32))
        with pytest.raises(ValueError):
            P.rtm_read_field_async(sim.h, np.empty(9, np.float32))
        with pytest.raises(ValueError):
            P.rtm_set_velocity_async(sim.h, np.ones(9, np.float32))
        out = np.empty(shape, np.float32)
        P.rtm_read_field(sim.h, out)  # the exact shape still works
    with P.Simulation(16, 10, 12, 10.0, 1e-3, C32, shots=3) as sim:
        assert P.rtm_get_dims(sim.h) == (16, 10, 12, 3)
        sim.set_velocity(v)
        with pytest.raises(ValueError):
            P.rtm_read_field(sim.h, np.empty(shape, np.float32))
        assert sim.read_field().shape == (3,) + shape


# ----------------------------------------------------------------------------- slab data plane
def _slabs(P, v, steps, u0, up0, src, G, halo, host_ordered=0, graphs=1, chunks=None):
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=[0] * G) as sim:
        P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
        P.rtm_set_option(sim.h, P.RTM_OPT_HOST_ORDERED, host_ordered)
        P.rtm_set_option(sim.h, P.RTM_OPT_GRAPHS, graphs)
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        for k in (chunks or [steps]):
            sim.step(k)
        return sim.read_fields(), P.rtm_last_enqueue_ms(sim.h)


@pytest.mark.parametrize("G,host_ordered", [(2, 0), (3, 0), (4, 0), (3, 1)])
def test_multislab_copy_engine_pull_bitwise(P, G, host_ordered):
    """Halo mode 3 in-process: boundary planes, 'boundary ready' flags, copy-engine pulls from
    the neighbours' buffers on the comm streams overlapped with the interior, 'step complete'
    flags (WAR) — bitwise equal to G = 1, through reset and resume restarts."""
    v, u0, up0, src = _case(30 + G)
    ref_u, ref_up = _single(P, v, 21, u0, up0, src)
    (u, up), _ = _slabs(P, v, 21, u0, up0, src, G, 3, host_ordered, chunks=[1, 3, 17])
    assert np.array_equal(u, ref_u) and np.array_equal(up, ref_up)
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=[0] * G) as sim:
        P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, 3)
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        sim.step(9)
        a, b = sim.read_fields()
        sim.reset()
        sim.step(5)
        sim.set_fields(a, b)
        P.rtm_set_step_count(sim.h, 9)
        sim.step(12)
        u2, up2 = sim.read_fields()
    assert np.array_equal(u2, ref_u) and np.array_equal(up2, ref_up)


@pytest.mark.parametrize("halo", [0, 1])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_slab_step_graphs_bitwise_and_cheaper_to_enqueue(P, G, halo):
    """The G > 1 step captured in CUDA graphs (16 steps per replay; halo modes 0 and 1:
    boundary launch, events, copies, interior / the event-ordered fused push) is bitwise equal
    to direct launches, from both parities, and costs less host time to enqueue."""
    shape = (80, 37, 64)
    v, u0, up0, src = _case(50 + G, shape)
    ref_u, ref_up = _single(P, v, 70, u0, up0, src)
    # 1 direct; 1 direct + 32 in 2 replays + 3 direct (capture); 1 direct + 32 in 2 replays
    (u, up), t_graph = _slabs(P, v, 70, u0, up0, src, G, halo, graphs=1, chunks=[1, 36, 33])
    assert np.array_equal(u, ref_u) and np.array_equal(up, ref_up)
    (u, up), _ = _slabs(P, v, 70, u0, up0, src, G, halo, graphs=1, chunks=[70])
    assert np.array_equal(u, ref_u) and np.array_equal(up, ref_up)
    (u, up), t_direct = _slabs(P, v, 70, u0, up0, src, G, halo, graphs=0, chunks=[1, 36, 33])
    assert np.array_equal(u, ref_u) and np.array_equal(up, ref_up)
    print(f"G={G} halo={halo}: enqueue of 33 steps: graphs {t_graph:.3f} ms, direct {t_direct:.3f} ms")
    if G >= 4:  # 2 replays + 1 direct step vs 33 direct steps of G slabs
        assert t_graph < 0.5 * t_direct, (t_graph, t_direct)


# ----------------------------------------------------------------------------- multi-step (kind 6)
def _ms_ids(P):
    return [t for t in range(P.rtm_num_tiles()) if (P.rtm_tile_name(t) or "").startswith("ms")]


def _run_tile(P, v, chunks, u0, up0, src, tile, zchunk=0, shots=1, order=0, profiling=0):
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, shots=shots) as sim:
        sim.set_tile(tile)
        P.rtm_set_zchunk(sim.h, zchunk)
        P.rtm_set_option(sim.h, P.RTM_OPT_SHOT_ORDER, order)
        P.rtm_set_profiling(sim.h, profiling)
        sim.set_velocity(v)
        for k in range(shots):
            for (x, y, z, w) in src:
                P.rtm_inject_source_shot(sim.h, k, (x + 7 * k) % nx, y, z, w)
        if u0 is not None:
            sim.set_fields(np.stack([u0] * shots) if shots > 1 else u0,
                           np.stack([up0] * shots) if shots > 1 else up0)
        for c in chunks:
            sim.step(c)
        return sim.read_fields(), P.rtm_launch_count(sim.h)


@pytest.mark.parametrize("zchunk", [0, 6, 11])
def test_multistep_launch_bitwise_equals_single_steps(P, zchunk):
    """k_stream<..., MS> runs many time steps in ONE cooperative launch, each work unit waiting
    only for its face-neighbour units' flags: the bits equal one k_stream launch per step
    (ragged grid, sources on tile / chunk edges and the z ends, odd starts, 1-step calls)."""
    shape = (45, 67, 100)
    rng = np.random.default_rng(404)
    v = rng.uniform(1500, 4300, shape).astype(np.float32)
    u0, up0 = ri.random_fields(shape, seed=404)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 60)
    src = [(0, 0, 0, w), (99, 66, 44, -w), (63, 29, 11, w), (64, 30, 12, 0.5 * w), (31, 7, 22, w),
           (32, 60, 33, -w)]
    ref, _ = _run_tile(P, v, [37], u0, up0, src, 35, zchunk=zchunk)
    for t in _ms_ids(P):
        for chunks in ([37], [1, 1, 35], [3, 34]):
            got, launches = _run_tile(P, v, chunks, u0, up0, src, t, zchunk=zchunk)
            assert np.array_equal(got[0], ref[0]), (P.rtm_tile_name(t), chunks)
            assert np.array_equal(got[1], ref[1]), (P.rtm_tile_name(t), chunks)
            assert launches == len(chunks)  # one launch per rtm_step call


@pytest.mark.parametrize("order", [1, 2])
def test_multistep_batched_shots_bitwise(P, order):
    shape = (30, 40, 64)
    rng = np.random.default_rng(9)
    v = rng.uniform(1500, 4300, shape).astype(np.float32)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 40)
    src = [(20, 20, 15, w), (3, 39, 29, -w)]
    ref, _ = _run_tile(P, v, [23], None, None, src, 1, shots=3, order=order)
    for t in _ms_ids(P)[:2]:
        got, _ = _run_tile(P, v, [4, 19], None, None, src, t, shots=3, order=order)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]), P.rtm_tile_name(t)


def test_multistep_c2_full_run_vs_oracle_and_profiled(P):
    """C2 (256^3, 500 steps) with the multi-step kernel: within the north-star tolerance of the
    fp32 oracle, bitwise equal to per-step launches; the profiled path (events around each
    launch) gives the same bits."""
    import oracle
    cfg = ri.make_config(2)
    v = cfg.velocity()
    src = cfg.sources()
    ms = _ms_ids(P)[0]
    got, launches = _run_tile(P, v, [cfg.steps], None, None, src, ms)
    assert launches == 1
    ref, _ = _run_tile(P, v, [cfg.steps], None, None, src, 35)
    assert np.array_equal(got[0], ref[0])
    prof, _ = _run_tile(P, v, [cfg.steps], None, None, src, ms, profiling=1)
    assert np.array_equal(prof[0], ref[0])
    orc = oracle.run(v, cfg.dx, cfg.dt, C32, cfg.steps, sources=src)
    m = float(np.abs(orc).max())
    assert float(np.abs(got[0].astype(np.float64) - orc).max()) <= 1e-4 * m


# ----------------------------------------------------------------------------- z sweep direction
def test_alternating_z_sweep_is_bitwise(P):
    """RTM_OPT_ZDIR = 1: k_stream sweeps z downward on odd-parity steps (the register queue is
    filled in sweep order; the z pair sums are commutative), bitwise equal to upward sweeps for
    every k_stream variant (single- and multi-step), with z-chunks, sources and odd starts."""
    shape = (41, 45, 76)
    rng = np.random.default_rng(808)
    v = rng.uniform(1500, 4300, shape).astype(np.float32)
    u0, up0 = ri.random_fields(shape, seed=808)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 40)
    src = [(0, 0, 0, w), (75, 44, 40, -w), (33, 20, 13, w), (34, 21, 27, 0.5 * w)]
    nz, ny, nx = shape
    ref, _ = _run_tile(P, v, [19], u0, up0, src, 35)
    ids = [t for t in range(1, P.rtm_num_tiles()) if (P.rtm_tile_name(t) or "").startswith(("stream", "ms", "s2r"))]
    for t in ids:
        for zc, zd in ((0, 1), (7, 1), (7, 2), (5, 3), (6, 4), (5, 6)):
            with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
                sim.set_tile(t)
                P.rtm_set_zchunk(sim.h, zc)
                P.rtm_set_option(sim.h, P.RTM_OPT_ZDIR, zd)
                sim.set_velocity(v)
                for s in src:
                    sim.inject_source(*s)
                sim.set_fields(u0, up0)
                sim.step(1)
                sim.step(18)
                u, up = sim.read_fields()
            assert np.array_equal(u, ref[0]) and np.array_equal(up, ref[1]), (P.rtm_tile_name(t), zc, zd)


@pytest.mark.parametrize("halo", [0, 1, 2, 3])
def test_alternating_z_sweep_with_slabs_is_bitwise(P, halo):
    v, u0, up0, src = _case(91)
    ref_u, ref_up = _single(P, v, 20, u0, up0, src)
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=[0, 0, 0]) as sim:
        P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
        P.rtm_set_option(sim.h, P.RTM_OPT_ZDIR, 3)
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        sim.step(3)
        sim.step(17)
        u, up = sim.read_fields()
    assert np.array_equal(u, ref_u) and np.array_equal(up, ref_up)


# ----------------------------------------------------------------------------- peer-context errors
def test_peer_context_contract(P):
    """rtm_create_peer: world 1 behaves like a single-GPU context (bitwise); a rank with
    neighbours refuses to step before its neighbours' records are imported, validates records
    (magic, grid, world, rank, nzl) before opening anything, rejects halo mode 0 (no NCCL) and
    fails collective calls without a rank barrier."""
    v, u0, up0, src = _case(61, (30, 20, 32))
    ref_u, _ = _single(P, v, 9, u0, up0, src)
    nz, ny, nx = v.shape
    h = P.rtm_create_peer(nx, ny, nz, 10.0, 1e-3, C32, 0, 1, 0)
    try:
        assert P.rtm_get_option(h, P.RTM_OPT_HALO_MODE) == 3
        P.rtm_set_velocity(h, v)
        for s in src:
            P.rtm_inject_source(h, *s)
        P.rtm_set_fields(h, u0, up0)
        P.rtm_step(h, 9)
        u = np.empty_like(u0)
        P.rtm_read_field(h, u)
        assert np.array_equal(u, ref_u)
    finally:
        P.rtm_destroy(h)
    h0 = P.rtm_create_peer(nx, ny, nz, 10.0, 1e-3, C32, 0, 2, 0)
    h1 = P.rtm_create_peer(nx + 4, ny, nz, 10.0, 1e-3, C32, 1, 2, 0)  # another grid
    try:
        assert P.rtm_get_dims(h0) == (nx, ny, 15, 1)
        P.rtm_set_velocity(h0, v[:15])
        with pytest.raises(P.RtmError) as e:
            P.rtm_step(h0, 1)
        assert e.value.code == P.RTM_ESTATE
        with pytest.raises(P.RtmError) as e:   # rank 0 of 2 needs a hi record
            P.rtm_ipc_import(h0, None, None)
        assert e.value.code == P.RTM_EINVAL
        with pytest.raises(P.RtmError) as e:
            P.rtm_ipc_import(h0, None, bytes(512))
        assert e.value.code == P.RTM_EINVAL and "not an RTM IPC record" in str(e.value)
        with pytest.raises(P.RtmError) as e:   # rank 1's record, but of a different grid
            P.rtm_ipc_import(h0, None, P.rtm_ipc_export(h1))
        assert e.value.code == P.RTM_EINVAL and "grid" in str(e.value)
        with pytest.raises(P.RtmError) as e:
            P.rtm_set_option(h0, P.RTM_OPT_HALO_MODE, 0)
        assert e.value.code == P.RTM_EINVAL
        with pytest.raises(P.RtmError) as e:   # collective, no rank barrier installed
            P.rtm_reset(h0)
        assert e.value.code in (P.RTM_ESTATE, P.RTM_EINVAL)
    finally:
        P.rtm_destroy(h0)
        P.rtm_destroy(h1)


def test_autotune_in_pull_mode_and_host_ordered_in_process(P):
    """Halo mode 3 in-process through the collective restarts: autotune (new flag generation),
    reset, resume; host-ordered stepping interleaved with device-ordered stepping."""
    v, u0, up0, src = _case(123, (60, 33, 72))
    ref_u, ref_up = _single(P, v, 26, u0, up0, src)
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=[0, 0, 0, 0]) as sim:
        P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, 3)
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        sim.step(4)
        P.rtm_autotune(sim.h, 3, tiles=[35, 10, 1], zchunks=[0, 0, 5])
        sim.step(7)
        P.rtm_set_option(sim.h, P.RTM_OPT_HOST_ORDERED, 1)
        sim.step(6)
        P.rtm_set_option(sim.h, P.RTM_OPT_HOST_ORDERED, 0)
        sim.step(9)
        u, up = sim.read_fields()
    assert np.array_equal(u, ref_u) and np.array_equal(up, ref_up)


def test_c_example_matches_the_oracle(P, tmp_path):
    """examples/rtm_c1.c (plain C through include/rtm.h) runs C1 on the GPU; its max|u| equals
    the fp32 oracle's within the north-star tolerance."""
    import re
    import subprocess
    import sys
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent))
    from test_abi_cpu import _build_c_example
    import oracle
    exe = _build_c_example(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    m = float(re.search(r"max\|u\| = ([0-9.eE+-]+)", r.stdout).group(1))
    cfg = ri.make_config(1)
    ref = oracle.run(cfg.velocity(), cfg.dx, cfg.dt, C32, cfg.steps, sources=cfg.sources())
    mref = float(np.abs(ref).max())
    assert abs(m - mref) <= 1e-4 * mref, (m, mref)


@pytest.mark.parametrize("halo", [0, 1, 2, 3])
def test_two_row_and_u11_variants_in_slab_modes(P, halo):
    """The tuner may pick a two-row (k_stream2) or U = 11 variant for a slab context: boundary
    2-range launches (modes 0, 3) and epilogue pushes (modes 1, 2) stay bitwise equal to G = 1."""
    v, u0, up0, src = _case(202, (50, 30, 68))
    ref_u, ref_up = _single(P, v, 13, u0, up0, src)
    nz, ny, nx = v.shape
    ids = [t for t in range(1, P.rtm_num_tiles())
           if (P.rtm_tile_name(t) or "").startswith("s2r") or (P.rtm_tile_name(t) or "").endswith("u11")]
    for t in ids:
        with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=[0, 0, 0]) as sim:
            sim.set_tile(t)
            P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
            sim.set_velocity(v)
            for s in src:
                sim.inject_source(*s)
            sim.set_fields(u0, up0)
            sim.step(13)
            u, up = sim.read_fields()
        assert np.array_equal(u, ref_u) and np.array_equal(up, ref_up), P.rtm_tile_name(t)


@pytest.mark.parametrize("halo", [0, 1, 2, 3])
def test_slab_share_bitwise(P, halo):
    """RTM_OPT_SLAB_SHARE: slabs sharing a device split its SMs (smaller persistent grids,
    z-chunks chosen for the share) — bitwise equal to G = 1, with and without graphs."""
    v, u0, up0, src = _case(303, (64, 33, 72))
    ref_u, ref_up = _single(P, v, 37, u0, up0, src)
    nz, ny, nx = v.shape
    for graphs in (0, 1):
        with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=[0] * 4) as sim:
            P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
            P.rtm_set_option(sim.h, P.RTM_OPT_SLAB_SHARE, 1)
            P.rtm_set_option(sim.h, P.RTM_OPT_GRAPHS, graphs)
            sim.set_velocity(v)
            for s in src:
                sim.inject_source(*s)
            sim.set_fields(u0, up0)
            sim.step(37)
            u, up = sim.read_fields()
        assert np.array_equal(u, ref_u) and np.array_equal(up, ref_up), graphs


@pytest.mark.parametrize("zchunk", [2, 3, 5])
def test_multistep_chunks_shorter_than_the_halo(P, zchunk):
    """Multi-step launches with z-chunks shorter than the 5-plane halo: a unit's boxes then reach
    two or more chunks up and down, all of which must have published the previous step.  (A round-2
    stress run found the kernel waiting only for chunks c±1: 517 of 2304 runs differed; the wait now
    covers every chunk the halo intersects — `profiles/ms_stress_r02.log`.)"""
    rng = np.random.default_rng(31 + zchunk)
    shape = (46, 57, 55)
    v = rng.uniform(1500, 4300, shape).astype(np.float32)
    u0, up0 = ri.random_fields(shape, seed=zchunk)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 40)
    nz, ny, nx = shape
    src = [(0, 0, 0, w), (nx - 1, ny - 1, nz - 1, -w), (nx // 2, ny // 3, nz // 2, w)]
    ref, _ = _run_tile(P, v, [23], u0, up0, src, 35)
    for t in _ms_ids(P):
        for rep in range(3):
            got, _ = _run_tile(P, v, [1, 22], u0, up0, src, t, zchunk=zchunk)
            assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]), (P.rtm_tile_name(t), rep)
