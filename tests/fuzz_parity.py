"""Randomised parity fuzz (GPU): random ragged shapes, velocities, initial conditions, sources
and step counts; every kernel variant must equal the naive kernel bitwise and the fp32 oracle
within the one-step tolerance scaled by the step count (random z sweep direction, RTM_OPT_ZDIR);
slab decompositions (halo modes 0-3, host-ordered or not, graphs or not) must equal the
single-slab result bitwise.  Usage: python tests/fuzz_parity.py [cases] [seed]"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402  (test infrastructure: the fuzz is a test)
import paper_1310_8232_b200 as P  # noqa: E402
import rtm_inputs as ri  # noqa: E402

C32 = ri.COEFFS_F32


def run(v, steps, u0, up0, src, tile=None, devices=None, halo=0, tb_ctas=0, asyn=False, zdir=0,
        host_ordered=0, graphs=1):
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=devices) as sim:
        P.rtm_set_option(sim.h, P.RTM_OPT_ZDIR, zdir)
        P.rtm_set_option(sim.h, P.RTM_OPT_GRAPHS, graphs)
        if halo:
            P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
            P.rtm_set_option(sim.h, P.RTM_OPT_HOST_ORDERED, host_ordered)
        if tile is not None:
            sim.set_tile(tile)
        if tb_ctas:
            P.rtm_set_option(sim.h, P.RTM_OPT_TB_CTAS, tb_ctas)
        if asyn:
            P.rtm_set_velocity_async(sim.h, v)
        else:
            sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        if asyn:
            out = np.empty(v.shape, np.float32)
            P.rtm_step_async(sim.h, steps)
            P.rtm_read_field_async(sim.h, out)
            P.rtm_sync(sim.h)
            return out
        sim.step(steps)
        return sim.read_field()


def run_shots(v, steps, u0, up0, src, tile):
    """Two shots: shot 0 = (u0, up0, src), shot 1 = (up0, u0, no source)."""
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, shots=2) as sim:
        sim.set_tile(tile)
        sim.set_velocity(v)
        for (x, y, z, w) in src:
            P.rtm_inject_source_shot(sim.h, 0, x, y, z, w)
        sim.set_fields(np.stack([u0, up0]), np.stack([up0, u0]))
        sim.step(steps)
        return sim.read_field()


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
    scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0  # size multiplier
    ntiles = P.rtm_num_tiles()
    fails = 0
    t0 = time.time()
    for c in range(cases):
        nz = int(rng.integers(1, int(41 * scale) + 1))
        ny = int(rng.integers(1, int(71 * scale) + 1))
        nx = int(rng.integers(1, int(141 * scale) + 1))
        steps = int(rng.integers(1, int(10 * scale) + 1))
        v = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
        u0, up0 = ri.random_fields(v.shape, seed=int(rng.integers(1 << 30)))
        src = []
        for _ in range(int(rng.integers(0, 5))):
            w = ri.source_samples(float(rng.uniform(1500, 4300)), 1e-3, 15.0, steps)
            src.append((int(rng.integers(nx)), int(rng.integers(ny)), int(rng.integers(nz)), w))
        ref = oracle.run(v, 10.0, 1e-3, C32, steps, u0=u0, up0=up0, sources=src)
        base = run(v, steps, u0, up0, src, tile=0)
        m = float(np.abs(ref).max()) or 1.0
        err = float(np.abs(base.astype(np.float64) - ref).max()) / m
        bad = []
        if err > 1e-5 * max(steps, 1) * 2:
            bad.append(f"naive vs oracle {err:.2e}")
        zdir = int(rng.integers(0, 8))
        for t in range(1, ntiles):
            out = run(v, steps, u0, up0, src, tile=t, zdir=zdir)
            if not np.array_equal(out, base):
                d = out != base
                bad.append(f"{P.rtm_tile_name(t)} zdir={zdir}: {int(d.sum())} pts differ")
        tbs = [t for t in range(ntiles) if (P.rtm_tile_name(t) or "").startswith("tb2")]
        for t in tbs[:1]:  # multi-band two-step plans
            ctas = int(rng.integers(1, 13))
            out = run(v, steps, u0, up0, src, tile=t, tb_ctas=ctas)
            if not np.array_equal(out, base):
                bad.append(f"{P.rtm_tile_name(t)} tb_ctas={ctas}")
        out = run(v, steps, u0, up0, src, asyn=True)
        if not np.array_equal(out, base):
            bad.append("async pipeline")
        t_sh = int(rng.integers(0, ntiles))
        sh = run_shots(v, steps, u0, up0, src, t_sh)
        other = run(v, steps, up0, u0, [], tile=0)
        if not (np.array_equal(sh[0], base) and np.array_equal(sh[1], other)):
            bad.append(f"2 shots ({P.rtm_tile_name(t_sh)})")
        for G in (2, 3):
            if nz >= 10 * G:
                for halo in (0, 1, 2, 3):
                    ho, gr = int(rng.integers(0, 2)), int(rng.integers(0, 2))
                    out = run(v, steps, u0, up0, src, devices=[0] * G, halo=halo, zdir=zdir,
                              host_ordered=ho, graphs=gr)
                    if not np.array_equal(out, base):
                        bad.append(f"slabs G={G} halo={halo} host_ordered={ho} graphs={gr}")
        status = "OK" if not bad else "FAIL " + "; ".join(bad[:4])
        fails += bool(bad)
        print(f"case {c:3d} shape=({nz},{ny},{nx}) steps={steps} src={len(src)} oracle_err={err:.1e} {status}",
              flush=True)
    print(f"{cases} cases, {fails} failing, {time.time() - t0:.0f} s", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
