"""Repeat the two-step vs single-step bitwise comparison per tb2 variant and report mismatch
statistics (deterministic bug vs timing-dependent race)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1310_8232_b200 as P  # noqa: E402
import rtm_inputs as ri  # noqa: E402

C32 = ri.COEFFS_F32


def run(v, steps, u0, up0, src, tile, tb_ctas=0):
    nz, ny, nx = v.shape
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
        sim.set_tile(tile)
        P.rtm_set_option(sim.h, P.RTM_OPT_TB_CTAS, tb_ctas)
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        sim.step(steps)
        return sim.read_fields()


shapes = [(23, 150, 200), (64, 300, 512)]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
tbs = [t for t in range(P.rtm_num_tiles()) if P.rtm_tile_name(t).startswith("tb2")]
for shape in shapes:
    rng = np.random.default_rng(77)
    v = rng.uniform(1500, 4300, shape).astype(np.float32)
    u0, up0 = ri.random_fields(shape, seed=77)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 9)
    src = [(5, 0, 0, w), (100, 75, 12, w)]
    ref = run(v, 8, u0, up0, src, 35)
    for t in tbs:
        for ctas in (0, 24):
            bad = []
            for r in range(reps):
                u, up = run(v, 8, u0, up0, src, t, ctas)
                for name, a, b in (("u", u, ref[0]), ("up", up, ref[1])):
                    d = a != b
                    if d.any():
                        z, y, x = np.nonzero(d)
                        bad.append(f"{name}: {d.sum()} pts z[{z.min()},{z.max()}] y[{y.min()},{y.max()}] "
                                   f"x[{x.min()},{x.max()}] maxdiff {np.abs(a - b).max():.3g}")
            print(shape, P.rtm_tile_name(t), "ctas", ctas, "OK" if not bad else bad[:3], flush=True)
