"""Locate a two-step vs single-step mismatch: the failing parity case, stepped 1..9."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1310_8232_b200 as P  # noqa: E402
import rtm_inputs as ri  # noqa: E402

C32 = ri.COEFFS_F32
nz, ny, nx = 23, 150, 200
rng = np.random.default_rng(77)
v = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
u0, up0 = ri.random_fields(v.shape, seed=77)
w = ri.source_samples(3000.0, 1e-3, 15.0, 9)
src_all = [(5, 0, 0, w), (199, 149, 22, -w), (130, 36, 11, w), (64, 37, 3, 0.5 * w),
           (63, 38, 19, w), (100, 75, 12, w), (196, 112, 7, -w), (17, 113, 7, w)]


def run(steps, tile, src):
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
        sim.set_tile(tile)
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        sim.step(steps)
        return sim.read_fields()


tiles = [int(a) for a in sys.argv[1:]] or [38]
for t in tiles:
    for srcset in ("all", "none"):
        src = src_all if srcset == "all" else []
        for steps in (2, 4, 9):
            ref = run(steps, 35, src)
            got = run(steps, t, src)
            for name, a, b in (("u", got[0], ref[0]), ("up", got[1], ref[1])):
                d = a != b
                if d.any():
                    z, y, x = np.nonzero(d)
                    print(P.rtm_tile_name(t), srcset, steps, name, int(d.sum()), "z", z.min(), z.max(),
                          "y", y.min(), y.max(), "x", x.min(), x.max(), "maxdiff", float(np.abs(a - b).max()),
                          flush=True)
                else:
                    print(P.rtm_tile_name(t), srcset, steps, name, "OK", flush=True)
