"""Per-step time of k_resident vs grid size (tiny grids ~ the grid-barrier cost)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1310_8232_b200 as P  # noqa: E402
import rtm_inputs as ri  # noqa: E402

names = {P.rtm_tile_name(t): t for t in range(P.rtm_num_tiles())}
for n in (16, 32, 64, 96):
    v = np.full((n, n, n), 2000.0, np.float32)
    for name in ("resident512x1", "resident256x2", "resident128x4", "stream32x28k8d4u4"):
        with P.Simulation(n, n, n, 10.0, 1e-3, ri.COEFFS_F32) as sim:
            sim.set_tile(names[name])
            sim.set_velocity(v)
            sim.step(200)
            best = 1e9
            for _ in range(3):
                sim.step(1000)
                best = min(best, P.rtm_last_elapsed_ms(sim.h))
            print(f"{n}^3 {name}: {1e3 * best / 1000:.2f} us/step, {n**3 * 1000 / best / 1e6:.1f} Gpt/s", flush=True)
