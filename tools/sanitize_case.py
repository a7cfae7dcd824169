"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck): every kernel family
(naive, k_tiled, k_stream with and without the u_prev/C ring, U = 11, the two-row k_stream2,
the cooperative multi-step and resident kernels, the two-step k_tb2s, batched shots, slabs
with copy, fused, flag-protocol and pull halo modes, the asynchronous pipeline) on ragged grids
of 16^3-64^3."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1310_8232_b200 as P  # noqa: E402
import rtm_inputs as ri  # noqa: E402


def run(shape, tile, steps=3, shots=1, devices=None, halo=0, tb_ctas=0):
    nz, ny, nx = shape
    v = np.full(shape, 2500.0, np.float32)
    u0, up0 = ri.random_fields(shape, seed=1)
    w = np.ones(steps, np.float32)
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, ri.COEFFS_F32, devices=devices, shots=shots) as sim:
        if halo:
            P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
        if tile is not None:
            sim.set_tile(tile)
        if tb_ctas:
            P.rtm_set_option(sim.h, P.RTM_OPT_TB_CTAS, tb_ctas)
        sim.set_velocity(v)
        sim.inject_source(nx // 2, ny // 2, nz // 2, w)
        if shots > 1:
            sim.set_fields(np.stack([u0] * shots), np.stack([up0] * shots))
        else:
            sim.set_fields(u0, up0)
        sim.step(steps)
        out = sim.read_field()
    assert np.isfinite(out).all()


if __name__ == "__main__":
    names = {P.rtm_tile_name(i): i for i in range(P.rtm_num_tiles())}
    picks = ["naive", "tma64x16k10", "stream64x16k8d4u11", "stream64x14k10d5u4", "stream64x16k9d0u4",
             "stream128x7k8d4u4", "stream64x30k10d6u4", "stream64x30k10d6u11", "stream128x7k8d4u11",
             "s2r64x28k10d6", "ms128x7k8d4u4", "ms64x30k10d6u11", "resident512x1"]
    picks = [n for n in picks if n in names]
    for name in picks:
        run((21, 37, 68), names[name])
        run((16, 16, 16), names[name])
    run((19, 30, 64), names["stream64x16k8d4u11"], shots=3)
    run((40, 24, 32), None, devices=[0, 0])
    run((40, 24, 32), None, devices=[0, 0, 0], halo=1)
    run((40, 24, 32), None, devices=[0, 0, 0], halo=2)
    run((40, 24, 32), None, devices=[0, 0, 0], halo=3)
    tb = [i for n, i in names.items() if n.startswith("tb2s_")][0]
    run((21, 37, 68), tb, steps=5)
    run((13, 61, 132), tb, steps=4, tb_ctas=6)       # several y-bands
    shape = (12, 20, 40)
    v = np.full(shape, 2500.0, np.float32)
    out = np.empty(shape, np.float32)
    with P.Simulation(40, 20, 12, 10.0, 1e-3, ri.COEFFS_F32) as sim:   # asynchronous pipeline
        for _ in range(2):
            P.rtm_set_velocity_async(sim.h, v)
            P.rtm_reset(sim.h)
            P.rtm_step_async(sim.h, 3)
            P.rtm_read_field_async(sim.h, out)
        P.rtm_sync(sim.h)
    print("sanitize cases done")
