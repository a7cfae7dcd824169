"""Stress of the cooperative multi-step kernels (ms* variants, GPU only): random grids whose
z-chunks may be shorter than the 5-plane halo, random chunk counts and step counts; bitwise vs
the one-step path.  Result: profiles/ms_stress_r02.log.    python tools/stress/ms_stress.py
"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1310_8232_b200 as P, rtm_inputs as ri
C32 = ri.COEFFS_F32
fails = 0; runs = 0
rng0 = np.random.default_rng(5)
ms = [t for t in range(P.rtm_num_tiles()) if (P.rtm_tile_name(t) or "").startswith("ms")]
for case in range(12):
    shape = (int(rng0.integers(20, 60)), int(rng0.integers(20, 70)), int(rng0.integers(30, 140)))
    rng = np.random.default_rng(case)
    v = rng.uniform(1500, 4300, shape).astype(np.float32)
    u0, up0 = ri.random_fields(shape, seed=case)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 40)
    nz, ny, nx = shape
    src = [(0, 0, 0, w), (nx - 1, ny - 1, nz - 1, -w), (nx // 2, ny // 3, nz // 2, w)]
    def run(t, zc, zd, chunks):
        with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32) as sim:
            sim.set_tile(t); P.rtm_set_zchunk(sim.h, zc); P.rtm_set_option(sim.h, P.RTM_OPT_ZDIR, zd)
            sim.set_velocity(v)
            for s in src: sim.inject_source(*s)
            sim.set_fields(u0, up0)
            for c in chunks: sim.step(c)
            return sim.read_fields()[0]
    ref = run(35, 0, 0, (23,))
    for t in ms:
        for zc in (0, 3, 5, 7):
            for zd in (0, 2, 4, 6):
                for chunks in ((23,), (1, 22)):
                    runs += 1
                    if not np.array_equal(run(t, zc, zd, chunks), ref):
                        fails += 1
                        print("FAIL", shape, P.rtm_tile_name(t), zc, zd, chunks, flush=True)
print("runs", runs, "fails", fails)
