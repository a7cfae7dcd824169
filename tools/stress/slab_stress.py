"""Stress of in-process z-slabs on one GPU (GPU only; run from the repo root):
40 random grids, G = 2-8 slabs at 10-11 planes each, halo modes 0-3, random z direction, host
ordering and graphs, 4-call step schedules; every run must be bitwise equal to one slab.
Result: profiles/slab_stress_r02.log.    python tools/stress/slab_stress.py
"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1310_8232_b200 as P, rtm_inputs as ri
C32 = ri.COEFFS_F32
rng0 = np.random.default_rng(77)
runs = fails = 0
for case in range(40):
    G = int(rng0.integers(2, 9))
    nz = int(rng0.integers(10 * G, 10 * G + 12))
    ny, nx = int(rng0.integers(8, 50)), int(rng0.integers(8, 90))
    shape = (nz, ny, nx)
    rng = np.random.default_rng(case)
    v = rng.uniform(1500, 4300, shape).astype(np.float32)
    u0, up0 = ri.random_fields(shape, seed=case)
    w = ri.source_samples(3000.0, 1e-3, 15.0, 60)
    src = [(int(rng.integers(nx)), int(rng.integers(ny)), int(rng.integers(nz)), w) for _ in range(3)]
    steps = [int(x) for x in rng.integers(1, 9, size=4)]
    n = sum(steps)
    def run(devices, halo=0, zdir=2, ho=0, graphs=1):
        with P.Simulation(nx, ny, nz, 10.0, 1e-3, C32, devices=devices) as sim:
            if halo: P.rtm_set_option(sim.h, P.RTM_OPT_HALO_MODE, halo)
            P.rtm_set_option(sim.h, P.RTM_OPT_ZDIR, zdir)
            P.rtm_set_option(sim.h, P.RTM_OPT_GRAPHS, graphs)
            if halo: P.rtm_set_option(sim.h, P.RTM_OPT_HOST_ORDERED, ho)
            sim.set_velocity(v)
            for s in src: sim.inject_source(*s)
            sim.set_fields(u0, up0)
            for k in steps: sim.step(k)
            return sim.read_field()
    ref = run(None)
    for halo in (0, 1, 2, 3):
        for rep in range(2):
            runs += 1
            zd = int(rng0.integers(0, 8)); ho = int(rng0.integers(0, 2)) if halo >= 2 else 0
            out = run([0] * G, halo, zd, ho, int(rng0.integers(0, 2)))
            if not np.array_equal(out, ref):
                fails += 1
                print("FAIL", shape, G, halo, zd, ho, steps, flush=True)
print("runs", runs, "fails", fails)
