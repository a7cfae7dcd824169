"""Stress of cross-process peer contexts sharing one GPU (GPU only): 8 random grids x world
2/3/4 x halo modes 2/3, launched with torch.distributed.run (gloo bootstrap, CUDA IPC records,
host-ordered steps); the gathered field must be bitwise equal to one in-process context.
Result: profiles/peer_stress_r02.log.    python tools/stress/peer_stress.py
"""
import os, sys, subprocess, socket, tempfile
from pathlib import Path
ROOT = Path(os.getcwd()); sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tools" / "stress"))
import numpy as np
import paper_1310_8232_b200 as P, rtm_inputs as ri
import importlib.util
fails = runs = 0
for seed in range(8):
    for world in (2, 3, 4):
        for halo in (2, 3):
            os.environ["WORLD_SIZE"] = str(world)
            spec = importlib.util.spec_from_file_location("w", ROOT / "tools" / "stress" / "peer_stress_worker.py")
            W = importlib.util.module_from_spec(spec); spec.loader.exec_module(W)
            (nz, ny, nx), v, u0, up0, src, steps = W.case(seed)
            with P.Simulation(nx, ny, nz, 10.0, 1e-3, ri.COEFFS_F32) as sim:
                sim.set_velocity(v)
                for s in src: sim.inject_source(*s)
                sim.set_fields(u0, up0); sim.step(sum(steps)); ref = sim.read_field()
            with socket.socket() as s_: s_.bind(("127.0.0.1", 0)); port = s_.getsockname()[1]
            td = Path(tempfile.mkdtemp())
            env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1"); env.pop("WORLD_SIZE")
            r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                                "--master-addr", "127.0.0.1", "--master-port", str(port),
                                str(ROOT / "tools" / "stress" / "peer_stress_worker.py"), str(td), str(halo), str(seed)],
                               capture_output=True, text=True, timeout=300, env=env)
            runs += 1
            if r.returncode != 0:
                fails += 1; print("ERROR", seed, world, halo, r.stderr[-800:], flush=True); continue
            got = np.concatenate([np.load(td / f"rank{k}.npy") for k in range(world)])
            ok = np.array_equal(got, ref)
            fails += (not ok)
            print(("OK" if ok else "FAIL"), seed, world, halo, (nz, ny, nx), steps, flush=True)
print("runs", runs, "fails", fails)
