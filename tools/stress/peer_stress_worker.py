"""One rank of tools/stress/peer_stress.py: argv = out_dir halo_mode seed."""
import os, sys
from pathlib import Path
ROOT = Path(os.environ["GRAFT_REPO_ROOT"] if "GRAFT_REPO_ROOT" in os.environ else os.getcwd())
sys.path.insert(0, str(ROOT))
import numpy as np
import rtm_inputs as ri

def case(seed):
    rng = np.random.default_rng(seed)
    world = int(os.environ["WORLD_SIZE"])
    nz = int(rng.integers(10 * world, 10 * world + 15)); ny = int(rng.integers(8, 40)); nx = int(rng.integers(8, 70))
    v = rng.uniform(1500, 4300, (nz, ny, nx)).astype(np.float32)
    u0, up0 = ri.random_fields((nz, ny, nx), seed=seed)
    w = ri.source_samples(2500.0, 1e-3, 15.0, 60)
    src = [(int(rng.integers(nx)), int(rng.integers(ny)), int(rng.integers(nz)), w) for _ in range(4)]
    steps = [int(x) for x in rng.integers(1, 8, size=3)]
    return (nz, ny, nx), v, u0, up0, src, steps

def main():
    out_dir, halo, seed = Path(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    import torch, torch.distributed as dist
    import paper_1310_8232_b200 as P
    from paper_1310_8232_b200 import dist as pd
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo"); torch.cuda.set_device(0)
    (nz, ny, nx), v, u0, up0, src, steps = case(seed)
    h = pd.create_peer(nx, ny, nz, 10.0, 1e-3, ri.COEFFS_F32, rank, world, 0, halo_mode=halo, host_ordered=True)
    z0, nzl = P.rtm_slab_range(nz, world, rank); sl = slice(z0, z0 + nzl)
    P.rtm_set_option(h, P.RTM_OPT_ZDIR, seed % 8)
    P.rtm_set_velocity(h, v[sl])
    for s in src: P.rtm_inject_source(h, *s)
    P.rtm_set_fields(h, u0[sl], up0[sl])
    for k in steps: P.rtm_step(h, k)
    u = np.empty((nzl, ny, nx), np.float32); P.rtm_read_field(h, u)
    np.save(out_dir / f"rank{rank}.npy", u)
    dist.barrier(); P.rtm_destroy(h); dist.destroy_process_group()

if __name__ == "__main__":
    main()
