"""One rank of a peer-context run (rtm_create_peer: CUDA-IPC halo data plane, no NCCL),
launched by tests/test_gpu_xproc.py through torch.distributed.run.  Every rank uses the same
GPU (cuda:0) and RTM_OPT_HOST_ORDERED=1, so no device-side wait ever spans processes (ranks
on one GPU must not wait on each other on the device; B200_PROFILING.md); the IPC mappings,
the flag words, the pushes / pulls across processes and the collective restarts are real.

    worker.py OUT_DIR HALO_MODE

Writes OUT_DIR/rank{r}.npz with the slab's u^n and u^{n-1} at the end of the schedule."""
from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import rtm_inputs as ri  # noqa: E402

SHAPE = (60, 40, 72)  # nz, ny, nx: slabs of 30 / 20 planes at world 2 / 3
STEPS = (7, 4, 9)     # schedule: run a, reset + run b, resume from the saved state + run c


def case():
    rng = np.random.default_rng(1310)
    v = rng.uniform(1500, 4300, SHAPE).astype(np.float32)
    u0, up0 = ri.random_fields(SHAPE, seed=8232)
    w = ri.source_samples(2500.0, 1e-3, 15.0, 40)
    nz = SHAPE[0]
    # sources on every slab boundary of world 2 and 3 (planes 19/20, 29/30, 39/40) and the ends
    src = [(5, 6, 20, w), (7, 8, 19, -w), (9, 3, 30, w), (11, 12, 29, 0.5 * w), (13, 14, 40, w),
           (2, 2, 39, -w), (1, 1, 0, w), (70, 38, nz - 1, w)]
    return v, u0, up0, src


def main():
    out_dir, halo = Path(sys.argv[1]), int(sys.argv[2])
    import torch
    import torch.distributed as dist
    import paper_1310_8232_b200 as P
    from paper_1310_8232_b200 import dist as pd
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    v, u0, up0, src = case()
    nz, ny, nx = SHAPE
    h = pd.create_peer(nx, ny, nz, 10.0, 1e-3, ri.COEFFS_F32, rank, world, 0, halo_mode=halo,
                       host_ordered=True)
    z0, nzl = P.rtm_slab_range(nz, world, rank)
    sl = slice(z0, z0 + nzl)
    assert P.rtm_get_dims(h) == (nx, ny, nzl, 1)
    P.rtm_set_velocity(h, v[sl])
    for (x, y, z, w) in src:
        P.rtm_inject_source(h, x, y, z, w)
    P.rtm_set_fields(h, u0[sl], up0[sl])                 # collective (halo pull)
    a, b, c = STEPS
    P.rtm_step(h, a)
    u = np.empty((nzl, ny, nx), np.float32)
    up = np.empty_like(u)
    P.rtm_read_fields(h, u, up)
    P.rtm_reset(h)                                       # collective restart
    P.rtm_step(h, b)
    P.rtm_set_fields(h, u, up)                           # resume from step a
    P.rtm_set_step_count(h, a)                           # collective, new flag generation
    P.rtm_step(h, c)
    res, _ = P.rtm_autotune(h, 2, tiles=[35, 1], zchunks=[0, 0])  # collective, state restored
    P.rtm_step(h, 3)
    P.rtm_read_fields(h, u, up)
    np.savez(out_dir / f"rank{rank}.npz", u=u, up=up, z0=z0, nzl=nzl,
             enqueue_ms=P.rtm_last_enqueue_ms(h))
    dist.barrier()                                       # nobody unmaps a live neighbour
    P.rtm_destroy(h)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
