"""World-size-2 (and 3) CPU test of the N > 1 path's host logic over torch.distributed/gloo.

Each rank takes its slab from the library's own plan helpers (rtm_slab_range, rtm_halo_plan —
the same functions rtm_create_dist uses to place its NCCL send/recv buffers), keeps the sources
it owns, advances its slab with the oracle's explicit-z-halo step, and exchanges the 5-plane
halos with gloo isend/irecv at exactly the offsets the plan gives.  The gathered field must
equal the unsplit oracle bitwise (reading R14).  No GPU needed.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(buf, rank, world, offs, cnt):
    flat = torch.from_numpy(buf.reshape(-1))
    reqs = []
    if offs[0] >= 0:  # lower neighbour
        reqs.append(dist.isend(flat[offs[0]:offs[0] + cnt].clone(), rank - 1))
        reqs.append(dist.irecv(flat[offs[1]:offs[1] + cnt], rank - 1))
    if offs[2] >= 0:  # upper neighbour
        reqs.append(dist.isend(flat[offs[2]:offs[2] + cnt].clone(), rank + 1))
        reqs.append(dist.irecv(flat[offs[3]:offs[3] + cnt], rank + 1))
    for r in reqs:
        r.wait()


def _worker(rank, world, port, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1310_8232_b200 as P
        import rtm_inputs as ri
        cfg = ri.make_config(3, shape=(41, 18, 20), steps=steps)
        v = cfg.velocity()
        nz, ny, nx = v.shape
        u0, up0 = ri.random_fields(v.shape, seed=31)
        srcs = cfg.sources()
        z0, nzl = P.rtm_slab_range(nz, world, rank)
        offs, cnt = P.rtm_halo_plan(nx, ny, nzl, rank, world)
        # extra sources right on every slab boundary (owned by exactly one rank)
        for r in range(1, world):
            b, _ = P.rtm_slab_range(nz, world, r)
            srcs = srcs + [(3, 5, b, srcs[0][3]), (4, 6, b - 1, -srcs[0][3])]
        U = np.zeros((nzl + 10, ny, nx), np.float32)
        Pb = np.zeros_like(U)
        U[5:5 + nzl] = u0[z0:z0 + nzl]
        Pb[5:5 + nzl] = up0[z0:z0 + nzl]
        C = oracle.cfield_f32(np.ascontiguousarray(v[z0:z0 + nzl]), cfg.dx, cfg.dt)
        _exchange(U, rank, world, offs, cnt)
        _exchange(Pb, rank, world, offs, cnt)
        for n in range(steps):
            oracle.slab_step_f32(ri.COEFFS_F32, C, U, Pb, nthreads=1)
            for (x, y, z, w) in srcs:
                if z0 <= z < z0 + nzl and n < len(w):
                    Pb[z - z0 + 5, y, x] = np.float32(Pb[z - z0 + 5, y, x] + w[n])
            _exchange(Pb, rank, world, offs, cnt)
            U, Pb = Pb, U
        part = torch.from_numpy(np.ascontiguousarray(U[5:5 + nzl]))
        if rank == 0:  # slabs differ in size: point-to-point gather
            parts = [part] + [torch.empty((P.rtm_slab_range(nz, world, r)[1], ny, nx))
                              for r in range(1, world)]
            for r in range(1, world):
                dist.recv(parts[r], r)
            got = np.concatenate([p.numpy() for p in parts])
            ref = oracle.run(v, cfg.dx, cfg.dt, ri.COEFFS_F32, steps, u0=u0, up0=up0, sources=srcs)
            q.put(("ok", bool(np.array_equal(got, ref)), float(np.abs(got - ref).max())))
        else:
            dist.send(part, 0)
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e), 0.0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slabs_equal_unsplit_oracle(world):
    from conftest import build_library
    build_library()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 9, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    status, equal, err = q.get(timeout=10)
    assert status == "ok", equal
    assert equal, err


def _rec_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1310_8232_b200 import dist as pd
        rec = bytes([rank]) * 512  # stands in for rtm_ipc_export's 512-byte record
        lo, hi = pd.exchange_neighbour_records(rec, rank, world)
        q.put((rank, None if lo is None else lo[0], None if hi is None else hi[0],
               None if lo is None else len(lo)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ipc_record_exchange_gives_each_rank_its_neighbours(world):
    """The peer-context bootstrap (paper_1310_8232_b200.dist): every rank receives exactly the
    records of rank-1 and rank+1 (None at the ends), unmodified."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rec_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    got = sorted(q.get(timeout=10) for _ in range(world))
    for rank, lo, hi, n in got:
        assert lo == (rank - 1 if rank > 0 else None)
        assert hi == (rank + 1 if rank < world - 1 else None)
        assert n in (None, 512)
