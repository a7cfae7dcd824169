"""Cross-process halo data plane on one B200: 2 and 3
processes, each a peer context (rtm_create_peer: CUDA-IPC mappings of the neighbours' buffers
and flag words, no NCCL) on cuda:0, bootstrapped over a gloo group (paper_1310_8232_b200.dist).
Halo mode 2 (fused push: the stencil epilogue stores into the neighbour's IPC-mapped halo) and
mode 3 (copy-engine pull from the neighbour's IPC-mapped boundary planes).  The ranks share one
GPU, so they run host-ordered (RTM_OPT_HOST_ORDERED: every device-side flag wait is satisfied
before it is enqueued; waits across processes on one GPU are not allowed on this pool).  The
schedule crosses the collective restarts: reset, set_fields + set_step_count (resume), autotune.
The gathered field must equal the single-context run bitwise (R14) and the oracle within
tolerance."""
from __future__ import annotations

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle
import rtm_inputs as ri

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tests"))
import peer_worker as W  # noqa: E402


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from conftest import build_library
    build_library()
    import paper_1310_8232_b200 as P
    return P


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def reference(P):
    v, u0, up0, src = W.case()
    a, b, c = W.STEPS
    n = a + c + 3
    nz, ny, nx = W.SHAPE
    with P.Simulation(nx, ny, nz, 10.0, 1e-3, ri.COEFFS_F32) as sim:
        sim.set_velocity(v)
        for s in src:
            sim.inject_source(*s)
        sim.set_fields(u0, up0)
        sim.step(n)
        u, up = sim.read_fields()
    orc = oracle.run(v, 10.0, 1e-3, ri.COEFFS_F32, n, u0=u0, up0=up0, sources=src)
    return u, up, orc


@pytest.mark.parametrize("world,halo", [(2, 3), (3, 3), (2, 2), (3, 2)])
def test_peer_processes_on_one_gpu_bitwise_equal_single(P, reference, tmp_path, world, halo):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "tests" / "peer_worker.py"), str(tmp_path), str(halo)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=str(ROOT))
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-5000:])
    ref_u, ref_up, orc = reference
    u = np.empty_like(ref_u)
    up = np.empty_like(ref_up)
    covered = 0
    for k in range(world):
        d = np.load(tmp_path / f"rank{k}.npz")
        z0, nzl = int(d["z0"]), int(d["nzl"])
        assert (z0, nzl) == P.rtm_slab_range(W.SHAPE[0], world, k)
        u[z0:z0 + nzl] = d["u"]
        up[z0:z0 + nzl] = d["up"]
        covered += nzl
    assert covered == W.SHAPE[0]
    assert np.array_equal(u, ref_u) and np.array_equal(up, ref_up)
    m = float(np.abs(orc).max())
    assert float(np.abs(u.astype(np.float64) - orc).max()) <= 1e-4 * m


def test_bench_n2_path_with_peer_contexts_on_one_gpu():
    """The N > 1 bench path (torchrun, slab ranges, collective reset / autotune, max-over-ranks
    timing, e2e through the async host-buffer calls, one JSON line from rank 0) run as 2 ranks of
    peer contexts on one GPU (`--peer`, host-ordered): a functional check of the line, not a
    scaling number (the line says so in `test_mode`)."""
    import json
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "bench.py"), "--gpus", "2", "--peer", "--config", "1", "--steps", "2",
           "--warmup", "3", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-5000:])
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and "test_mode" in d and d["finite"] is True
    assert d["config"]["parallelism"] == "z-slab x2" and d["config"]["halo"] == "IPC copy-engine pull"
    assert d["e2e"]["value"] > 0 and d["e2e"]["matches_device_result"] is True
    # the untimed slab-by-slab check against one single-GPU context of the whole grid
    sp = d["slab_parity"]
    assert sp["bitwise"] is True and sp["slabs"] == 2 and sp["mismatched_ranks"] == []
