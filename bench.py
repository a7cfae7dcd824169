#!/usr/bin/env python
"""Benchmark of the RTM 3D-model time step (arxiv 1310.8232) on B200 — driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: NCCL z-slabs)

One bench "step" = one pass of the whole hot path over the config's
synthetic input: a1 C(p) from the velocity, u = u_prev = 0, the config's time steps of the
31-point star + leapfrog with fused source injection (a2, a3), halo exchange for N > 1
(a5, a6), and the readback of u^N (a7).  ``value`` = grid points x time steps / second
(Gpoints/s) with the velocity already resident in HBM; ``e2e`` = the same through the
public host-buffer API (pinned H2D of v, D2H of u^N inside the timed region).
Default workload: config 4 (1024^3, 100 time steps; strong scaling across N).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

BYTES_PER_POINT = 16  # compulsory fp32 traffic per point update: read u, u_prev, C; write u_next
# two-step passes (k_tb2s): read u^n, u^{n-1}, C; write u^{n+1}, u^{n+2}
# = 20 B per two point updates
BYTES_PER_POINT_TB2 = 10
METRIC = "stencil Gpoints/s and achieved HBM GB/s (% of ~8 TB/s) at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--tile", type=int, default=-1,
                    help="kernel variant; -1 = choose with rtm_autotune (untimed, before warm-up)")
    ap.add_argument("--tune-ni", type=int, default=12,
                    help="autotune iterations per candidate (raised automatically on small grids)")
    ap.add_argument("--tune-refine", type=int, default=6,
                    help="re-time the N fastest tuner candidates in 3 interleaved rounds of >= 100 ms "
                         "windows and keep the lowest mean (power-cap drift, DESIGN.md §7); <= 1: off")
    ap.add_argument("--lattice", type=int, default=0,
                    help="P > 1: autotune over the stream tiles x the paper's P-parts z-chunk "
                         "lattice (PAPER.md:296-301); 0: automatic z-chunk per tile")
    ap.add_argument("--zchunk", type=int, default=0)
    ap.add_argument("--nsteps", type=int, default=0, help="override the config's time steps")
    ap.add_argument("--shots", type=int, default=1,
                    help="batched independent shots on the config's velocity model (f3)")
    ap.add_argument("--halo", type=int, default=0, choices=[0, 2, 3],
                    help="N > 1 halo exchange: 0 NCCL send/recv (default), 2 fused push over "
                         "CUDA-IPC peer stores + flag protocol (SURVEY §8(f) f1), 3 copy-engine "
                         "pull from CUDA-IPC mappings + flag protocol (SURVEY §8(e))")
    ap.add_argument("--pdl", type=int, default=-1, choices=[-1, 0, 1],
                    help="programmatic dependent launch of consecutive steps (-1: library default)")
    ap.add_argument("--peer", action="store_true",
                    help="N > 1 test mode: peer contexts (CUDA IPC, no NCCL) over a gloo group; "
                         "ranks may share a GPU (then host-ordered) - exercises the N > 1 bench "
                         "path on one GPU, not a scaling measurement")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-verify", action="store_true",
                    help="N > 1: skip the untimed slab-by-slab bitwise check against a "
                         "single-GPU context on rank 0")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ncu", action="store_true", help="short run for ncu captures (no extras)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(cfg_name, tile_name):
    """dram read+write bytes per launch of the dominant kernel from the committed ncu
    --set full summary (profiles/ncu_full_<workload>_<round>.json) for this workload and
    kernel variant, if one exists."""
    for p in sorted((ROOT / "profiles").glob("ncu_full_*.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
            if (d.get("workload") == cfg_name and d.get("tile") == tile_name
                    and d.get("dram_bytes_per_launch")):
                return float(d["dram_bytes_per_launch"]), p.name
        except Exception:
            continue
    return None, None


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------ reference arm
def bench_config(cfg, world, shots, halo, nsteps, peer=False):
    """The `config` object of the JSON line — identical in both arms (workload only; the
    kernel variant the autotuner picks is reported outside it)."""
    nzl = cfg.nz // world if world > 1 else cfg.nz
    wl = f"C{cfg.k}" if shots == 1 else f"C{cfg.k}x{shots}shots"
    return {"workload": wl, "grid": [cfg.nx, cfg.ny, cfg.nz], "time_steps": nsteps,
            "sources": len(cfg.sources_xyz), "shots": shots,
            "parallelism": f"z-slab x{world}",
            "halo": ({0: "NCCL send/recv", 2: "fused IPC push + flags",
                      3: "IPC copy-engine pull"}.get(halo or (3 if peer else 0))) if world > 1 else None,
            "l2": "inputs larger than L2 (3 fields > 126 MB)"
            if cfg.nx * cfg.ny * nzl * shots * 4 > 126e6 else "L2-resident (no flush)"}


def oracle_sample(cfg, v_full, planes_per_mib):
    """The bounded CPU sample of the workload both CPU legs time: the first planes of the
    velocity model (about planes_per_mib planes of 1024x1024, at least 10)."""
    planes = max(10, min(cfg.nz, int(planes_per_mib * (1024 * 1024) / (cfg.nx * cfg.ny))))
    return np.ascontiguousarray(v_full[:planes]), planes


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on a bounded sample of the workload.
    Timed like cpu_baseline: the oracle's own steady_clock around its step loop (allocation,
    C(p) set-up and copies excluded), on the same sample (first 64 z-planes of the config)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    import rtm_inputs as ri
    cfg = ri.make_config(args.config, G=args.gpus if args.config == 5 else 1)
    nsteps_cfg = args.nsteps or cfg.steps
    v_full = cfg.velocity()
    v, planes = oracle_sample(cfg, v_full, 64)
    nsteps = 8  # time steps per bench step (~1 s of host work per bench step at C4)
    srcs = [(x, y, z, w[:nsteps]) for (x, y, z, w) in cfg.sources(v_full) if z < planes]
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))

    def one():
        oracle.run(v, cfg.dx, cfg.dt, ri.COEFFS_F32, nsteps, sources=srcs, nthreads=cores)
        return oracle.last_loop_seconds()

    for _ in range(args.warmup):
        one()
    ts = [one() for _ in range(args.steps)]
    pts = v.size * nsteps
    val = pts * len(ts) / sum(ts) / 1e9
    sample = (f"first {planes} z-planes of C{cfg.k} ({cfg.nx}x{cfg.ny}x{planes}), "
              f"{nsteps} time steps per bench step, step loop only")
    model, sockets = host_cpu()
    line = {"impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": "Gpoints/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * sum(ts) / len(ts), 3), "higher_is_better": True,
            "scaling": "strong" if args.config in (1, 2, 3, 4) else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded, rtm_inputs)",
            "config": bench_config(cfg, args.gpus, 1, args.halo, nsteps_cfg),
            "cpu_baseline": {"value": round(val, 4), "unit": "Gpoints/s", "cores": cores,
                             "kind": "oracle", "sample": sample,
                             "cpu_model": model, "sockets": sockets},
            "e2e": {"value": round(val, 4), "unit": "Gpoints/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def host_cpu():
    """(model name, sockets) of the host from /proc/cpuinfo (state the CPU)."""
    model, sockets = None, set()
    try:
        for line in open("/proc/cpuinfo"):
            k, _, val = line.partition(":")
            k = k.strip()
            if k == "model name" and model is None:
                model = val.strip()
            elif k == "physical id":
                sockets.add(val.strip())
    except OSError:
        pass
    return model, (len(sockets) or None)


def cpu_baseline(cfg, v_full):
    """Oracle timed on the host cores on a bounded sample (~12 s) of the workload: the same
    sample and the same clock (the oracle's step loop) as the --impl reference arm."""
    import oracle
    import rtm_inputs as ri
    cores = len(os.sched_getaffinity(0))
    v, planes = oracle_sample(cfg, v_full, 64)
    oracle.run(v, cfg.dx, cfg.dt, ri.COEFFS_F32, 2, nthreads=cores)
    per_step = max(oracle.last_loop_seconds() / 2, 1e-3)
    n = int(max(1, min(200, 12.0 / per_step)))
    oracle.run(v, cfg.dx, cfg.dt, ri.COEFFS_F32, n, nthreads=cores)
    dt = oracle.last_loop_seconds()
    val = v.size * n / dt / 1e9
    model, sockets = host_cpu()
    return {"value": round(val, 4), "unit": "Gpoints/s", "cores": cores, "kind": "oracle",
            "cpu_model": model, "sockets": sockets,
            "sample": f"first {planes} z-planes of C{cfg.k} ({cfg.nx}x{cfg.ny}x{planes}), "
                      f"{n} time steps, step loop only, {dt:.1f} s"}


# ------------------------------------------------------------------------------ b200 arm
def field_sums(t, planes_per_chunk=64):
    """Two 64-bit sums of the fp32 bit patterns of a (nz, ny, nx) field: plain and
    position-weighted (weight = flat index mod 1021 + 1), so equal sums mean equal bits up to a
    collision, and a shifted or transposed plane changes the weighted sum.  Chunked over planes
    to bound the int64 temporaries."""
    import torch
    s1 = s2 = 0
    plane = t.shape[-1] * t.shape[-2]
    for z in range(0, t.shape[0], planes_per_chunk):
        b = t[z:z + planes_per_chunk].reshape(-1).view(torch.int32).to(torch.int64)
        w = torch.arange(z * plane, z * plane + b.numel(), device=t.device, dtype=torch.int64) % 1021 + 1
        s1 += int(b.sum().item())
        s2 += int((b * w).sum().item())
        del b, w
    return s1, s2


def refine_selection(P, h, nI, cands, zcs, times, top, rounds=3, window_ms=100.0):
    """Second tuner pass over the `top` fastest (tile, z-chunk) candidates of the selection
    phase: `rounds` interleaved rounds of 3 nI steps each (one rtm_autotune call whose candidate
    list repeats the finalists), keeping the lowest MEAN time.  A single nI-step window per
    candidate ranks variants 1-2 % apart by the clock they happened to get: under the board's
    power cap the SM clock drifts during the tuner, so the candidates timed later run slower,
    and short windows favour variants that only win at full clock.  Each
    refinement window runs max(3 nI, ~window_ms) steps.  Times are max over ranks (library), so every rank picks the same."""
    zcs = list(zcs) if zcs is not None else [0] * len(cands)
    order = sorted((t, k) for k, t in enumerate(times) if np.isfinite(t))
    fin = []
    for _, k in order:
        if (cands[k], zcs[k]) not in fin:
            fin.append((cands[k], zcs[k]))
        if len(fin) == top:
            break
    if len(fin) < 2:
        return {"finalists": len(fin), "selected": P.rtm_tile_name(fin[0][0]) if fin else None,
                "zchunk": fin[0][1] if fin else None}
    t2 = [t for _ in range(rounds) for t, _ in fin]
    z2 = [z for _ in range(rounds) for _, z in fin]
    # windows of >= ~100 ms (the bench step is sustained load; C3's 29-step selection windows
    # are 10 ms), at least 3 nI steps
    nI2 = int(min(20000, max(3 * nI, np.ceil(window_ms / (order[0][0] / nI)))))
    _, tt = P.rtm_autotune(h, nI2, tiles=t2, zchunks=z2)
    mean = [float(np.mean(tt[j::len(fin)])) for j in range(len(fin))]
    best = int(np.argmin(mean))
    P.rtm_set_tile(h, fin[best][0])
    P.rtm_set_zchunk(h, fin[best][1])
    return {"finalists": len(fin), "rounds": rounds, "nI": nI2,
            "mean_ms_per_step": {f"{P.rtm_tile_name(t)}/z{z}": round(m / nI2, 5)
                                 for (t, z), m in zip(fin, mean)},
            "selected": P.rtm_tile_name(fin[best][0]), "zchunk": fin[best][1]}


def verify_slabs(args, P, ri, cfg, v_full, nsteps, d_out, z0, nzl, rank, world, dev, tdist, barrier):
    """Slab-by-slab bitwise check of the distributed result (u^N of the last bench step, in
    d_out) against a single-GPU context of the whole grid run by rank 0 with the same velocity,
    sources and time steps.  Returns the record rank 0 adds to the JSON line (None elsewhere)."""
    import torch
    mine = (z0, nzl) + field_sums(d_out[0])
    got = [None] * world
    tdist.all_gather_object(got, mine)
    if rank != 0:
        barrier()
        return None
    t0 = time.perf_counter()
    h1 = P.rtm_create(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, ri.COEFFS_F32)
    try:
        P.rtm_set_velocity(h1, np.ascontiguousarray(v_full))
        for (x, y, z, w) in cfg.sources(v_full):
            P.rtm_inject_source(h1, x, y, z, w[:nsteps] if len(w) > nsteps else w)
        P.rtm_step(h1, nsteps)
        full = torch.empty((cfg.nz, cfg.ny, cfg.nx), dtype=torch.float32, device=dev)
        P.rtm_read_field_device(h1, full.data_ptr())
        torch.cuda.synchronize(dev)
        bad = []
        for r, (zr, nr, s1, s2) in enumerate(got):
            if field_sums(full[zr:zr + nr]) != (s1, s2):
                bad.append(r)
        finite = bool(torch.isfinite(full).all().item())
        del full
    finally:
        P.rtm_destroy(h1)
    barrier()
    return {"reference": "single-GPU context of the whole grid on rank 0 (rtm_create, same "
                         "velocity, sources and time steps, default variant)",
            "time_steps": nsteps, "slabs": world, "bitwise": not bad and finite,
            "mismatched_ranks": bad, "method": "per-slab sums of the fp32 bit patterns "
            "(plain and position-weighted)", "seconds": round(time.perf_counter() - t0, 2)}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as tdist

    import paper_1310_8232_b200 as P
    import rtm_inputs as ri

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    ndev = torch.cuda.device_count()
    shared = args.peer and ndev < world  # test mode: several ranks per GPU
    devi = local % ndev if args.peer else local
    torch.cuda.set_device(devi)
    dev = torch.device("cuda", devi)
    if world > 1:
        if args.peer:
            tdist.init_process_group("gloo")
        else:
            tdist.init_process_group("nccl", device_id=dev)

    cfg = ri.make_config(args.config, G=world if args.config == 5 else 1)
    nsteps = args.nsteps or cfg.steps
    v_full = cfg.velocity()
    if world > 1 and args.peer:
        from paper_1310_8232_b200 import dist as pdist
        z0, nzl = P.rtm_slab_range(cfg.nz, world, rank)
        h = pdist.create_peer(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, ri.COEFFS_F32, rank, world,
                              devi, halo_mode=args.halo or 3, host_ordered=shared)
    elif world > 1:
        z0, nzl = P.rtm_slab_range(cfg.nz, world, rank)
        uid = [P.rtm_get_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(uid, src=0)
        h = P.rtm_create_dist(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, ri.COEFFS_F32, rank, world,
                              uid[0], local)
        if args.halo:
            P.rtm_set_option(h, P.RTM_OPT_HALO_MODE, args.halo)  # collective
    elif args.shots > 1:
        z0, nzl = 0, cfg.nz
        h = P.rtm_create_batch(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, ri.COEFFS_F32, args.shots)
    else:
        z0, nzl = 0, cfg.nz
        h = P.rtm_create(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, ri.COEFFS_F32)
    if args.pdl != -1:
        P.rtm_set_option(h, P.RTM_OPT_PDL, args.pdl)
    if args.tile != -1:
        P.rtm_set_tile(h, args.tile)
    if args.zchunk:
        P.rtm_set_zchunk(h, args.zchunk)
    shots = max(1, args.shots) if world == 1 else 1
    for k in range(shots):  # shot k: the config's sources moved along x (a shot line)
        for (x, y, z, w) in cfg.sources(v_full):
            xs = x if shots == 1 else (x + (k - shots // 2) * max(1, cfg.nx // (2 * shots))) % cfg.nx
            P.rtm_inject_source_shot(h, k, xs, y, z, w[:nsteps] if len(w) > nsteps else w)
    stream = torch.cuda.Stream(device=dev)  # a real stream (the legacy default stream 0 cannot be adopted)
    P.rtm_set_stream(h, stream.cuda_stream)
    v_local = np.ascontiguousarray(v_full[z0:z0 + nzl])
    d_v = torch.from_numpy(v_local).to(dev)
    d_out = torch.empty((shots,) + tuple(d_v.shape), dtype=torch.float32, device=dev)
    pts_local = cfg.nx * cfg.ny * nzl * shots
    pts_global = cfg.nx * cfg.ny * cfg.nz * shots
    tune = None
    if args.tile == -1 and not args.ncu:
        # the paper's two-phase blocksize selection, GPU analogue: every
        # stream-kernel variant timed on this grid (max over ranks = MWMB), winner verified
        P.rtm_set_velocity_device(h, d_v.data_ptr())
        # two-step passes need a single-slab single-shot context and the resident kernel a
        # single slab; elsewhere they would run their paired k_stream variant.  The multi-step
        # variants ("ms*") are left out (measured slower on C1-C5); the two-row
        # variants ("s2r*", fewer instructions per point) stay in: on a power-capped box the
        # lower-instruction variants can win (the tuner measures on the box it runs on)
        kinds = ("stream", "s2r") + (("resident",) if world == 1 else ()) + \
            (("tb2",) if world == 1 and args.shots == 1 else ())
        cands = [t for t in range(P.rtm_num_tiles()) if (P.rtm_tile_name(t) or "").startswith(kinds)]
        zcs = None
        if args.lattice > 1:  # the paper's nC = |tiles| x |b_z| candidates (selection phase)
            lat = P.rtm_blocksize_lattice(nzl, args.lattice)
            cands, zcs = [t for t in cands for _ in lat], [z for _ in cands for z in lat]
        # nI scaled so every candidate's timed window is ~>= 30 ms on small grids (8 steps of C2
        # are 0.4 ms: too short to rank variants 1-2 % apart); C3-C5 keep --tune-ni
        nI = int(min(400, max(args.tune_ni, 4e9 // pts_local)))
        res, times = P.rtm_autotune(h, nI, tiles=cands, zchunks=zcs)
        tune = {"selected": P.rtm_tile_name(res["best_tile"]), "candidates": len(cands),
                "nI": nI, "min_time_ms": round(res["min_time_ms"], 4),
                "zchunk": res.get("best_zchunk"), "lattice_P": args.lattice or None,
                "actual_time_ms": round(res["actual_time_ms"], 4),
                "quality_pct": round(res["quality_pct"], 2)}
        if args.tune_refine > 1:
            tune["refine"] = refine_selection(P, h, nI, cands, zcs, times, args.tune_refine)
            tune["selected"] = tune["refine"]["selected"]
            tune["zchunk"] = tune["refine"]["zchunk"]

    def barrier():
        if world > 1:
            if args.peer:
                torch.cuda.synchronize(dev)
                tdist.barrier()
            else:
                tdist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    def kernel_step():
        P.rtm_set_velocity_device(h, d_v.data_ptr())     # a1 from HBM-resident v
        P.rtm_reset(h)                                    # u = u_prev = 0
        P.rtm_step(h, nsteps)                             # a2..a6
        P.rtm_read_field_device(h, d_out.data_ptr())      # a7 (device-resident result)

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if args.peer else dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    w0 = torch.cuda.Event(enable_timing=True)
    w1 = torch.cuda.Event(enable_timing=True)
    for k in range(args.warmup):
        if k == args.warmup - 1:
            w0.record(stream)
        kernel_step()
    w1.record(stream)
    barrier()
    # Single-slab single-step runs are profiled live: CUDA events around every direct launch
    # and around every 16-launch graph replay (back-to-back launches on the device, so the
    # average is per launch including any inter-launch gap).  Where profiling would disable
    # graph replay (two-step passes, slab steps) and launches are short, the roofline comes
    # from a second, profiled pass instead, so `value` is not distorted.
    est_launch_ms = w0.elapsed_time(w1) / max(nsteps, 1) if args.warmup else 1.0
    tname0 = P.rtm_tile_name(P.rtm_get_tile(h))
    live = est_launch_ms >= 0.1 or (world == 1 and not tname0.startswith("tb2"))
    roof_src = ("live: CUDA events on the launching stream around every stencil launch / graph "
                "replay in the timed region" if live else
                "separate profiled pass of the same K steps (launches < 0.1 ms; graphs off)")
    launches0 = P.rtm_launch_count(h)
    P.rtm_set_profiling(h, 1 if live else 0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    with clocks:
        barrier()
        torch.cuda.nvtx.range_push("bench_timed")  # ncu --nvtx --nvtx-include bench_timed/
        e0.record(stream)
        for _ in range(args.steps):
            kernel_step()
        e1.record(stream)
        torch.cuda.nvtx.range_pop()
        barrier()
    ms = e0.elapsed_time(e1)
    gpu_launches = P.rtm_launch_count(h) - launches0 + args.steps  # + 1 a1 kernel per step
    if not live:
        P.rtm_set_profiling(h, 1)
        for _ in range(args.steps):
            kernel_step()
        barrier()
    kl, kms = P.rtm_kernel_stats(h)
    P.rtm_set_profiling(h, 0)
    ms_max = max_over_ranks(ms)
    value = pts_global * nsteps * args.steps / (ms_max / 1e3) / 1e9

    # roofline of the dominant kernel (the stencil): algorithmic 16 B/pt over its own
    # launch durations measured with CUDA events on the launching stream
    peak, peak_src = measured_peak()
    # batched shots share C: 12 B/pt for u, u_prev, u_next + 4 B/pt of C per shot batch
    bytes_per_pt = BYTES_PER_POINT if shots == 1 else 12.0 + 4.0 / shots
    tile_name = P.rtm_tile_name(P.rtm_get_tile(h))
    two_step = tile_name.startswith("tb2") and shots == 1 and world == 1 and nsteps >= 2
    if two_step:  # every launch is a two-step band pass (odd remainders: one k_stream step)
        bytes_per_pt = BYTES_PER_POINT_TB2
    alg_bytes = bytes_per_pt * pts_local * nsteps * args.steps
    achieved = alg_bytes / (kms / 1e3) / 1e9 if kms > 0 else None
    wl = f"C{cfg.k}" if shots == 1 else f"C{cfg.k}x{shots}shots"
    traffic, traffic_src = ncu_traffic(wl, tile_name)

    # checksum of the result vs a plain host recomputation is in tests/; here a sanity read
    finite = bool(torch.isfinite(d_out).all().item())

    # e2e through the public host-buffer API (pinned host memory): every bench step copies its
    # velocity model H2D and reads u^N back D2H inside the timed region.  The asynchronous calls
    # pipeline them across steps (step k+1's H2D and step k's D2H overlap the stencil steps on
    # a copy stream), as a user streaming velocity models through the library would.
    e2e = None
    if not args.no_e2e and not args.ncu:
        hv = torch.from_numpy(v_local).pin_memory()
        houts = [torch.empty(tuple(d_out.shape), dtype=torch.float32).pin_memory() for _ in range(2)]
        hv_np, hout_np = hv.numpy(), [t.numpy() for t in houts]

        def e2e_step(k):
            P.rtm_set_velocity_async(h, hv_np)            # H2D of the step's input
            P.rtm_reset(h)
            P.rtm_step_async(h, nsteps)
            P.rtm_read_field_async(h, hout_np[k % 2])     # D2H of the step's result

        e2e_step(0)
        P.rtm_sync(h)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for k in range(args.steps):
            e2e_step(k)
        P.rtm_sync(h)                                     # joins the copy stream, checks CFL
        f1.record(stream)
        barrier()
        ems = max_over_ranks(f0.elapsed_time(f1))
        e2e = {"value": round(pts_global * nsteps * args.steps / (ems / 1e3) / 1e9, 3),
               "unit": "Gpoints/s", "h2d_bytes_per_step": int(hv.numel() * 4),
               "d2h_bytes_per_step": int(houts[0].numel() * 4), "ms_per_step": round(ems / args.steps, 3),
               "pipelined": "rtm_set_velocity_async / rtm_step_async / rtm_read_field_async, rtm_sync"}
        # the synchronous host-buffer calls, one step at a time, for reference
        def sync_step():
            P.rtm_set_velocity(h, hv_np)
            P.rtm_reset(h)
            P.rtm_step(h, nsteps)
            P.rtm_read_field(h, hout_np[0])
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        g0.record(stream)
        sync_step()
        g1.record(stream)
        barrier()
        sms = max_over_ranks(g0.elapsed_time(g1))
        e2e["sync_value"] = round(pts_global * nsteps / (sms / 1e3) / 1e9, 3)
        # the result of the last pipelined step is the device result (recorded, never fatal)
        e2e["matches_device_result"] = bool(np.array_equal(hout_np[(args.steps - 1) % 2],
                                                           d_out.cpu().numpy()))

    # N > 1: the distributed result checked against ONE single-GPU context of the whole grid
    # (same inputs, same time steps) on rank 0 — bitwise, slab by slab (every slab
    # decomposition is bitwise equal to G = 1).  Untimed; makes every scaling line self-validating.
    slab_parity = None
    if world > 1 and not args.no_verify and not args.ncu:
        slab_parity = verify_slabs(args, P, ri, cfg, v_full, nsteps, d_out, z0, nzl, rank, world,
                                   dev, tdist, barrier)

    cpu = None
    if rank == 0 and not args.no_cpu and not args.ncu:
        cpu = cpu_baseline(cfg, v_full)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Gpoints/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
            "higher_is_better": True, "scaling": "strong" if cfg.k in (1, 2, 3, 4) else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, rtm_inputs)",
            "config": bench_config(cfg, world, shots, args.halo, nsteps, args.peer),
            "kernel_variant": tile_name,
            "hbm_effective_gbs": round(value * bytes_per_pt, 1),
            "hbm_frac_of_8tbs": round(value * bytes_per_pt / 8000.0, 4),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
                         "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4) if achieved else None,
                         "traffic": traffic, "peak_source": peak_src,
                         "kernel": ("k_tb2s" if two_step else "k_resident" if tile_name.startswith("resident") else
                                    "k_stream(multi-step)" if tile_name.startswith("ms") else
                                    "k_stream" if tile_name.startswith(("stream", "tb2")) else
                                    "k_tiled" if tile_name.startswith("tma") else "k_naive")
                                   + f"<{tile_name}>", "launches": kl,
                         "measured": roof_src,
                         "avg_launch_ms": round(kms / kl, 4) if kl else None,
                         "alg_bytes_per_pt": bytes_per_pt,
                         "alg_bytes_note": ("20 B per two point updates (read u^n, u^{n-1}, C; "
                                            "write u^{n+1}, u^{n+2}), per y-band launch"
                                            if two_step else "16 B per point update (read u, "
                                            "u_prev, C; write u_next)"),
                         "alg_bytes_per_launch": int(alg_bytes // max(kl, 1)),
                         "traffic_source": traffic_src},
            "e2e": e2e, "gpu_launches": gpu_launches, "clocks": clocks.summary(),
            "paper_context": {"note": "context only (other hardware, CPU, no GPU numbers in the paper)",
                              "source": "PAPER.md:559-560 Table ExecTime3, 200x200x800 x 448 it.",
                              "hardware": "2x Xeon E5410 quad-core 2.33 GHz (PAPER.md:478)",
                              "efficient_blocksize_1core_gpts": 0.0612,
                              "efficient_blocksize_8core_gpts": 0.235},
            "autotune": tune,
            "cpu_baseline": cpu, "finite": finite,
        }
        if slab_parity is not None:
            line["slab_parity"] = slab_parity
        if args.peer:
            line["test_mode"] = (f"peer contexts over gloo, {world} ranks on {min(ndev, world)} GPU(s)"
                                 + (", host-ordered: not a scaling measurement" if shared else ""))
        print(json.dumps(line), flush=True)
    if world > 1:
        barrier()  # no rank unmaps or frees buffers a neighbour still reads
    P.rtm_destroy(h)
    if world > 1:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
