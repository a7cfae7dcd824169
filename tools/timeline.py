"""Device timeline of the slab step (nsys is not in this image): torch.profiler's CUPTI
activity trace records every kernel and copy the library issues, on every stream, with device
timestamps.  Runs G in-process z-slabs on one GPU (halo mode 0: boundary kernel -> copy-engine
exchange on the comm streams -> interior kernel; mode 3: the flag-ordered pull) and reports,
per step, how much of the halo-copy time overlaps the interior stencil kernels.

    python tools/timeline.py --config 3 --slabs 2 --halo 0 --steps 4 --out profiles/x.json
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--slabs", type=int, default=2)
    ap.add_argument("--halo", type=int, default=0)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--tile", type=int, default=35)
    ap.add_argument("--graphs", type=int, default=0)
    ap.add_argument("--out", default="")
    ap.add_argument("--trace", default="", help="also write the raw chrome trace here")
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_1310_8232_b200 as P
    import rtm_inputs as ri
    cfg = ri.make_config(a.config)
    v = cfg.velocity()
    if a.slabs > 1:
        h = P.rtm_create_multi(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, ri.COEFFS_F32, [0] * a.slabs)
        P.rtm_set_option(h, P.RTM_OPT_HALO_MODE, a.halo)
    else:
        h = P.rtm_create(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, ri.COEFFS_F32)
    P.rtm_set_option(h, P.RTM_OPT_GRAPHS, a.graphs)  # 0: one trace entry per direct launch
    P.rtm_set_tile(h, a.tile)
    P.rtm_set_velocity(h, v)
    for s in cfg.sources(v):
        P.rtm_inject_source(h, *s)
    P.rtm_step(h, 36)  # warm-up (tensor maps, graphs)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        P.rtm_step(h, a.steps)
        torch.cuda.synchronize()
    if a.trace:
        prof.export_chrome_trace(a.trace)
    ev = []
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        name = e.name
        kind = ("copy" if "emcpy" in name or "Memcpy" in name else
                "stencil" if "k_stream" in name or "k_tiled" in name or "k_naive" in name else
                "signal" if "k_signal" in name else "other")
        t0 = e.time_range.start
        ev.append({"name": name[:60], "kind": kind, "t0_us": t0, "t1_us": e.time_range.end,
                   "stream": getattr(e, "device_resource_id", None)})
    ev.sort(key=lambda x: x["t0_us"])
    if not ev:
        print("no device activity recorded")
        return 1
    base = ev[0]["t0_us"]
    for x in ev:
        x["t0_us"] -= base
        x["t1_us"] -= base
    stencils = [x for x in ev if x["kind"] == "stencil"]
    copies = [x for x in ev if x["kind"] == "copy"]
    # interior launches are the long stencil launches; boundary launches the short ones
    durs = sorted(x["t1_us"] - x["t0_us"] for x in stencils)
    cut = durs[len(durs) // 2] * 0.5 if durs else 0
    interior = [x for x in stencils if x["t1_us"] - x["t0_us"] > cut]

    def overlap(c):
        tot = 0.0
        for k in interior:
            lo, hi = max(c["t0_us"], k["t0_us"]), min(c["t1_us"], k["t1_us"])
            tot += max(0.0, hi - lo)
        return min(tot, c["t1_us"] - c["t0_us"])
    copy_t = sum(c["t1_us"] - c["t0_us"] for c in copies)
    ov = sum(overlap(c) for c in copies)
    span = ev[-1]["t1_us"]
    # consecutive stencil launches: device gap between the end of one and the start of the next
    gaps = [b["t0_us"] - a_["t1_us"] for a_, b in zip(stencils, stencils[1:])]
    kd = [x["t1_us"] - x["t0_us"] for x in stencils]
    res = {"config": f"C{cfg.k}", "grid": [cfg.nx, cfg.ny, cfg.nz], "slabs": a.slabs, "halo": a.halo,
           "tile": P.rtm_tile_name(a.tile), "steps": a.steps, "span_us": round(span, 1),
           "us_per_step": round(span / a.steps, 1), "stencil_launches": len(stencils),
           "interior_launches": len(interior), "copies": len(copies),
           "copy_us_total": round(copy_t, 1), "copy_us_overlapped_by_interior": round(ov, 1),
           "overlap_frac": round(ov / copy_t, 3) if copy_t else None,
           "stencil_us_mean": round(sum(kd) / len(kd), 2) if kd else None,
           "gap_us_mean": round(sum(gaps) / len(gaps), 2) if gaps else None,
           "gap_us_max": round(max(gaps), 2) if gaps else None,
           "source": "torch.profiler (CUPTI activity records: device timestamps)",
           "events": [{k: (round(v, 2) if isinstance(v, float) else v) for k, v in x.items()}
                      for x in ev[:400]]}
    print(json.dumps({k: v for k, v in res.items() if k != "events"}))
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))
    P.rtm_destroy(h)
    return 0


if __name__ == "__main__":
    sys.exit(main())
