"""Tile-variant sweep on a config's real grid (the GPU analogue of the paper's blocksize
selection phase): every variant runs nI time steps from the config's
state, timed with CUDA events; prints ms/step, Gpt/s and effective GB/s per variant."""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--ni", type=int, default=20)
    ap.add_argument("--tiles", default="")
    ap.add_argument("--zchunk", default="0")
    ap.add_argument("--cache", default="", help="comma list of RTM_OPT_CACHE_MODE values (hex ok)")
    ap.add_argument("--repeat", type=int, default=1, help="interleaved repetitions (min is kept)")
    ap.add_argument("--shots", type=int, default=1)
    ap.add_argument("--shot-order", default="0", help="comma list of RTM_OPT_SHOT_ORDER values")
    ap.add_argument("--slabs", type=int, default=1, help="in-process z-slabs (all on visible GPUs round-robin)")
    ap.add_argument("--halo", type=int, default=0, help="RTM_OPT_HALO_MODE for --slabs > 1")
    ap.add_argument("--graphs", type=int, default=1, help="RTM_OPT_GRAPHS (CUDA-graph replays)")
    ap.add_argument("--share", type=int, default=0, help="RTM_OPT_SLAB_SHARE for --slabs > 1")
    ap.add_argument("--pdl", default="0", help="comma list of RTM_OPT_PDL values (interleaved)")
    ap.add_argument("--zdir", default="0", help="comma list of RTM_OPT_ZDIR values (interleaved)")
    ap.add_argument("--l2persist", default="", help="comma list of cudaLimitPersistingL2CacheSize "
                    "values in MB (interleaved; the L2 set-aside for evict_last / persisting lines)")
    args = ap.parse_args()
    import torch
    import paper_1310_8232_b200 as P
    import rtm_inputs as ri
    cfg = ri.make_config(args.config)
    v = cfg.velocity()
    if args.slabs > 1:
        ndev = torch.cuda.device_count()
        h = P.rtm_create_multi(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, ri.COEFFS_F32,
                               [k % ndev for k in range(args.slabs)])
        P.rtm_set_option(h, P.RTM_OPT_HALO_MODE, args.halo)
        P.rtm_set_option(h, P.RTM_OPT_SLAB_SHARE, args.share)
    elif args.shots > 1:
        h = P.rtm_create_batch(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, ri.COEFFS_F32, args.shots)
    else:
        h = P.rtm_create(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, ri.COEFFS_F32)
    P.rtm_set_option(h, P.RTM_OPT_GRAPHS, args.graphs)
    P.rtm_set_velocity(h, v)
    for s in cfg.sources(v):
        P.rtm_inject_source(h, *s)
    st = torch.cuda.Stream()
    if args.slabs == 1:
        P.rtm_set_stream(h, st.cuda_stream)
    tiles = [int(t) for t in args.tiles.split(",")] if args.tiles else list(range(P.rtm_num_tiles()))
    res = []
    for t in [t for _ in range(args.repeat) for t in tiles]:
        for zc, cm, so, pdl, zd, l2 in [(int(z), c, int(o), int(q), int(d), m)
                                        for z in args.zchunk.split(",")
                                        for c in ([int(x, 0) for x in args.cache.split(",")] if args.cache else [None])
                                        for o in args.shot_order.split(",") for q in args.pdl.split(",")
                                        for d in args.zdir.split(",")
                                        for m in ([int(x) for x in args.l2persist.split(",")] if args.l2persist else [None])]:
            if l2 is not None:
                from cuda.bindings import runtime as crt
                torch.cuda.synchronize()
                err, = crt.cudaDeviceSetLimit(crt.cudaLimit.cudaLimitPersistingL2CacheSize, l2 << 20)
                assert err == crt.cudaError_t.cudaSuccess, err
            P.rtm_set_option(h, P.RTM_OPT_SHOT_ORDER, so)
            P.rtm_set_option(h, P.RTM_OPT_PDL, pdl)
            P.rtm_set_option(h, P.RTM_OPT_ZDIR, zd)
            P.rtm_set_tile(h, t)
            P.rtm_set_zchunk(h, zc)
            if cm is not None:
                P.rtm_set_option(h, P.RTM_OPT_CACHE_MODE, cm)
            P.rtm_reset(h)
            P.rtm_step(h, 36)  # warm-up: tensor maps, graphs (built at the first 32-step run)
            if args.slabs == 1:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                P.rtm_step(h, args.ni)
                e1.record(st)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / args.ni
            else:  # the library's own CUDA-event time of the rtm_step call (all slabs joined)
                P.rtm_step(h, args.ni)
                ms = P.rtm_last_elapsed_ms(h) / args.ni
            gpts = cfg.points * args.shots / ms / 1e6
            r = {"tile": t, "name": P.rtm_tile_name(t), "zchunk": zc, "shot_order": so, "pdl": pdl,
                 "zdir": zd, "l2persist_mb": l2,
                 "slabs": args.slabs, "halo": args.halo, "graphs": args.graphs, "share": args.share,
                 "enqueue_ms_per_step": round(P.rtm_last_enqueue_ms(h) / args.ni, 4),
                 "cache": hex(P.rtm_get_option(h, P.RTM_OPT_CACHE_MODE)), "ms_per_step": round(ms, 4),
                 "gpts": round(gpts, 2), "eff_gbs": round(16 * gpts, 1)}
            res.append(r)
            print(json.dumps(r), flush=True)
    agg = {}
    for r in res:
        k = (r["tile"], r["zchunk"], r["cache"], r["shot_order"], r["pdl"], r["zdir"], r["l2persist_mb"])
        if k not in agg or r["ms_per_step"] < agg[k]["ms_per_step"]:
            agg[k] = r
    for r in sorted(agg.values(), key=lambda r: r["ms_per_step"]):
        print("MIN", json.dumps(r))
    best = min(res, key=lambda r: r["ms_per_step"])
    print("BEST", json.dumps(best))
    P.rtm_destroy(h)


if __name__ == "__main__":
    main()
