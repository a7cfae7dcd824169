"""Energy per time step of kernel variants (NVML total-energy counter around a timed run):
on power-capped boxes (1 kW) a variant that draws less power keeps higher clocks.

    python tools/energy.py --config 4 --tiles 35,48 --ni 200 --repeat 2
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--tiles", default="35")
    ap.add_argument("--ni", type=int, default=200)
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args()
    import pynvml
    import torch
    import paper_1310_8232_b200 as P
    import rtm_inputs as ri
    pynvml.nvmlInit()
    nv = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    cfg = ri.make_config(a.config)
    v = cfg.velocity()
    h = P.rtm_create(cfg.nx, cfg.ny, cfg.nz, cfg.dx, cfg.dt, ri.COEFFS_F32)
    P.rtm_set_velocity(h, v)
    for s in cfg.sources(v):
        P.rtm_inject_source(h, *s)
    for _ in range(a.repeat):
        for t in [int(x) for x in a.tiles.split(",")]:
            P.rtm_set_tile(h, t)
            P.rtm_reset(h)
            P.rtm_step(h, 36)
            time.sleep(0.5)  # let the rails settle between variants
            e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(nv)  # mJ
            clk = []
            P.rtm_step(h, a.ni)
            ms = P.rtm_last_elapsed_ms(h)
            e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(nv)
            clk.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM))
            j = (e1 - e0) / 1e3
            print(json.dumps({"tile": P.rtm_tile_name(t), "ms_per_step": round(ms / a.ni, 4),
                              "joule_per_step": round(j / a.ni, 4), "avg_w": round(j / (ms / 1e3), 1),
                              "gpts": round(cfg.points * a.ni / ms / 1e6, 2),
                              "nj_per_point": round(j / (cfg.points * a.ni) * 1e9, 3),
                              "sm_mhz_end": clk[-1]}), flush=True)
    P.rtm_destroy(h)


if __name__ == "__main__":
    main()
