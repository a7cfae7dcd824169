"""Summarise an ncu --set full report (raw page) into the metrics the roofline needs."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "sm__cycles_elapsed.avg.per_second", "dram__bytes.sum.per_second"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:80]}
        for k in KEYS:
            if k in hdr:
                d[k] = f"{vals[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(vals[i])
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        res.append(d)
    return res


def _num(v):
    return float(v.split()[0])


def _scale(v):
    num, unit = v.split()[0], (v.split()[1] if len(v.split()) > 1 else "")
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(num) * f


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--workload", default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--tile-name", default=None, help="variant name (rtm_tile_name) profiled")
    a = ap.parse_args()
    res = summary(a.rep)
    if a.workload:  # bench-consumable record for the dominant (first) kernel
        k = res[0]
        rd, wr = _scale(k["dram__bytes_read.sum"]), _scale(k["dram__bytes_write.sum"])
        res = {"workload": a.workload, "tile": a.tile_name, "report": a.rep.split("/")[-1],
               "kernel": k["kernel"],
               "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
               "duration_ms": _num(k["gpu__time_duration.sum"]), "detail": k}
    txt = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(txt + "\n")
    print(txt)
