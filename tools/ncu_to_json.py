"""Write the profiles/ncu_full_<workload>_<round>_<tile>.json summary the bench's roofline.traffic
reads, from an .ncu-rep of one k_stream launch (tools/ncu_summary.py metrics)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import summary  # noqa: E402


def num(s):
    v, unit = s.split()[0], (s.split()[1] if len(s.split()) > 1 else "")
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1, "us": 1e-3, "ns": 1e-6}
    return float(v) * scale.get(unit, 1)


def main(rep, workload, tile, rnd, out_dir="profiles"):
    d = summary(rep)[0]
    rd, wr = num(d["dram__bytes_read.sum"]), num(d["dram__bytes_write.sum"])
    res = {"workload": workload, "tile": tile, "report": f"{Path(rep).name} (launch 0)",
           "kernel": d["kernel"], "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd,
           "dram_write_bytes": wr, "duration_ms": num(d["gpu__time_duration.sum"]), "detail": d}
    p = Path(out_dir) / f"ncu_full_{workload}_{rnd}_{tile}.json"
    p.write_text(json.dumps(res, indent=1) + "\n")
    print(p, res["dram_bytes_per_launch"], res["duration_ms"])


if __name__ == "__main__":
    main(*sys.argv[1:])
