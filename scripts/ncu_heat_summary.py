#!/usr/bin/env python
"""Summarise an `ncu --set full` capture of the bench's heat2d kernel into the JSON the bench
reads for roofline.traffic: DRAM read + write bytes per launch next to the algorithmic bytes."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct", "launch__shared_mem_per_block_static",
        "launch__occupancy_limit_shared_mem"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def main(rep, out, rows, cols, command):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows_ = list(csv.reader(io.StringIO(txt)))
    head, units, row = rows_[0], rows_[1], rows_[2]
    d = dict(zip(head, row))
    u = dict(zip(head, units))
    res = {k: {"value": d[k], "unit": u[k]} for k in KEYS if k in d}
    rd = float(d["dram__bytes_read.sum"]) * SCALE.get(u["dram__bytes_read.sum"], 1.0)
    wr = float(d["dram__bytes_write.sum"]) * SCALE.get(u["dram__bytes_write.sum"], 1.0)
    alg = 8 * rows * cols
    res.update({"traffic_bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": (rd + wr) / alg,
                "kernel": d.get("Kernel Name", ""), "command": command})
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
