#!/usr/bin/env python
"""Summarise an `ncu --set full` capture of the Leja kernel into profiles/leja_traffic.json.

  python tools/ncu_traffic.py gpurun_out/leja_tb2_full.ncu-rep 16,16,14,10 4096 tb2 "capture description"
  python tools/ncu_traffic.py gpurun_out/vert3d.ncu-rep 10:13:16 512 vert3d "..."   # 3D K=3 call, n^3 points

per launch: dram read/write bytes (traffic), gpu time, the algorithmic bytes of that launch
(bench.leja_bytes_per_point x N) and their ratio (traffic well above 1 = wasted re-reads)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import leja_bytes_per_point, leja_bytes_per_point_vertical_tb2  # noqa: E402

MET = ("dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size,"
       "launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,"
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed")
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-3, "ms": 1.0, "ns": 1e-6, "msecond": 1.0,
         "usecond": 1e-3, "nsecond": 1e-6}


def main():
    rep, n, kind, desc = sys.argv[1], int(sys.argv[3]), sys.argv[4], sys.argv[5]
    # per launch: an iteration count, or (vert3d) the accumulators' iteration counts joined by ':'
    iters = [[int(y) for y in x.split(":")] for x in sys.argv[2].split(",")]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", MET],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, name):
        return float(r[col[name]].replace(",", "")) * SCALE.get(units[col[name]], 1.0)

    launches = []
    N = n ** 3 if kind == "vert3d" else n * n
    for r, mk in zip(data, iters):
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        m = mk if kind == "vert3d" else mk[0]
        alg = N * (leja_bytes_per_point_vertical_tb2(mk) if kind == "vert3d" else leja_bytes_per_point(m, kind == "tb2"))
        launches.append({"iters": m, "gpu_time_ms": val(r, "gpu__time_duration.sum"), "dram_read_bytes": rd,
                         "dram_write_bytes": wr, "traffic_bytes": rd + wr, "algorithmic_bytes": alg,
                         "traffic_over_algorithmic": (rd + wr) / alg})
    d0 = data[0]
    res = {"kernel": d0[col["Kernel Name"]], "capture": desc, "launches": launches,
           "traffic_bytes_per_launch": sum(x["traffic_bytes"] for x in launches) / len(launches),
           "algorithmic_bytes_per_launch": sum(x["algorithmic_bytes"] for x in launches) / len(launches),
           "registers_per_thread": val(d0, "launch__registers_per_thread"),
           "grid": val(d0, "launch__grid_size"),
           "dram_throughput_pct_of_peak_elapsed": val(d0, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
           "l2_throughput_pct": val(d0, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
           "warps_active_pct": val(d0, "sm__warps_active.avg.pct_of_peak_sustained_active")}
    res["traffic_over_algorithmic"] = res["traffic_bytes_per_launch"] / res["algorithmic_bytes_per_launch"]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
