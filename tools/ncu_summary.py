#!/usr/bin/env python
"""Summarise an ncu --set full report (raw page) for one kernel: the numbers bench/DESIGN cite."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "dram__bytes_read.sum.per_second", "l1tex__t_bytes.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            key = h.split(".", 1)[1] if h.startswith(("TPC.", "SM_", "LTS.", "FBSP.")) and "TriageCompute" in h else h
            key = key.replace("TriageCompute.", "")
            if key in WANT or h == "Kernel Name":
                d[key] = (v, u)
        res.append(d)
    return res


if __name__ == "__main__":
    for d in summary(sys.argv[1]):
        for k in ["Kernel Name"] + WANT:
            if k in d:
                print(f"{k:80s} {d[k][0]} {d[k][1]}")
        print()
