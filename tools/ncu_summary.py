#!/usr/bin/env python
"""Compact summary of an `ncu --page raw --csv` export (one or more kernels):
duration, DRAM bytes and throughput, SM / L1 / L2 / fp64 / DMMA utilisation,
occupancy, top warp-stall reasons.  Usage: python tools/ncu_summary.py raw.csv"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe % (active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe cycles %"),
    ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "fp64 tensor (DMMA) %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    stall = [i for i, h in enumerate(hdr)
             if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        print(r[hdr.index("Kernel Name")][:110])
        for k, name in KEYS:
            if k in hdr and r[hdr.index(k)] not in ("", "n/a"):
                print(f"  {name:30s} {r[hdr.index(k)]} {units[hdr.index(k)]}")
        st = sorted(((float(r[i] or 0), hdr[i]) for i in stall), reverse=True)[:5]
        print("  top stalls (cycles per issued instruction): " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.2f}"
            for v, h in st))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
