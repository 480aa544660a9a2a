#!/usr/bin/env python
"""Summarise an `ncu --set full` report (.ncu-rep) of one scan_kernel launch
into the compact metric CSV kept under profiles/ (metric,unit,value): pipe
utilisation, issue activity, shared-memory wavefronts and conflicts, DRAM
traffic, registers, occupancy and the top warp-stall reasons.

    python scripts/ncu_summary.py gpurun_out/prof_x.ncu-rep > profiles/r1_ncu_x.csv
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma_type_fp16.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    w = csv.writer(sys.stdout)
    w.writerow(["metric", "unit", "value"])
    w.writerow(["Kernel Name", "", d.get("Kernel Name", ("", ""))[1]])
    for k in KEYS:
        if k in d:
            w.writerow([k, d[k][0], d[k][1]])
    stalls = [(h, d[h]) for h in hdr
              if h.startswith("smsp__average_warps_issue_stalled_")
              and h.endswith("_per_issue_active.ratio")]
    stalls.sort(key=lambda kv: -float(kv[1][1] or 0))
    for h, (u, v) in stalls[:8]:
        w.writerow([h, u, v])


if __name__ == "__main__":
    main(sys.argv[1])
