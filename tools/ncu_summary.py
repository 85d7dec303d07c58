"""Summarise ncu reports (one kernel each) into a text table for profiles/:
python tools/ncu_summary.py LABEL=report.ncu-rep ... > profiles/<name>.txt"""
import csv, io, subprocess, sys

METRICS = [
    ("time", "gpu__time_duration.sum"),
    ("dram read", "dram__bytes_read.sum"),
    ("dram write", "dram__bytes_write.sum"),
    ("dram % peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 hit %", "lts__t_sector_hit_rate.pct"),
    ("L1 hit %", "l1tex__t_sector_hit_rate.pct"),
    ("SM busy %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("FMA pipe %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("XU pipe %", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("LSU pipe %", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("ALU pipe %", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("issue active %", "sm__issue_active.avg.pct_of_peak_sustained_active"),
    ("warps active/SM", "sm__warps_active.avg.per_cycle_active"),
    ("registers", "launch__registers_per_thread"),
    ("block", "launch__block_size"),
    ("grid", "launch__grid_size"),
]

for arg in sys.argv[1:]:
    label, path = arg.rsplit("=", 1)
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    print(f"== {label}: {v[h.index('Kernel Name')]}")
    for name, key in METRICS:
        if key in h:
            i = h.index(key)
            print(f"  {name:16s} {v[i]:>14s} {u[i]}")
    print()
