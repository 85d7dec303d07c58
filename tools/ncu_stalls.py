"""Warp-stall and pipe summary of an ncu report (one kernel): where the warps
wait (smsp__average_warps_issue_stalled_* per issued instruction), pipe
utilisations, L1TEX / texture / L2 throughput, and the per-opcode stall
samples of the SASS source page.

    python tools/ncu_stalls.py LABEL=report.ncu-rep ... > profiles/<name>.txt
"""
import collections
import csv
import io
import subprocess
import sys

PIPES = [
    ("FMA pipe %", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("XU pipe %", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("ALU pipe %", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("LSU pipe %", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("TEX pipe %", "sm__inst_executed_pipe_tex.avg.pct_of_peak_sustained_active"),
    ("issue active %", "sm__issue_active.avg.pct_of_peak_sustained_active"),
    ("L1TEX throughput %", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("L1 hit %", "l1tex__t_sector_hit_rate.pct"),
    ("L2 throughput %", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 hit %", "lts__t_sector_hit_rate.pct"),
    ("DRAM throughput %", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("dram read bytes", "dram__bytes_read.sum"),
    ("L1 global sectors", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
    ("L1 global requests", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"),
    ("tex sectors", "l1tex__t_sectors_pipe_tex_mem_texture.sum"),
    ("tex requests", "l1tex__t_requests_pipe_tex_mem_texture.sum"),
    ("L1 wavefronts (data)", "l1tex__data_pipe_lsu_wavefronts.sum"),
    ("tex wavefronts", "l1tex__data_pipe_tex_wavefronts.sum"),
    ("L1TEX lookups (tag) %", "l1tex__t_set_accesses.avg.pct_of_peak_sustained_active"),
    ("time", "gpu__time_duration.sum"),
    ("cycles active", "sm__cycles_active.avg"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def source(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[1], rows[2:]


for arg in sys.argv[1:]:
    label, path = arg.rsplit("=", 1)
    v, u = raw(path)
    print(f"== {label}: {v.get('Kernel Name', '?')}")
    for name, key in PIPES:
        if key in v:
            print(f"  {name:24s} {v[key]:>16s} {u.get(key, '')}")
    stalls = sorted(((k.split("stalled_")[1].replace("_per_issue_active.ratio", ""), float(v[k]))
                     for k in v if k.startswith("smsp__average_warps_issue_stalled_")
                     and k.endswith("_per_issue_active.ratio")), key=lambda x: -x[1])
    print("  warp stalls per issued instruction:")
    for k, x in stalls:
        if x >= 0.05:
            print(f"    {k:28s} {x:8.3f}")
    hdr, data = source(path)
    if "Source" in hdr:
        H = {h: i for i, h in enumerate(hdr)}
        agg = collections.defaultdict(collections.Counter)
        tot = 0
        for r in data:
            src = r[H["Source"]].strip()
            parts = src.split()
            if not parts:
                continue
            op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
            op = op.split(".")[0]
            n = int(r[H["Warp Stall Sampling (All Samples)"]] or 0)
            tot += n
            agg[op]["all"] += n
            for k in ("stall_math", "stall_long_sb", "stall_short_sb", "stall_mio", "stall_tex", "stall_lg",
                      "stall_wait", "stall_not_selected", "stall_selected", "stall_barrier", "stall_dispatch"):
                if k in H:
                    agg[op][k] += int(r[H[k]] or 0)
        print(f"  stall samples by opcode (total {tot}):")
        for op, c in sorted(agg.items(), key=lambda x: -x[1]["all"])[:10]:
            top = ", ".join(f"{k[6:]} {c[k]}" for k in sorted(c, key=lambda k: -c[k]) if k != "all" and c[k])[:150]
            print(f"    {op:10s} {c['all']:8d} ({100 * c['all'] / max(tot, 1):4.1f}%)  {top}")
    print()
