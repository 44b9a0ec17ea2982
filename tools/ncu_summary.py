#!/usr/bin/env python
"""Summaries of ncu outputs for profiles/ (run here, on the files gpurun brought back).

    python tools/ncu_summary.py launches gpurun_out/r01b/launches.csv > profiles/x_launches.txt
    python tools/ncu_summary.py full gpurun_out/r01b/group_full.ncu-rep > profiles/x_ncu_group.txt
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
]


def short(name, w=70):
    name = name.split("(")[0]
    return name if len(name) <= w else name[-w:]


def launches(path):
    text = open(path).read()
    i = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[i:])))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + us)
    OURS = ("pp::", "ss_group", "reduce_count", "scan_swap", "tile_scan", "locate_kernel", "swap_kernel",
            "small_partition", "count_kernel", "qs_", "bps_", "stable_", "swap_ranges")
    ours = {k: v for k, v in agg.items() if k.startswith("void pp") or any(t in k for t in OURS)}
    tot = sum(t for _, t in ours.values()) or 1.0
    print(f"{'kernel':72s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share_of_pp':>11s}")
    for k, (c, t) in agg.items():
        share = f"{100 * t / tot:.1f}%" if k in ours else "-"
        tag = "" if k in ours else "torch: "
        print(f"{(tag + k)[:72]:72s} {c:8d} {t:10.1f} {t / c:9.2f} {share:>11s}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        print("Kernel Name:", vals[hdr.index("Kernel Name")])
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"{m}: {vals[i]} {units[i]}")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
