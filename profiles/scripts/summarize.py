"""Summaries of ncu captures for profiles/ (run here, on the CPU box):

    python profiles/scripts/summarize.py rep  gpurun_out/x.ncu-rep  > profiles/x.txt
    python profiles/scripts/summarize.py launches gpurun_out/launches.csv > profiles/y.txt
    python profiles/scripts/summarize.py traffic gpurun_out/traffic.csv > profiles/dram_traffic.json
"""
import collections
import csv
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(f"== {r[hdr.index('Kernel Name')].split('(')[0]}")
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"   {m:80s} {r[i]:>16s} {units[i]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'time_us':>12s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:70]:70s} {v[0]:8d} {v[1] / 1e3:12.1f} {v[1] / tot:7.3f}")


# kernel-name prefix -> the class name bench.py times it under
CLASSES = {"k_trace_closest": "trace_closest", "k_shadow": "trace_shadow", "k_shade": "shade",
           "k_primary": "primary", "k_probe_bench": "probe"}


def traffic(path):
    """dram read+write bytes per launch, averaged over every launch of each
    kernel class in the capture (one whole render), as JSON."""
    import json
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, vi, mi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"),
                      hdr.index("Metric Unit"))
    idi = hdr.index("ID")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        name = r[ki].split("(")[0].split("::")[-1].split("<")[0]
        cls = next((v for k, v in CLASSES.items() if name.startswith(k)), None)
        if cls:
            per[cls][r[idi]] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    out = {k: sum(v.values()) / len(v) for k, v in per.items()}
    out["_launches"] = {k: len(v) for k, v in per.items()}
    print(json.dumps(out, indent=1, sort_keys=True))


if __name__ == "__main__":
    {"rep": rep, "launches": launches, "traffic": traffic}[sys.argv[1]](sys.argv[2])
