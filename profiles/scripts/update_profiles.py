"""Copies one profiling pass (profiles/scripts/prof.sh TAG, results in
gpurun_out/) into the tracked profiles/ directory:

  profiles/r2_launches_TAG.txt   launch list of one bench step (ncu gpu__time_duration)
  profiles/r2_ncu_TAG.txt        --set full summary of the captured launches
  profiles/dram_traffic.json     DRAM bytes per launch per kernel class (one full render), stamped
  profiles/kernel_efficiency.json  issue/occupancy figures bench.py quotes, stamped
  profiles/bench_r2_TAG.json     the bench line of the same build

    python profiles/scripts/update_profiles.py TAG
"""
import csv
import io
import json
import os
import subprocess
import sys
from contextlib import redirect_stdout

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
import summarize  # noqa: E402

tag = sys.argv[1]
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def cap(fn, arg):
    buf = io.StringIO()
    with redirect_stdout(buf):
        fn(arg)
    return buf.getvalue()


with open(os.path.join(P, f"r2_launches_{tag}.txt"), "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, one bench step "
            f"(profiles/scripts/prof.sh {tag})\n")
    f.write(cap(summarize.launches, os.path.join(G, f"launches_{tag}.csv")))
rep = os.path.join(G, f"prof_{tag}.ncu-rep")
with open(os.path.join(P, f"r2_ncu_{tag}.txt"), "w") as f:
    f.write(f"# ncu --set full --clock-control none, mid-render launches of the bench workload "
            f"(profiles/scripts/prof.sh {tag})\n")
    f.write(cap(summarize.rep, rep))
tr = json.loads(cap(summarize.traffic, os.path.join(G, f"traffic_{tag}.csv")))
tr["_source"] = (f"profiles/scripts/prof.sh {tag}: ncu dram__bytes_read.sum + dram__bytes_write.sum over every "
                 f"launch of one 1920x1080x128 bench render, averaged per kernel class")
with open(os.path.join(P, "dram_traffic.json"), "w") as f:
    json.dump(tr, f, indent=1, sort_keys=True)
# issue figures per kernel class from the --set full capture (first launch of each)
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
SECS = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}
eff = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1].split("<")[0]
    cls = next((v for k, v in summarize.CLASSES.items() if name.startswith(k)), None)
    if not cls or cls in eff:
        continue

    def g(m):
        i = hdr.index(m)
        return float(r[i].replace(",", "")) * BYTES.get(units[i], SECS.get(units[i], 1.0))
    eff[cls] = {"issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "threads_per_warp_instruction": g("smsp__thread_inst_executed_per_inst_executed.ratio"),
                "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "registers": g("launch__registers_per_thread"),
                "dram_gbs": (g("dram__bytes_read.sum") + g("dram__bytes_write.sum")) /
                            g("gpu__time_duration.sum") / 1e9,
                "source": f"profiles/r2_ncu_{tag}.txt (ncu --set full, one launch)"}
with open(os.path.join(P, "kernel_efficiency.json"), "w") as f:
    json.dump(eff, f, indent=1, sort_keys=True)
try:
    line = open(os.path.join(G, f"bench_{tag}.json")).read().strip().splitlines()[-1]
    with open(os.path.join(P, f"bench_r2_{tag}.json"), "w") as f:
        f.write(line + "\n")
except (OSError, IndexError):
    pass
print("updated profiles/ from", tag)
