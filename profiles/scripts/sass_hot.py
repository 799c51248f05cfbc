"""Instruction/stall breakdown of one kernel of an ncu report, in SASS order
(blocks of N instructions): python profiles/scripts/sass_hot.py REP KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
blk = int(sys.argv[3]) if len(sys.argv) > 3 else 16
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 5]
# the page lists every launch captured; keep the first listing
seen, first = set(), []
for r in data:
    if r[0] in seen:
        break
    seen.add(r[0])
    first.append(r)


def I(x):
    try:
        return int(x)
    except ValueError:
        return 0


iS = hdr.index("Warp Stall Sampling (All Samples)")
iI = hdr.index("Instructions Executed")
iT = hdr.index("Avg. Threads Executed")
iSrc = hdr.index("Source")
tot = sum(I(r[iS]) for r in first) or 1
toti = sum(I(r[iI]) for r in first) or 1
print(f"samples {tot}  warp-instructions {toti}  sass {len(first)}")
for b in range(0, len(first), blk):
    chunk = first[b:b + blk]
    s = sum(I(r[iS]) for r in chunk)
    i = sum(I(r[iI]) for r in chunk)
    if s > tot * 0.01 or i > toti * 0.01:
        thr = sum(I(r[iI]) * float(r[iT] or 0) for r in chunk) / max(1, i)
        print(f"{b:5d} stall {s / tot * 100:5.1f}%  inst {i / toti * 100:5.1f}%  thr {thr:4.1f}  "
              f"{chunk[0][iSrc].strip()[:44]:44s} .. {chunk[-1][iSrc].strip()[:36]}")
