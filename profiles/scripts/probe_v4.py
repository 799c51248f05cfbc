"""Probe variants x blocks/SM on the 1e7 x 10 table (insert-all, lookup-all, mix)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2305_07238_b200 import Context, MaterialCache  # noqa: E402

ctx = Context(0)
n = 1 << 26
nc, ne = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (10_000_000, 10)
t = MaterialCache(nc, ne, ctx)
for v in (0, 4):
    for bps in (2, 4, 8):
        t.clear()
        out = []
        for ph in (0, 1, 2):
            if ph == 2:
                t.clear()
                t.probe_bench(n // 2, 7, 0 + 16 * v + 256 * bps, 1)  # half full
            ms, by = t.probe_bench(n, 7, ph + 16 * v + 256 * bps, 1)
            out.append(f"{['ins', 'look', 'mix'][ph]} {n / ms / 1e6:5.1f} G/s {by / ms / 1e6:5.0f} GB/s")
        print(f"Nc={nc} Ne={ne} v{v} b{bps}: " + " | ".join(out), flush=True)
