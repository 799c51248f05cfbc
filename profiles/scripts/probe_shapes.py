"""Probe throughput vs table shape: is the probe bound by the DRAM blocks an
80-byte cell straddles? Same descriptor stream, tables with 64-byte-aligned
cells (Ne = 8) vs 80-byte cells (Ne = 10), at equal total memory."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2305_07238_b200 import Context, MaterialCache  # noqa: E402

ctx = Context(0)
n = 1 << 26
for nc, ne in ((10_000_000, 10), (12_500_000, 8), (10_000_000, 8), (20_000_000, 4), (40_000_000, 2)):
    t = MaterialCache(nc, ne, ctx)
    for v in (0, 3):
        t.clear()
        ms_i, b_i = t.probe_bench(n, 7, 0 + 16 * v + 256 * 2, 1)
        ms_l, b_l = t.probe_bench(n, 7, 1 + 16 * v + 256 * 2, 1)
        print(f"Nc={nc:>9} Ne={ne:>2} v{v}: insert {n / ms_i / 1e6:6.1f} G/s  lookup {n / ms_l / 1e6:6.1f} G/s "
              f"({b_l / ms_l / 1e6:6.0f} GB/s algorithmic)", flush=True)
    t.close()
