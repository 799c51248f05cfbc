"""Probe variants 4 (cooperative) vs 5/6/7 (software-pipelined, U = 2/4/1
batches per warp step) x blocks/SM on the 1e7 x 10 table, same call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2305_07238_b200 import Context, MaterialCache  # noqa: E402

ctx = Context(0)
n = 1 << 26
nc, ne = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (10_000_000, 10)
t = MaterialCache(nc, ne, ctx)
VAR = eval(sys.argv[3]) if len(sys.argv) > 3 else ((4, (4, 8)), (7, (4, 8)), (5, (2, 4, 6, 8)), (6, (1, 2, 4)))
for v, bpss in VAR:
    for bps in bpss:
        out = []
        for rep in range(2):
            t.clear()
            res = []
            for ph in (0, 1, 2):
                if ph == 2:
                    t.clear()
                    t.probe_bench(n // 2, 7, 0 + 16 * v + 256 * bps, 1)  # half full
                it = 1 if ph == 0 else 3
                ms, by = t.probe_bench(n, 7 if ph < 2 else 8, ph + 16 * v + 256 * bps, it)
                res.append((n / ms / 1e6, by / ms / 1e6))
            out.append(res)
        best = [max(out[0][k], out[1][k]) for k in range(3)]
        print(f"Nc={nc} Ne={ne} v{v} b{bps}: " + " | ".join(
            f"{nm} {g:5.1f} G/s {b:5.0f} GB/s ({b / 6547.5:.3f})" for nm, (g, b) in zip(("ins", "look", "mix"), best)),
            flush=True)
