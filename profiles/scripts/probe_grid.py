"""Probe-kernel sweep: variant x blocks/SM on the 1e7 x 10 table."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2305_07238_b200 import Context, MaterialCache
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
ctx = Context(0)
n = 1 << 26
for v in (0, 3):
    for per_sm in (1, 2, 3, 4, 8):
        t = MaterialCache(10_000_000, 10, ctx)
        enc = 16 * v + 256 * per_sm
        ms_i, by_i = t.probe_bench(n, 7, 0 + enc, 1)
        ms_l, by_l = t.probe_bench(n, 7, 1 + enc, 3)
        ms_m, by_m = t.probe_bench(n, 8, 2 + enc, 3)
        print(json.dumps({"variant": v, "blocks_per_sm": per_sm,
                          "insert": round(by_i / ms_i / 1e6 / peak, 3), "lookup": round(by_l / ms_l / 1e6 / peak, 3),
                          "mix": round(by_m / ms_m / 1e6 / peak, 3), "lookup_Gps": round(n / ms_l / 1e6, 2)}))
        t.close()
