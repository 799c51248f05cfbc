"""Probe-kernel variants on the 1e7 x 10 table (2^26 descriptors): insert-all,
lookup-all, 50/50 mix; prints achieved algorithmic GB/s and the fraction of
the measured HBM peak."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2305_07238_b200 import Context, MaterialCache
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
ctx = Context(0)
n = 1 << 26
out = {}
for v in (0, 1, 2):
    t = MaterialCache(10_000_000, 10, ctx)
    res = {}
    for name, ph, seed, it in (("insert_all", 0, 7, 1), ("lookup_all", 1, 7, 3), ("mix", 2, 8, 3)):
        if name == "lookup_all":
            t.probe_bench(n, 7, 1 + 16 * v, 1)  # warm
        ms, by = t.probe_bench(n, seed, ph + 16 * v, it)
        res[name] = {"ms": round(ms, 3), "GBps": round(by / ms / 1e6, 1), "frac": round(by / ms / 1e6 / peak, 3),
                     "Gprobe_s": round(n / ms / 1e6, 2)}
    out[f"variant{v}"] = res
    t.close()
print(json.dumps(out, indent=1))
