"""One probe-bench configuration (for ncu): variant, blocks/SM, phase."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2305_07238_b200 import Context, MaterialCache
v, per_sm = int(sys.argv[1]), int(sys.argv[2])
n_cells = int(sys.argv[3]) if len(sys.argv) > 3 else 10_000_000
ctx = Context(0)
t = MaterialCache(n_cells, 10, ctx)
n = 1 << 26
t.probe_bench(n, 7, 0 + 16 * v + 256 * per_sm, 1)   # fill
t.probe_bench(n, 7, 1 + 16 * v + 256 * per_sm, 1)   # lookup-all (profiled: 2nd launch)
