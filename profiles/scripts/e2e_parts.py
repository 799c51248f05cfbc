import sys, os, time, tempfile, ctypes as C
sys.path.insert(0, "/root/repo"); os.chdir("/root/repo")
import bench, torch
from paper_2305_07238_b200 import Context, RenderConfig, load_scene
from paper_2305_07238_b200 import _native as N
ctx = Context(0)
scene = load_scene(bench.make_scene(tempfile.mkdtemp()))
L = N.lib()
for _ in range(3):
    t0 = time.perf_counter(); N.check(L.mcg_upload_scene(ctx.handle, scene.handle)); ctx.synchronize(); t1 = time.perf_counter()
    print("upload ms", (t1 - t0) * 1e3)
W, H = bench.W, bench.H
rad = torch.zeros(H * W * 3, dtype=torch.float64).pin_memory()
t0 = time.perf_counter(); rad.zero_(); t1 = time.perf_counter(); print("zero rad ms", (t1 - t0) * 1e3)
