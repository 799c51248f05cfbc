import sys, tempfile, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_2305_07238_b200 import Context, load_scene, scenes
ctx = Context(0)
path = scenes.build_scene(scenes.SceneSpec("cornell", 16, 16, tris_per_side=8), tempfile.mkdtemp())
s = load_scene(path); ctx.upload(s)
r = np.random.default_rng(4); n = 20000
o = r.uniform([-7.9, 0.01, -9.9], [7.9, 4.99, 9.9], (n, 3)); d = r.normal(size=(n, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
rays = np.concatenate([o, d], 1).astype(np.float32)
a = ctx.intersect_batch(rays, 1e-4, np.inf, 0); b = ctx.intersect_batch(rays, 1e-4, np.inf, 3)
bad = np.where((a.view(np.uint32) != b.view(np.uint32)).any(1))[0]
print("mismatch", len(bad), "of", n)
for i in bad[:5]:
    print(i, "scalar found/t", a[i,:2], "slot", a[i,10], "packed", b[i,:2], b[i,10])
oa = ctx.occluded_batch(rays, 1e-4, np.full(n, 5.0, np.float32), 0); ob = ctx.occluded_batch(rays, 1e-4, np.full(n, 5.0, np.float32), 5)
print("occluded mismatch", int((oa != ob).sum()))
cols = np.where((a.view(np.uint32) != b.view(np.uint32)).any(0))[0]
print("differing columns", cols)
i = bad[0]
print("scalar", a[i]); print("packed", b[i])
