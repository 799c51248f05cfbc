"""Seeded synthetic scenes in the reference's own file formats.

The reference ships no scenes or fixtures; its loaders define the
formats: scene JSON (src/scene.cpp:300-387), material graph JSON
(src/graph.cpp:242-287) and binary PPM textures (src/image.cpp:102-126).
This module writes such files so that both the reference (oracle/_ref) and
this framework load byte-identical inputs.

Scene analogues: the five paper scenes are proprietary, so each
analogue reproduces the property that drove its measured speed-up:

* ``classroom``  - few heavy (>=100-node) procedural materials, one high cache
  point over FBM / texture / ramp stacks, modest uv tiling.
* ``junkshop``   - more materials, two mid-level cache points each.
* ``italianflat`` / ``monster`` - many cheap, low-level cache points.
* ``bmw``        - uv footprints far below the finest virtual texel (the
  level clamps at 24), so texels are unique per sample, hits ~ 0 and every
  miss inserts: the cache's pure overhead.
* ``cornell``    - the small C1 parity scene (one depth-8 material per wall).

Every material's post-order starts with an Other-class operand: the
reference compiler rejects programs that open with a CacheLookup
(src/stackvm.cpp:232-236).
"""
from __future__ import annotations

import json
import math
import os
import random
from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 0x230507238


class Graph:
    """Material graph builder: ids are dense and inputs precede consumers."""

    def __init__(self, material_id: int):
        self.material_id = material_id
        self.nodes: list[dict] = []

    def add(self, kind: str, inputs=(), **params) -> int:
        nid = len(self.nodes)
        node = {"id": nid, "kind": kind, "inputs": list(inputs)}
        if params:
            node["params"] = params
        self.nodes.append(node)
        return nid

    def finish(self, albedo: int) -> dict:
        diffuse = self.add("bsdf_diffuse", [albedo])
        out = self.add("bsdf_output", [diffuse])
        return {"material_id": self.material_id, "output": out, "nodes": self.nodes}


def _f(x: float) -> float:
    return float(np.float32(x))


class UvExpr:
    """Random uv-only (cacheable) expressions."""

    def __init__(self, g: Graph, rng: random.Random, textures: list[str], uv_scale: float,
                 libm_ops: bool, noise_freq: float = 1.0):
        self.g, self.rng, self.textures = g, rng, textures
        self.uv_scale, self.libm_ops, self.noise_freq = uv_scale, libm_ops, noise_freq

    def const(self, color: bool) -> int:
        r = self.rng
        if color:
            return self.g.add("const_color", rgb=[_f(r.uniform(0.05, 0.95)) for _ in range(3)])
        return self.g.add("const_float", value=_f(r.uniform(0.1, 0.9)))

    def leaf(self) -> int:
        r, g = self.rng, self.g
        k = r.random()
        if k < 0.45:
            return g.add("noise_fbm", octaves=r.randint(4, 8),
                         frequency=_f(r.uniform(2.0, 9.0) * self.uv_scale * self.noise_freq),
                         lacunarity=_f(r.uniform(1.8, 2.3)), gain=_f(r.uniform(0.4, 0.6)))
        if k < 0.6:
            return g.add("checker", scale=_f(r.choice([2.0, 4.0, 8.0, 16.0]) * self.uv_scale *
                                                self.noise_freq))
        if k < 0.75 and self.textures:
            return g.add("tex_image", image=r.choice(self.textures),
                         wrap=r.choice(["repeat", "repeat", "clamp"]))
        if k < 0.85:
            return g.add("uv", channel=r.choice(["u", "v", "uv"]))
        return self.const(r.random() < 0.5)

    def expr(self, depth: int) -> int:
        r, g = self.rng, self.g
        if depth <= 0:
            return self.leaf()
        k = r.random()
        if k < 0.22:
            return g.add("mix", [self.expr(depth - 1), self.expr(depth - 1), self.expr(depth - 2)])
        if k < 0.36:
            return g.add("color_ramp", [self.expr(depth - 1)], stops=self.ramp_stops())
        if k < 0.48:
            return g.add("mul", [self.expr(depth - 1), self.expr(depth - 1)])
        if k < 0.6:
            return g.add("add", [self.expr(depth - 1), self.const(r.random() < 0.5)])
        if k < 0.7:
            return g.add("clamp", [g.add("sub", [self.expr(depth - 1), self.expr(depth - 2)])])
        if k < 0.78 and self.libm_ops:
            return g.add("sin_wave", [self.expr(depth - 1)])
        if k < 0.84 and self.libm_ops:
            return g.add("power", [self.expr(depth - 1), self.const(False)])
        if k < 0.9:
            return g.add("div", [self.expr(depth - 1), g.add("add", [self.expr(depth - 2),
                                                                     self.const(False)])])
        return g.add("clamp", [self.expr(depth - 1)])

    def ramp_stops(self) -> list[dict]:
        n = self.rng.randint(2, 5)
        ts = sorted(_f(self.rng.uniform(0, 1)) for _ in range(n))
        return [{"t": t, "rgb": [_f(self.rng.uniform(0.05, 0.95)) for _ in range(3)]} for t in ts]

    def heavy(self, min_nodes: int) -> int:
        """A large uv subtree: layered FBM stacks mixed through ramps."""
        g, r = self.g, self.rng
        start = len(g.nodes)
        acc = self.layer()
        while len(g.nodes) - start < min_nodes:
            acc = g.add("mix", [acc, self.layer(), self.expr(2)])
        return g.add("clamp", [acc])

    def layer(self) -> int:
        g, r = self.g, self.rng
        n = g.add("noise_fbm", octaves=r.randint(5, 8),
                  frequency=_f(r.uniform(2.0, 12.0) * self.uv_scale * self.noise_freq),
                  lacunarity=_f(r.uniform(1.9, 2.2)), gain=_f(r.uniform(0.45, 0.6)))
        ramp = g.add("color_ramp", [n], stops=self.ramp_stops())
        return g.add("mix", [ramp, self.expr(2), self.expr(1)])


def other_gate(g: Graph) -> int:
    """Other-class scalar ~1 that opens every program."""
    n = g.add("normal")
    return g.add("clamp", [g.add("dot", [n, n])])


def material_heavy(mid, rng, textures, uv_scale, libm_ops, min_nodes=100, noise_freq=1.0):
    g = Graph(mid)
    gate = other_gate(g)
    cp = UvExpr(g, rng, textures, uv_scale, libm_ops, noise_freq).heavy(min_nodes)
    return g.finish(g.add("mul", [gate, cp]))


def material_midlevel(mid, rng, textures, uv_scale, libm_ops, noise_freq=1.0):
    g = Graph(mid)
    gate = other_gate(g)
    ex = UvExpr(g, rng, textures, uv_scale, libm_ops, noise_freq)
    a = g.add("mul", [gate, ex.heavy(25)])
    inc = g.add("incoming")
    fac = g.add("clamp", [g.add("dot", [inc, inc])])
    b = ex.heavy(25)
    return g.finish(g.add("mix", [a, b, g.add("mul", [fac, g.add("const_float", value=0.5)])]))


def material_lowlevel(mid, rng, textures, uv_scale, libm_ops, n_points=6, noise_freq=1.0):
    g = Graph(mid)
    acc = other_gate(g)
    ex = UvExpr(g, rng, textures, uv_scale, libm_ops, noise_freq)
    acc = g.add("mul", [acc, g.add("const_float", value=0.2)])
    for _ in range(n_points):
        small = ex.expr(1) if rng.random() < 0.5 else g.add(
            "mul", [ex.leaf(), ex.const(True)])
        pos = g.add("position")
        w = g.add("clamp", [g.add("dot", [pos, g.add("const_color", rgb=[0.0, 0.0, 0.0])])])
        term = g.add("mix", [small, ex.const(True), w])
        acc = g.add("add", [acc, g.add("mul", [term, g.add("const_float", value=_f(0.8 / n_points))])])
    return g.finish(g.add("clamp", [acc]))


def material_hostile(mid, rng, textures, uv_scale, libm_ops, n_terms=12, noise_freq=1.0):
    """Cache-hostile material (acceptance criterion 7): heavy FBM
    work whose every uv-only subtree is a single node consumed by an
    Other-class product, below analysis' min_subtree_size (3) -- zero cache
    points, so the cache can only add overhead."""
    g = Graph(mid)
    acc = g.add("mul", [other_gate(g), g.add("const_float", value=0.1)])
    ex = UvExpr(g, rng, textures, uv_scale, libm_ops, noise_freq)
    for _ in range(n_terms):
        leaf = g.add("noise_fbm", octaves=rng.randint(5, 8),
                     frequency=_f(rng.uniform(2.0, 9.0) * uv_scale * noise_freq),
                     lacunarity=_f(rng.uniform(1.8, 2.3)), gain=_f(rng.uniform(0.4, 0.6)))
        pos = g.add("position")
        w = g.add("clamp", [g.add("dot", [pos, g.add("const_color", rgb=[_f(0.05), _f(0.1), _f(0.02)])])])
        acc = g.add("add", [acc, g.add("mul", [leaf, w])])
    _ = ex
    return g.finish(g.add("clamp", [acc]))


def material_depth8(mid, rng, textures, libm_ops=False):
    """The C1 parity material: one depth-8 uv expression behind the gate."""
    g = Graph(mid)
    gate = other_gate(g)
    cp = UvExpr(g, rng, textures, 1.0, libm_ops).expr(8)
    return g.finish(g.add("mul", [gate, g.add("clamp", [cp])]))


def random_material(mid, rng, textures, libm_ops=True, depth=None):
    """Random valid graph for the VM-vs-oracle suite (200 graphs)."""
    g = Graph(mid)
    first = rng.random()
    if first < 0.3:
        gate = other_gate(g)
    elif first < 0.6:
        p = g.add("position")
        gate = g.add("mul", [p, g.add("const_float", value=_f(rng.uniform(0.1, 1)))])
    else:
        gate = g.add("incoming")
    ex = UvExpr(g, rng, textures, 1.0, libm_ops)
    d = depth if depth is not None else rng.randint(1, 7)
    body = ex.expr(d)
    op = rng.choice(["mul", "add", "mix", "sub"])
    if op == "mix":
        top = g.add("mix", [gate, body, ex.expr(2)])
    else:
        top = g.add(op, [gate, body])
    if rng.random() < 0.5:
        top = g.add("clamp", [top])
    return g.finish(top)


# ---------------------------------------------------------------- geometry

@dataclass
class Mesh:
    positions: list = field(default_factory=list)
    uvs: list = field(default_factory=list)
    indices: list = field(default_factory=list)
    material: int = 0

    def quad_grid(self, origin, eu, ev, nu, nv, uv_scale, uv_offset=(0.0, 0.0), uv_span=0.0):
        """Subdivided planar quad, uv = planar coordinates x uv_scale; with
        uv_span > 0 the quad's uv runs over [0, uv_span] on both axes
        whatever its size (one texture tile per surface, like an unwrapped
        asset: texel_indices' wrap (raycone.cpp:75-83) then never folds two
        surface points onto one virtual texel)."""
        o, eu, ev = np.asarray(origin, np.float64), np.asarray(eu, np.float64), np.asarray(ev, np.float64)
        base = len(self.positions) // 3
        lu, lv = np.linalg.norm(eu), np.linalg.norm(ev)
        if uv_span > 0.0:
            uv_scale, lu, lv = uv_span, 1.0, 1.0
        for j in range(nv + 1):
            for i in range(nu + 1):
                p = o + eu * (i / nu) + ev * (j / nv)
                self.positions += [_f(c) for c in p]
                self.uvs += [_f(uv_offset[0] + uv_scale * lu * i / nu),
                             _f(uv_offset[1] + uv_scale * lv * j / nv)]
        for j in range(nv):
            for i in range(nu):
                a = base + j * (nu + 1) + i
                b, c, d = a + 1, a + nu + 1, a + nu + 2
                self.indices += [a, b, d, a, d, c]

    def box(self, lo, hi, n, uv_scale, uv_span=0.0):
        lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
        dx, dy, dz = hi - lo
        X, Y, Z = np.array([dx, 0, 0]), np.array([0, dy, 0]), np.array([0, 0, dz])
        self.quad_grid(lo, X, Z, n, n, uv_scale, uv_span=uv_span)                 # bottom
        self.quad_grid(lo + Y, Z, X, n, n, uv_scale, uv_span=uv_span)             # top
        self.quad_grid(lo, Y, X, n, n, uv_scale, uv_span=uv_span)                 # front (z = lo)
        self.quad_grid(lo + Z, X, Y, n, n, uv_scale, uv_span=uv_span)             # back
        self.quad_grid(lo, Z, Y, n, n, uv_scale, uv_span=uv_span)                 # left
        self.quad_grid(lo + X, Y, Z, n, n, uv_scale, uv_span=uv_span)             # right

    def to_json(self):
        return {"positions": self.positions, "uvs": self.uvs, "indices": self.indices,
                "material": self.material}


def write_ppm(path: str, img: np.ndarray) -> None:
    h, w, _ = img.shape
    with open(path, "wb") as f:
        f.write(b"P6\n# synthetic texture\n%d %d\n255\n" % (w, h))
        f.write(np.ascontiguousarray(img, dtype=np.uint8).tobytes())


def make_textures(out_dir: str, rng: random.Random, n: int = 2, size: int = 128) -> list[str]:
    names = []
    for t in range(n):
        y, x = np.mgrid[0:size, 0:size].astype(np.float64) / size
        fx, fy = rng.uniform(2, 9), rng.uniform(2, 9)
        r = 0.5 + 0.5 * np.sin(2 * np.pi * (fx * x + 0.3 * y))
        g = 0.5 + 0.5 * np.cos(2 * np.pi * fy * y)
        b = ((np.floor(x * 8) + np.floor(y * 8)) % 2) * 0.7 + 0.15
        img = np.stack([r, g, b], -1) * 255.0
        name = f"tex_{t}.ppm"
        write_ppm(os.path.join(out_dir, name), np.clip(np.round(img), 0, 255))
        names.append(name)
    return names


@dataclass
class SceneSpec:
    kind: str
    width: int = 1920
    height: int = 1080
    seed: int = 0
    libm_ops: bool = True
    tris_per_side: int = 10
    spheres: int = 0           # analytic spheres (scene.cpp:80-97, 222-249) inside the room
    uv_span: float = 0.0       # > 0: every quad's uv spans [0, uv_span] (no tiling; Mesh.quad_grid)


def _room(materials: list[int], rng: random.Random, uv_scale: float, n: int,
          objects: int = 6, uv_span: float = 0.0) -> list[Mesh]:
    """A box room (open towards the camera) with a few boxes inside."""
    meshes = []
    def surface(mat, fn):
        m = Mesh(material=mat)
        fn(m)
        meshes.append(m)
    W, H, D = 8.0, 5.0, 10.0
    mats = iter(materials * 8)
    surface(next(mats), lambda m: m.quad_grid([-W, 0, -D], [0, 0, 2 * D], [2 * W, 0, 0], n, n, uv_scale, uv_span=uv_span))   # floor
    surface(next(mats), lambda m: m.quad_grid([-W, H, -D], [2 * W, 0, 0], [0, 0, 2 * D], n, n, uv_scale, uv_span=uv_span))   # ceiling
    surface(next(mats), lambda m: m.quad_grid([-W, 0, -D], [2 * W, 0, 0], [0, H, 0], n, n, uv_scale, uv_span=uv_span))       # back
    surface(next(mats), lambda m: m.quad_grid([-W, 0, D], [0, 0, -2 * D], [0, H, 0], n, n, uv_scale, uv_span=uv_span))      # left
    surface(next(mats), lambda m: m.quad_grid([W, 0, -D], [0, 0, 2 * D], [0, H, 0], n, n, uv_scale, uv_span=uv_span))       # right
    for k in range(objects):
        cx, cz = rng.uniform(-W + 1.5, W - 1.5), rng.uniform(-D + 2, 2)
        sx, sy, sz = rng.uniform(0.5, 1.5), rng.uniform(0.5, 2.5), rng.uniform(0.5, 1.5)
        surface(next(mats), lambda m: m.box([cx - sx, 0.0, cz - sz], [cx + sx, sy, cz + sz],
                                            max(2, n // 4), uv_scale, uv_span))
    return meshes


def build_scene(spec: SceneSpec, out_dir: str) -> str:
    """Writes scene.json + materials + textures; returns the scene path."""
    os.makedirs(out_dir, exist_ok=True)
    rng = random.Random(BASE_SEED + spec.seed * 7919 + hash(spec.kind) % 1000)
    rng = random.Random(f"{BASE_SEED}:{spec.kind}:{spec.seed}")
    textures = make_textures(out_dir, rng)
    mats: list[dict] = []
    uv_scale, noise_freq = 0.5, 1.0
    kind = spec.kind
    if kind == "classroom":
        for i in range(3):
            mats.append(material_heavy(i, rng, textures, 1.0, spec.libm_ops, min_nodes=100))
        uv_scale = 0.35
    elif kind == "junkshop":
        for i in range(8):
            mats.append(material_midlevel(i, rng, textures, 1.0, spec.libm_ops))
        uv_scale = 0.5
    elif kind in ("italianflat", "monster"):
        npts = 6 if kind == "italianflat" else 10
        for i in range(6):
            mats.append(material_lowlevel(i, rng, textures, 1.0, spec.libm_ops, n_points=npts))
        uv_scale = 0.5
    elif kind == "bmw":
        # uv footprints ~1e-8: the virtual level clamps at 24 and every
        # sample owns its texel; noise frequency compensates for appearance.
        for i in range(4):
            mats.append(material_heavy(i, rng, textures, 1.0, spec.libm_ops, min_nodes=60,
                                       noise_freq=2.0e4))
        uv_scale = 0.5e-4
    elif kind == "cornell":
        for i in range(3):
            mats.append(material_depth8(i, rng, textures, spec.libm_ops))
        uv_scale = 0.5
    elif kind == "hostile":
        for i in range(4):
            mats.append(material_hostile(i, rng, textures, 1.0, spec.libm_ops))
        uv_scale = 0.5
    else:
        raise ValueError(f"unknown scene kind {kind!r}")

    mat_files = []
    for m in mats:
        name = f"mat_{m['material_id']}.json"
        with open(os.path.join(out_dir, name), "w") as f:
            json.dump(m, f)
        mat_files.append(name)
    ids = [m["material_id"] for m in mats]
    meshes = _room(ids, rng, uv_scale, spec.tris_per_side, uv_span=spec.uv_span)
    scene = {
        "camera": {"position": [0.0, 2.4, 17.0], "look_at": [0.0, 1.6, 0.0], "up": [0.0, 1.0, 0.0],
                   "vfov_deg": 55.0, "width": spec.width, "height": spec.height},
        "materials": mat_files,
        "meshes": [m.to_json() for m in meshes],
        "lights": [
            {"type": "rect", "corner": [-2.0, 4.95, -3.0], "edge_u": [4.0, 0.0, 0.0],
             "edge_v": [0.0, 0.0, 3.0], "radiance": [6.0, 5.8, 5.4]},
            {"type": "point", "position": [3.0, 3.5, 4.0], "intensity": [20.0, 18.0, 16.0]},
        ],
        "env": [0.05, 0.06, 0.08],
    }
    if spec.spheres:
        srng = random.Random(f"{BASE_SEED}:{spec.kind}:{spec.seed}:spheres")
        scene["spheres"] = [
            {"center": [_f(srng.uniform(-6.5, 6.5)), _f(srng.uniform(0.6, 4.0)), _f(srng.uniform(-8.0, 6.0))],
             "radius": _f(srng.uniform(0.25, 0.9)), "material": ids[k % len(ids)]}
            for k in range(spec.spheres)]
    path = os.path.join(out_dir, "scene.json")
    with open(path, "w") as f:
        json.dump(scene, f)
    return path


def materials_only_scene(out_dir: str, n: int, seed: int, libm_ops: bool = True,
                         depth=None) -> str:
    """A geometry-free scene holding n random materials (VM parity suite)."""
    os.makedirs(out_dir, exist_ok=True)
    rng = random.Random(f"{BASE_SEED}:materials:{seed}")
    textures = make_textures(out_dir, rng, n=2, size=32)
    files = []
    for i in range(n):
        m = random_material(i, rng, textures, libm_ops=libm_ops, depth=depth)
        name = f"mat_{i}.json"
        with open(os.path.join(out_dir, name), "w") as f:
            json.dump(m, f)
        files.append(name)
    scene = {"camera": {"position": [0, 0, 5], "look_at": [0, 0, 0], "vfov_deg": 45.0},
             "materials": files}
    path = os.path.join(out_dir, "scene.json")
    with open(path, "w") as f:
        json.dump(scene, f)
    return path


def random_shading_points(n: int, seed: int, uv_range: float = 4.0) -> np.ndarray:
    """n x 15 float32: position, normal, incoming, uv, g1, g2."""
    r = np.random.default_rng(seed)
    pos = r.uniform(-3, 3, (n, 3))
    nrm = r.normal(size=(n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    inc = r.normal(size=(n, 3))
    inc /= np.linalg.norm(inc, axis=1, keepdims=True)
    uv = r.uniform(-uv_range, uv_range, (n, 2))
    g = np.exp(r.uniform(math.log(1e-6), math.log(0.5), (n, 4))) * r.choice([-1, 1], (n, 4))
    return np.concatenate([pos, nrm, inc, uv, g], axis=1).astype(np.float32)
