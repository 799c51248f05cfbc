"""Generates tests/golden/ from the reference itself (oracle/_ref/libmcref.so:
the reference's sources compiled in place, run here). The fixtures pin the
oracle and the CUDA path on machines without /root/reference.

    python tests/golden/make_golden.py

Contents (golden.json + golden.npz):
* App. A known answers: hashes, codec, mip level, texel indices,
  RNG, cone spread, footprint, memory_bytes;
* random-vector goldens: hash/codec/mip/texel/footprint/fbm/rng over seeded
  inputs, plus ops::sin_wave / ops::power from glibc (for the ulp report);
* the App. A material program: listing and execute() values (miss, hit);
* the C1-style parity scene (cornell, libm-free): program listings and a
  cache-off and an epoch-sequential cached render (radiance, nodes_found,
  table dump checksum).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from paper_2305_07238_b200 import descriptors, scenes  # noqa: E402
from _oracle import Ref, RenderParamsC, build_oracle  # noqa: E402

GOLDEN_SCENE = dict(kind="cornell", width=32, height=24, tris_per_side=4, libm_ops=False, seed=0)
EXAMPLE_MATERIAL = {
    "material_id": 7, "output": 9,
    "nodes": [
        {"id": 0, "kind": "normal"}, {"id": 1, "kind": "incoming"},
        {"id": 2, "kind": "dot", "inputs": [0, 1]},
        {"id": 3, "kind": "checker", "params": {"scale": 4.0}},
        {"id": 4, "kind": "noise_fbm", "params": {"octaves": 6, "frequency": 3.0}},
        {"id": 5, "kind": "const_float", "params": {"value": 0.5}},
        {"id": 6, "kind": "mix", "inputs": [3, 4, 5]},
        {"id": 7, "kind": "mul", "inputs": [2, 6]},
        {"id": 8, "kind": "bsdf_diffuse", "inputs": [7]},
        {"id": 9, "kind": "bsdf_output", "inputs": [8]},
    ],
}


def example_scene_dir(out: str) -> str:
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "mat.json"), "w") as f:
        json.dump(EXAMPLE_MATERIAL, f)
    scene = {"camera": {"position": [0, 0, 5], "look_at": [0, 0, 0], "vfov_deg": 45.0},
             "materials": ["mat.json"]}
    with open(os.path.join(out, "scene.json"), "w") as f:
        json.dump(scene, f)
    return os.path.join(out, "scene.json")


def random_inputs(seed: int = 7, n: int = 4096):
    r = np.random.default_rng(seed)
    desc = descriptors(r.integers(0, 8, n), r.integers(0, 300, n), r.integers(0, 25, n),
                       r.integers(0, 1 << 24, n), r.integers(0, 1 << 24, n))
    rgb = np.exp(r.uniform(np.log(1e-6), np.log(1e4), (n, 3))).astype(np.float32)
    rgb[: n // 8] *= np.float32(-1)
    rgb[n // 8: n // 4, 1] = 0
    uv = r.uniform(-3, 3, (n, 2)).astype(np.float32)
    g1 = (np.exp(r.uniform(np.log(1e-9), np.log(2.0), (n, 2))) * r.choice([-1, 1], (n, 2))).astype(np.float32)
    g2 = (np.exp(r.uniform(np.log(1e-9), np.log(2.0), (n, 2))) * r.choice([-1, 1], (n, 2))).astype(np.float32)
    fp_in = np.zeros((n, 17), np.float32)
    fp_in[:, 0] = r.uniform(0, 0.1, n)
    for a, b in ((1, 4), (4, 7)):
        v = r.normal(size=(n, 3))
        fp_in[:, a:b] = v / np.linalg.norm(v, axis=1, keepdims=True)
    fp_in[:, 7:13] = r.uniform(-2, 2, (n, 6))
    fp_in[:, 13:17] = r.uniform(-1, 1, (n, 4))
    fp_in[: n // 16, 4:7] = -fp_in[: n // 16, 1:4]  # perpendicular hits (any_tangent path)
    octaves = r.integers(1, 11, n).astype(np.int32)
    fbm_p = np.stack([r.uniform(0.5, 20, n), r.uniform(1.5, 2.5, n), r.uniform(0.3, 0.7, n)], 1).astype(np.float32)
    rng_px = r.integers(0, 1 << 22, n).astype(np.uint64)
    rng_s = r.integers(0, 512, n).astype(np.uint64)
    rng_d = r.integers(0, 400, n).astype(np.uint32)
    x = r.uniform(-50, 50, n).astype(np.float32)
    y = r.uniform(-3, 3, n).astype(np.float32)
    return dict(desc=desc, rgb=rgb, uv=uv, g1=g1, g2=g2, fp_in=fp_in, octaves=octaves, fbm_p=fbm_p,
                fbm_uv=uv, rng_px=rng_px, rng_s=rng_s, rng_d=rng_d, x=x, y=y)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    build_oracle(ref=True)
    ref = Ref()
    G: dict = {"source": "oracle/_ref/libmcref.so (reference sources compiled in place)"}
    # ---- App. A known answers
    app_desc = descriptors([0, 7, 1], [0, 42, 2], [0, 5, 24], [0, 3, 16777215], [0, 9, 0])
    cell, chk = ref.hash(app_desc)
    G["app_a_hash"] = {"desc": [[0, 0, 0, 0, 0], [7, 42, 5, 3, 9], [1, 2, 24, 16777215, 0]],
                       "cell": [f"{int(c):016x}" for c in cell], "check": [f"{int(c):08x}" for c in chk]}
    codec_in = np.array([[0, 0, 0], [1, 1, 1], [1000, .5, .25], [.2, .4, .6]], np.float32)
    enc = ref.encode(codec_in)
    G["app_a_codec"] = {"in": codec_in.tolist(), "enc": [f"{int(e):08x}" for e in enc],
                        "dec": ref.decode(enc).tolist()}
    mip_cases = [((.25, 0), (0, .25), 0), ((.3, 0), (0, .1), 0), ((1, 0), (0, 1), 0),
                 ((0, 0), (0, 0), 0), ((.25, 0), (0, .25), 1)]
    G["app_a_mip"] = []
    for g1, g2, off in mip_cases:
        m, _ = ref.mip_texel(np.zeros((1, 2)), np.array([g1]), np.array([g2]), off)
        G["app_a_mip"].append([list(g1), list(g2), off, int(m[0])])
    G["app_a_rng"] = ref.rng(1, np.zeros(3, np.uint64), np.zeros(3, np.uint64),
                             np.arange(3, dtype=np.uint32)).tolist()
    G["app_a_cone_spread_90deg_1080"] = float(ref.L.ref_cone_spread(np.float32(np.pi / 2), 1080))
    mb = np.zeros(1, np.uint64)
    ref.L.ref_memory_bytes(10**7, 10, mb.ctypes.data_as(__import__("ctypes").c_void_p))
    G["memory_bytes_1e7_10"] = int(mb[0])

    # ---- random vectors
    R = random_inputs()
    cell, chk = ref.hash(R["desc"])
    enc = ref.encode(R["rgb"])
    mip, txy = ref.mip_texel(R["uv"], R["g1"], R["g2"], 0)
    mip2, txy2 = ref.mip_texel(R["uv"], R["g1"], R["g2"], 2)
    fpo = ref.footprint(R["fp_in"])
    fbm = ref.fbm(R["octaves"], R["fbm_p"], R["fbm_uv"])
    rng = ref.rng(0x230507238, R["rng_px"], R["rng_s"], R["rng_d"])
    sinw = ref.sin_wave(R["x"])
    powv = ref.power(np.abs(R["x"]) * np.float32(0.05), R["y"])
    np.savez_compressed(os.path.join(HERE, "golden.npz"), cell=cell, check=chk, enc=enc,
                        dec=ref.decode(enc), mip=mip, txy=txy, mip2=mip2, txy2=txy2, footprint=fpo,
                        fbm=fbm, rng=rng, sin_wave=sinw, power=powv)

    # ---- App. A program
    ex = example_scene_dir(os.path.join("/tmp", "mcg_golden_example"))
    s = ref.scene_load(ex)
    G["example_listing"] = ref.disassemble(s, 0)
    sp = np.zeros((1, 15), np.float32)
    sp[0, 3:6] = [0, 0, 1]
    sp[0, 6:9] = [0, 0, -1]
    sp[0, 9:11] = [.3, .7]
    sp[0, 11:15] = [.01, 0, 0, .01]
    G["example_eval_reference"] = ref.eval_reference(s, 0, sp)[0, :3].tolist()
    c = ref.cache_new(1000, 4)
    miss = ref.execute(s, 0, sp, cache=c)
    hit = ref.execute(s, 0, sp, cache=c)
    G["example_execute"] = {"miss": miss[0][0, :3].tolist(), "hit": hit[0][0, :3].tolist(),
                            "nodes": [int(miss[1][0]), int(hit[1][0])],
                            "instrs": [int(miss[2][0]), int(hit[2][0])],
                            "counters": ref.cache_counters(c).tolist()}
    ref.cache_free(c)

    # ---- parity scene
    d = os.path.join("/tmp", "mcg_golden_scene")
    path = scenes.build_scene(scenes.SceneSpec(**GOLDEN_SCENE), d)
    s = ref.scene_load(path)
    n = ref.L.ref_scene_materials(s)
    G["scene"] = GOLDEN_SCENE
    G["scene_listings"] = [ref.disassemble(s, i) for i in range(n)]
    G["scene_analysis"] = [ref.analysis_json(s, i) for i in range(n)]
    w, h = GOLDEN_SCENE["width"], GOLDEN_SCENE["height"]
    renders = {}
    for name, mode in (("off", 0), ("sequential", 1)):
        P = RenderParamsC(w, h, 4, 4, mode, 0, 997, 4, 0, 1, 0.2, 16, 0, 1, 0, 0, 1)
        c = ref.cache_new(997, 4) if mode else None
        rad, nodes, samples, hps, st = ref.render(s, P, w, h, cache=c)
        r = {"radiance_sha": sha(rad), "nodes_sha": sha(nodes), "radiance_mean": float(rad.mean()),
             "nodes_sum": float(nodes.sum()), "samples": int(samples.sum()),
             "hits_per_sample": [int(x) for x in hps], "lookups": int(st.lookups),
             "hits": int(st.hits), "inserts_won": int(st.inserts_won),
             "instructions": int(st.instructions_executed)}
        if c is not None:
            r["table_sha"] = sha(ref.cache_slots(c, 997 * 4))
            ref.cache_free(c)
        renders[name] = r
    G["scene_renders"] = renders
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(G, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
