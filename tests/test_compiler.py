"""Host compiler / scene loader (libmcg) against the reference's own code
(oracle/_ref): identical analysis JSON and instruction listings for every
material, identical error classes for invalid inputs (graph.cpp:242-333,
analysis.cpp:73-184, stackvm.cpp:15-246, scene.cpp:300-387)."""
import json
import os

import numpy as np
import pytest

from paper_2305_07238_b200 import (CompileError, GraphError, ImageIoError, SceneError, load_scene,
                                   scenes)
from paper_2305_07238_b200 import _native as N


@pytest.mark.parametrize("kind", ["cornell", "classroom", "junkshop", "italianflat", "monster", "bmw"])
def test_scene_listings_match_reference(ref, scene_dir, kind):
    path = scenes.build_scene(scenes.SceneSpec(kind, 32, 24, tris_per_side=4), f"{scene_dir}/c_{kind}")
    s = load_scene(path)
    rs = ref.scene_load(path)
    assert s.n_materials == ref.L.ref_scene_materials(rs)
    for i in range(s.n_materials):
        assert s.disassemble(i) == ref.disassemble(rs, i)
        assert s.analysis_json(i) == ref.analysis_json(rs, i)
    ref.L.ref_scene_free(rs)


@pytest.mark.parametrize("seed", range(4))
def test_random_graph_listings_match_reference(ref, scene_dir, seed):
    """SPEC.md:503-style random graphs (30 per seed, sin/pow included)."""
    path = scenes.materials_only_scene(f"{scene_dir}/rg{seed}", 30, seed=100 + seed)
    s = load_scene(path)
    rs = ref.scene_load(path)
    for i in range(s.n_materials):
        assert s.disassemble(i) == ref.disassemble(rs, i), f"material {i}"
        assert s.analysis_json(i) == ref.analysis_json(rs, i), f"material {i}"
    ref.L.ref_scene_free(rs)


@pytest.mark.parametrize("min_subtree", [1, 2, 5])
def test_min_subtree_option(ref, scene_dir, min_subtree):
    path = scenes.materials_only_scene(f"{scene_dir}/ms{min_subtree}", 10, seed=7)
    s = load_scene(path, min_subtree_size=min_subtree)
    rs = ref.scene_load(path, min_subtree)
    for i in range(s.n_materials):
        assert s.analysis_json(i) == ref.analysis_json(rs, i)
        assert s.disassemble(i) == ref.disassemble(rs, i)


def _write_scene(d, materials, extra=None):
    os.makedirs(d, exist_ok=True)
    names = []
    for k, m in enumerate(materials):
        name = f"m{k}.json"
        with open(os.path.join(d, name), "w") as f:
            f.write(m if isinstance(m, str) else json.dumps(m))
        names.append(name)
    scene = {"camera": {"position": [0, 0, 5], "look_at": [0, 0, 0], "vfov_deg": 45.0},
             "materials": names}
    scene.update(extra or {})
    p = os.path.join(d, "scene.json")
    with open(p, "w") as f:
        json.dump(scene, f)
    return p


def _mat(nodes, output=None, mid=0):
    return {"material_id": mid, "output": output if output is not None else len(nodes) - 1,
            "nodes": [dict(n, id=i) for i, n in enumerate(nodes)]}


GOOD_TAIL = [{"kind": "bsdf_diffuse", "inputs": [None]}, {"kind": "bsdf_output", "inputs": [None]}]


def _chain(nodes):
    """nodes + diffuse(last) + output."""
    n = len(nodes)
    return nodes + [{"kind": "bsdf_diffuse", "inputs": [n - 1]}, {"kind": "bsdf_output", "inputs": [n]}]


BAD_GRAPHS = {
    "parse": "{not json",
    "unknown_kind": _mat(_chain([{"kind": "frobnicate"}])),
    "arity": _mat(_chain([{"kind": "add", "inputs": []}])),
    "forward_ref": _mat([{"kind": "const_float", "inputs": []}, {"kind": "clamp", "inputs": [2]},
                         {"kind": "bsdf_diffuse", "inputs": [1]}, {"kind": "bsdf_output", "inputs": [2]}]),
    "dangling": _mat(_chain([{"kind": "clamp", "inputs": [9]}])),
    "two_outputs": _mat([{"kind": "normal"}, {"kind": "bsdf_output", "inputs": [0]},
                         {"kind": "bsdf_output", "inputs": [0]}]),
    "output_not_bsdf": _mat(_chain([{"kind": "normal"}]), output=0),
    "octaves": _mat(_chain([{"kind": "noise_fbm", "params": {"octaves": 11}}])),
    "ramp_unsorted": _mat(_chain([{"kind": "uv", "params": {"channel": "u"}},
                                  {"kind": "color_ramp", "inputs": [0], "params": {"stops": [
                                      {"t": 0.5, "rgb": [1, 0, 0]}, {"t": 0.1, "rgb": [0, 1, 0]}]}}])),
    "ramp_empty": _mat(_chain([{"kind": "uv"}, {"kind": "color_ramp", "inputs": [0], "params": {"stops": []}}])),
    "bad_channel": _mat(_chain([{"kind": "uv", "params": {"channel": "w"}}])),
    "bad_wrap": _mat(_chain([{"kind": "tex_image", "params": {"image": "t.ppm", "wrap": "mirror"}}])),
    "rgb_len": _mat(_chain([{"kind": "const_color", "params": {"rgb": [1, 2]}}])),
    "sparse_ids": {"material_id": 0, "output": 2, "nodes": [
        {"id": 0, "kind": "normal"}, {"id": 2, "kind": "bsdf_diffuse", "inputs": [0]}]},
}


@pytest.mark.parametrize("case", sorted(BAD_GRAPHS))
def test_graph_errors_match_reference(built, scene_dir, case):
    path = _write_scene(f"{scene_dir}/bad_{case}", [BAD_GRAPHS[case]])
    with pytest.raises(GraphError):
        load_scene(path)
    import _oracle
    if _oracle.Ref.available():
        ref = _oracle.Ref()
        with pytest.raises(GraphError):
            ref.scene_load(path)


def test_compile_underflow_quirk(built, scene_dir):
    """A program that opens with a CacheLookup is rejected (stackvm.cpp:232-236,
    SURVEY App. B.1) -- by the reference and identically here."""
    m = _mat([{"kind": "uv", "params": {"channel": "u"}}, {"kind": "checker", "params": {"scale": 4}},
              {"kind": "mix", "inputs": [0, 1, 0]}, {"kind": "normal"},
              {"kind": "dot", "inputs": [2, 3]}, {"kind": "bsdf_diffuse", "inputs": [4]},
              {"kind": "bsdf_output", "inputs": [5]}])
    path = _write_scene(f"{scene_dir}/underflow", [m])
    with pytest.raises(CompileError, match="underflow"):
        load_scene(path)
    import _oracle
    if _oracle.Ref.available():
        with pytest.raises(CompileError):
            _oracle.Ref().scene_load(path)


def test_scene_errors(built, scene_dir):
    ok = _mat(_chain([{"kind": "normal"}]))
    p = _write_scene(f"{scene_dir}/se1", [ok], {"lights": [{"type": "spot", "position": [0, 0, 0]}]})
    with pytest.raises(SceneError, match="unknown light type"):
        load_scene(p)
    p = _write_scene(f"{scene_dir}/se2", [ok], {"meshes": [{"positions": [0, 0, 0, 1, 0, 0, 0, 1, 0],
                                                           "uvs": [0, 0, 1, 0, 0, 1], "indices": [0, 1, 2],
                                                           "material": 5}]})
    with pytest.raises(SceneError, match="does not resolve"):
        load_scene(p)
    p = _write_scene(f"{scene_dir}/se3", [ok], {"meshes": [{"positions": [0, 0, 0, 1, 0, 0, 0, 1, 0],
                                                           "uvs": [0, 0, 1, 0], "indices": [0, 1, 2],
                                                           "material": 0}]})
    with pytest.raises(SceneError, match="one uv per vertex"):
        load_scene(p)
    with pytest.raises(SceneError):
        load_scene(f"{scene_dir}/does_not_exist.json")


def test_missing_texture_is_image_io_error(built, scene_dir):
    m = _mat(_chain([{"kind": "tex_image", "params": {"image": "missing.ppm"}}]))
    p = _write_scene(f"{scene_dir}/tex_missing", [m])
    with pytest.raises(ImageIoError):
        load_scene(p)


def test_schedule_program_reproduces_compiler(built, scene_dir):
    """mcg_schedule_program (used by the C++ drop-in on reference programs)
    recomputes exactly the compiler's static stack slots and tags."""
    import ctypes as C
    path = scenes.build_scene(scenes.SceneSpec("monster", 16, 16, tris_per_side=2), f"{scene_dir}/sched")
    s = load_scene(path)
    f = s.flat
    code = np.ctypeslib.as_array(C.cast(f.code, C.POINTER(C.c_uint8)), shape=(f.n_code * 16,)).copy()
    for slot in range(f.n_programs):
        prog = f.programs[slot]
        mine = code[prog.code_offset * 16:(prog.code_offset + prog.code_len) * 16].copy()
        wiped = mine.reshape(-1, 16).copy()
        wiped[:, 2:4] = 0      # sp, tags
        wiped[:, 10] = 0       # store_ord
        buf = np.ascontiguousarray(wiped.reshape(-1))
        ms = C.c_uint32()
        N.check(N.lib().mcg_schedule_program(buf.ctypes.data_as(C.c_void_p), prog.code_len,
                                             C.cast(f.consts, C.c_void_p), f.n_consts, C.byref(ms)))
        np.testing.assert_array_equal(buf, mine)
        assert ms.value == prog.max_stack
