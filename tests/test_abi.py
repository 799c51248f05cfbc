"""The C-ABI library without a GPU: it loads, exports every entry point
include/mcg.h declares, and its host-side calls behave like the reference
(memory_bytes, audit_dump, scene queries, experiment outputs)."""
import ctypes as C
import json
import os
import re
import struct

import numpy as np
import pytest

import paper_2305_07238_b200 as P
from paper_2305_07238_b200 import _native as N

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "mcg.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mcg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_function(built):
    L = C.CDLL(N.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, f"not exported: {missing}"
    # and the Python binding covers all of them
    assert sorted(set(names) - set(N.EXPORTED)) == []
    assert N.lib().mcg_abi_version() == N.ABI_VERSION == 4


def test_memory_bytes():
    assert P.memory_bytes(10**7, 10) == 800_000_000   # SPEC.md:505 #1 ("about 763 MB")
    assert abs(P.memory_bytes(10**7, 10) / 2**20 - 762.94) < 0.01
    assert P.memory_bytes(0, 10) == 0
    with pytest.raises(OverflowError):
        P.memory_bytes(1 << 61, 16)


def _dump(path, nc, ne, words):
    with open(path, "wb") as f:
        f.write(struct.pack("<QQ", nc, ne))
        f.write(np.asarray(words, np.uint64).tobytes())


def test_audit_dump_cases(tmp_path, built):
    """audit_dump (cache.cpp:175-230): clean, duplicate check-hash, zero hash,
    truncation, trailing bytes, implausible sizes -- and the same verdicts as
    the reference's own audit when it is available."""
    import _oracle
    ref = _oracle.Ref() if _oracle.Ref.available() else None
    cases = {
        "clean": (3, 2, [0, 0, (5 << 32) | 1, (6 << 32) | 2, (5 << 32) | 9, 0], True, ""),
        "dup": (2, 3, [(7 << 32) | 1, (7 << 32) | 2, 0, 0, 0, 0], False, "duplicate check-hash in cell 0"),
        "zero_hash": (1, 2, [5, 0], False, "zero check-hash"),
        "trunc": (4, 2, [0, 0, 0], False, "truncated"),
        "trailing": (1, 1, [0, 0], False, "trailing"),
        "dims": (0, 4, [], False, "implausible"),
    }
    for name, (nc, ne, words, clean, problem) in cases.items():
        p = str(tmp_path / f"{name}.bin")
        _dump(p, nc, ne, words)
        rep = P.audit_dump(p)
        assert rep.clean == clean, name
        assert problem in rep.problem, (name, rep.problem)
        if ref is not None:
            out = np.zeros(4, np.uint64)
            prob = C.create_string_buffer(256)
            ok = ref.L.ref_audit(p.encode(), out.ctypes.data_as(C.c_void_p), prob, 256)
            assert bool(ok) == clean and prob.value.decode() == rep.problem, name
            assert int(out[2]) == rep.occupied
    rep = P.audit_dump(str(tmp_path / "nope.bin"))
    assert not rep.clean and "cannot open" in rep.problem


def test_no_device_raises_loudly(built):
    """No CPU fallback: without a GPU the device entry points fail."""
    try:
        ctx = P.Context(0)
    except P.NoDeviceError:
        return
    except P.CudaError:
        return
    ctx.close()
    pytest.skip("a GPU is present")


def test_image_error_and_stats_json():
    a = np.random.default_rng(0).uniform(0, 1, (8, 6, 3)).astype(np.float32)
    d = P.image_error(a, a)
    assert d.mean_abs == 0 and d.max_abs == 0 and not d.diff.any()       # SPEC.md:412 a == b
    d = P.image_error(a, a + np.float32(0.1))
    np.testing.assert_allclose(d.diff, 0.5, atol=1e-5)                    # 5 x 0.1
    with pytest.raises(ValueError):
        P.image_error(a, a[:4])
    fb = P.FrameBuffers(6, 8)
    fb.nodes_found[:] = 6.0
    fb.samples[:] = 3
    st = P.RenderStats(wall_time_s=1.5, lookups=10, hits=4, hit_rate=0.4)
    text = P.stats_to_json(st, fb)
    doc = json.loads(text)
    assert doc["hits"] == 4 and doc["lookups"] == 10 and len(doc["per_pixel_nodes_found"]) == 48
    sf = P.parse_stats_json(text)
    assert sf.width == 6 and sf.height == 8 and np.all(sf.per_pixel_nodes_found == 2.0)
    with pytest.raises(ValueError):
        P.parse_stats_json("{}")


def test_host_hash_codec_helpers_match_oracle(oracle):
    r = np.random.default_rng(2)
    d = P.descriptors(r.integers(0, 9, 64), r.integers(0, 999, 64), r.integers(0, 25, 64),
                      r.integers(0, 1 << 20, 64), r.integers(0, 1 << 20, 64))
    cell, chk = oracle.hash(d)
    for i in range(64):
        assert P.hash_cell(d[i]) == int(cell[i]) and P.hash_check(d[i]) == int(chk[i])
    rgb = r.uniform(-1, 50, (64, 3)).astype(np.float32)
    enc = oracle.encode(rgb)
    for i in range(64):
        assert P.encode_value(rgb[i]) == int(enc[i])
        assert P.decode_value(int(enc[i])) == tuple(oracle.decode(enc[i:i + 1])[0].tolist())


def test_codec_error_bound():
    """SPEC.md:509 #9: decode(encode(v)) max-channel relative error <= 1/256
    over log-uniform [0, 1e4]^3."""
    r = np.random.default_rng(5)
    v = np.exp(r.uniform(np.log(1e-6), np.log(1e4), (100_000, 3))).astype(np.float32)
    import _oracle
    o = _oracle.Oracle()
    dec = o.decode(o.encode(v))
    err = np.abs(dec.astype(np.float64) - v).max(axis=1) / v.max(axis=1)
    assert err.max() <= 1.0 / 256.0 + 1e-12
