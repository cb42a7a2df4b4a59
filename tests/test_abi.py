"""C-ABI checks that need no GPU: the library loads, exports every entry point
include/skan.h declares, and its host-side logic (planner, SKAN v1 header /
section validation with fault kinds and byte offsets) matches the reference.
"""
import ctypes as C
import os
import re
import struct

import numpy as np
import pytest

import oracle
import paper_2512_15742_b200 as hq
from paper_2512_15742_b200 import _lib, synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not oracle.have_ref(), reason="reference build oracle/_ref unavailable")


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "skan.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(skan_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert L.skan_abi_version() == 1


def test_status_names_match_reference_taxonomy():
    L = _lib.lib()
    names = [L.skan_status_name(s).decode() for s in range(7)]
    assert names == ["OK", "ShapeError", "ValueError", "ContractError", "FormatError", "PlanError", "CudaError"]


def test_index_bits_matches_oracle():
    for k in list(range(0, 300)) + [65535, 65536, 65537, 1 << 20, (1 << 32) - 1]:
        assert hq.index_bits(k) == oracle.port().oracle_index_bits(k)


def test_plan_memory_kats_through_abi():
    import json
    kats = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_kats.json")))
    for v in kats["plan_memory"]:
        h = hq.LayerHeader(v["in"], v["out"], v["G"], v["k"], flags=1 if v["int8"] else 0)
        p = hq.plan_memory([h])
        lp = p.layers[0]
        assert (lp.codebook_bytes, lp.index_bytes, lp.unpacked_index_bytes, lp.gain_bytes, lp.bias_bytes,
                p.scratch_bytes, p.payload_total, p.working_set_total) == (
            v["codebook"], v["index"], v["unpacked"], v["gain"], v["bias"], v["scratch"], v["payload"],
            v["working"]), v["src"]
    o = kats["plan_overflow"]
    with pytest.raises(hq.PlanError):
        hq.plan_memory([hq.LayerHeader(o["in"], o["out"], o["G"], o["k"])])
    with pytest.raises(hq.PlanError):
        hq.plan_memory([hq.LayerHeader(2, 3, 1, 4)])


def test_headline_head_plan():
    """cfg2 head {2048,1408,20}, K=65536, int8: payload 12,957,696 B."""
    hs = [hq.LayerHeader(2048, 1408, 10, 65536, flags=1), hq.LayerHeader(1408, 20, 10, 65536, flags=1)]
    p = hq.plan_memory(hs)
    assert p.payload_total == 12_957_696
    # device-resident form per layer: 4 B records, the int8 codebook padded to
    # 16 B rows (twice: as stored and with the codes biased by 0x80 for the
    # tensor-core GEMM), the (c[m], c[m+1]) pair table, gain LUTs and bias
    # sums; everything 256 B aligned
    def al(v):
        return (v + 255) // 256 * 256
    want = sum(2 * al(10 * 8) + al(4 * e) + 2 * al(65536 * 16) + al(65536 * 9 * 2) + al(1024) + al(2048) + al(8 * o)
               for e, o in ((2048 * 1408, 1408), (1408 * 20, 20)))  # node positions + keys first
    assert p.device_total == want
    assert p.device_total < 126e6  # fits the B200 L2


@needs_ref
def test_plan_matches_reference_random():
    rng = np.random.default_rng(3)
    for _ in range(100):
        hs = [hq.LayerHeader(int(rng.integers(1, 3000)), int(rng.integers(1, 3000)), int(rng.integers(2, 64)),
                             int(rng.choice([0, 1, 7, 256, 65536, 65537])), flags=int(rng.integers(0, 2)))
              for _ in range(int(rng.integers(1, 4)))]
        for h in hs:
            if h.k == 0:
                h.flags = 0
        p = hq.plan_memory(hs)
        dims = np.array([[h.in_dim, h.out_dim, h.grid_size, h.k] for h in hs], np.uint32).ravel()
        flags = np.array([h.flags for h in hs], np.uint32)
        per5 = np.zeros(5 * len(hs), np.uint64)
        tot = np.zeros(3, np.uint64)
        oracle.ref().hqref_plan_memory(dims.ctypes.data, flags.ctypes.data, len(hs), per5.ctypes.data,
                                       tot.ctypes.data)
        mine = [x for lp in p.layers for x in (lp.codebook_bytes, lp.index_bytes, lp.unpacked_index_bytes,
                                              lp.gain_bytes, lp.bias_bytes)]
        assert mine == list(map(int, per5))
        assert (p.scratch_bytes, p.payload_total, p.working_set_total) == tuple(map(int, tot))


# ---------------------------------------------------------------------------
# SKAN v1 loader fault contract: header faults and truncations with no index
# section before them are raised by the host parse before any device work;
# index range checks run on the device (the @gpu cases)

def _good_int8_bytes():
    return oracle.ref_random([3, 5, 2], 6, 0.4, 9, 4, True).serialize()


def _expect_same_fault(bad: bytes, fragment: str):
    with pytest.raises(oracle.RefError) as er:
        oracle.ref_deserialize(bad)
    with pytest.raises(hq.FormatError) as eg:
        hq.deserialize(bad)
    assert er.value.code == 4
    assert int(eg.value.fault) == er.value.fault
    assert eg.value.offset == er.value.offset
    assert fragment in str(eg.value) and fragment in str(er.value)
    assert str(eg.value) == str(er.value)  # identical message, incl. "(byte offset N)"


@needs_ref
def test_corrupted_files_report_reference_fault_and_offset():
    """test_lutham.cpp:214-286 fixtures, compared against the reference itself."""
    good = bytearray(_good_int8_bytes())
    cases = []
    b = bytearray(good); b[0] = ord("X"); cases.append((b, "magic"))
    b = bytearray(good); b[4] = 9; cases.append((b, "version"))
    b = bytearray(good); b[8], b[11] = b[11], b[8]; cases.append((b, "endian"))
    b = bytearray(good); b[12] = 0; cases.append((b, "layer count"))
    b = bytearray(good); b[16 + 8] = 1; cases.append((b, "grid"))
    b = bytearray(good); b[16 + 32] = 0xFE; cases.append((b, "flags"))
    b = bytearray(good); b[16 + 36] = 1; cases.append((b, "reserved"))
    b = bytearray(good); b[16 + 40:16 + 48] = struct.pack("<d", float("nan")); cases.append((b, "scale"))
    b = bytearray(good); b[16 + 56:16 + 64] = struct.pack("<d", 0.0); cases.append((b, "log"))
    b = bytearray(good); b[16 + 16:16 + 24] = struct.pack("<d", float("nan")); cases.append((b, "domain"))
    b = bytearray(good); b[16 + 64:16 + 72] = struct.pack("<d", -1.0); cases.append((b, "bias scale"))
    b = bytearray(good); b[16 + 48:16 + 56] = struct.pack("<d", float("inf")); cases.append((b, "minimum"))
    b = bytearray(good); b[16 + 72 + 0] ^= 1; cases.append((b, "chain"))
    cases.append((bytearray(good[:200]), "section"))
    cases.append((bytearray(good[:2]), "magic"))
    cases.append((bytearray(good[:40]), "header"))
    for bad, frag in cases:
        _expect_same_fault(bytes(bad), frag)


@needs_ref
@pytest.mark.gpu
def test_truncation_after_index_sections_on_device():
    """A truncated last section: the index sections before it are range-checked
    on the device first (deserialize's order), then the truncation is raised."""
    _expect_same_fault(bytes(bytearray(_good_int8_bytes())[:-1]), "section")


@needs_ref
@pytest.mark.gpu
def test_out_of_range_index_names_the_edge():
    """test_lutham.cpp:254-275: byte 192 holds {0,1} at 2 bits; 0x0F makes edge 0 index 3 == K."""
    cl = synthetic.crafted_layer(1, 2, 2, 3, 10)
    cl.indices = np.array([0, 1], np.uint32)
    good = bytearray(oracle.ref_build(synthetic.CompressedNetwork([cl])).serialize())
    assert good[192] == 0x04
    good[192] = 0x0F
    _expect_same_fault(bytes(good), "edge 0")
    with pytest.raises(hq.FormatError) as e:
        hq.deserialize(bytes(good))
    assert e.value.fault == hq.FormatFault.IndexOutOfRange and e.value.offset == 192 and "K=3" in str(e.value)


def test_missing_file_is_value_error():
    with pytest.raises(hq.ValueError):
        hq.load_model("/nonexistent/missing.skan")
