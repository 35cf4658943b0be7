"""The C-ABI library: loads without a GPU, exports every declared symbol, and
rejects bad arguments with the documented status codes (no device work)."""
import ctypes as C
import pathlib
import re

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "zigfast_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(zf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("zf_fill", "zf_fill_replay", "zf_fill_gid", "zf_tables_create", "zf_words",
                 "zf_stats", "zf_fill_stats", "zf_fill_batch", "zf_xoshiro_jump"):
        assert must in names


def test_library_exports_every_declared_symbol(built_lib):
    for name in declared_functions():
        assert hasattr(built_lib, name), f"missing export {name}"
    from paper_1403_6870_b200 import _lib
    assert set(_lib.EXPORTS) <= set(declared_functions())


def test_abi_version_and_strerror(built_lib):
    assert built_lib.zf_abi_version() == 1
    for code in (0, -1, -2, -3, -4, -5, -6, -7):
        assert built_lib.zf_strerror(code)
    assert b"invalid" in built_lib.zf_strerror(-1)


def test_invalid_arguments_rejected_without_device(built_lib):
    L = built_lib
    # null handle / null pointers: rejected before any CUDA call
    assert L.zf_fill(None, 0, 0, 1, 0, None, 10, None, None) == -1
    assert L.zf_fill_gid(None, 0, 0, 0, None, None, 0, None, 1, None, None, None) == -1
    assert L.zf_tables_create(None, None, 0, C.byref(C.c_void_p())) == -1
    assert L.zf_words(0, None, 0, None, None) == -1
    assert L.zf_xoshiro_jump(None, 5) == -1
    assert L.zf_tables_destroy(None) == 0


def test_table_pack_validation(built_lib):
    from paper_1403_6870_b200 import _lib, tables
    t = tables.default_tables(tables.EXPONENTIAL)
    dt = object.__new__(_lib.DeviceTables)
    dt._keep = []
    good = dt._cpack(tables.make_pack(t))
    bad = dt._cpack(tables.make_pack(t))
    bad.nslots = bad.lmax  # inconsistent slot count
    assert built_lib.zf_tables_create(C.byref(bad), C.byref(good), 0,
                                      C.byref(C.c_void_p())) == -6


def test_xoshiro_jump_matches_stepping(built_lib, orc):
    from paper_1403_6870_b200 import _lib
    for seed, k in ((1, 1), (42, 37), (7, 511), (7, 512), (123, 10_007), (42, 1_000_000)):
        st = orc.xoshiro_state(seed)
        _lib.check(built_lib.zf_xoshiro_jump(_lib.u64p(st), k))
        ref = orc.xoshiro_state(seed)
        out = np.empty(k, dtype=np.uint64)
        orc.lib().orc_words(orc.SRC_XOSHIRO, orc._u64p(ref), k, orc._u64p(out))
        assert np.array_equal(st, ref), (seed, k)


def test_xoshiro_jump_composes_for_large_distances(built_lib, orc):
    """Jumps by distances far beyond stepping reach (the high bits of k go
    through the precomputed x^(2^i) powers): jump(a) then jump(b) == jump(a + b)."""
    from paper_1403_6870_b200 import _lib
    for a, b in ((2**40 + 3, 2**33 + 7), (2**63 - 1, 2**62 + 12345), (999_983, 2**50)):
        s1 = orc.xoshiro_state(9)
        _lib.check(built_lib.zf_xoshiro_jump(_lib.u64p(s1), a))
        _lib.check(built_lib.zf_xoshiro_jump(_lib.u64p(s1), b))
        s2 = orc.xoshiro_state(9)
        _lib.check(built_lib.zf_xoshiro_jump(_lib.u64p(s2), a + b))
        assert np.array_equal(s1, s2), (a, b)


def test_published_jump_polynomial(built_lib):
    """x^(2^128) mod P is xoshiro256's published jump() constant: the
    characteristic polynomial recovered by Berlekamp-Massey is right."""
    out = np.zeros(4, dtype=np.uint64)
    from paper_1403_6870_b200 import _lib
    _lib.check(built_lib.zf_xoshiro_pow2_poly(128, _lib.u64p(out)))
    assert [int(x) for x in out] == [0x180EC6D33CFD0ABA, 0xD5A61266F0C9392C,
                                     0xA9582618E03FC9AA, 0x39ABDC4529B1661C]
    _lib.check(built_lib.zf_xoshiro_pow2_poly(192, _lib.u64p(out)))  # long_jump()
    assert [int(x) for x in out] == [0x76E15D3EFEFDCBBF, 0xC5004E441C522FB3,
                                     0x77710069854EE241, 0x39109BB02ACBE635]


def test_no_cpu_fallback(monkeypatch, tmp_path):
    """Without the built library the product raises instead of falling back."""
    import importlib

    from paper_1403_6870_b200 import _lib, errors
    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "missing.so")
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(errors.ExtensionMissing):
        _lib.lib()
    importlib.reload(_lib)
