"""Host-side table layer: shipped tables, both file formats, alias and packs."""
import json
import zlib

import numpy as np
import pytest

from helpers import hex_to_bits

from paper_1403_6870_b200 import tables as T
from paper_1403_6870_b200.errors import EmptyWeights, FormatError


@pytest.fixture(scope="module", params=[T.EXPONENTIAL, T.HALF_NORMAL])
def tab(request):
    return T.default_tables(request.param)


def test_lmax_and_tail_start():
    e, h = T.default_tables(T.EXPONENTIAL), T.default_tables(T.HALF_NORMAL)
    # reference tests/test_tables.py:22-24 and _packs.py:43,59
    assert (e.l_max, h.l_max) == (252, 253)
    assert e.x[1] == 7.569274694148063 and h.x[1] == 3.6360066255009458
    assert e.epsilon_max == 0.09258715630943215 and h.epsilon_max == 0.0
    assert e.i_max == h.i_max == 256


def test_geometry(tab):
    assert np.all(np.diff(tab.x) < 0.0) and np.all(np.diff(tab.f) > 0.0)
    assert tab.a.sum() == pytest.approx(1.0, abs=1e-12)
    assert np.array_equal(tab.scaled_x, tab.x * 2.0 ** -64)
    xl, xr, fb, ft = tab.box_bounds(tab.l_max)  # the cap
    assert xl == 0.0 and ft == 1.0
    with pytest.raises(IndexError):
        tab.box_bounds(0)


def test_binary_and_json_round_trip(tab, tmp_path):
    blob = T.to_binary(tab)
    assert T.from_binary(blob) == tab
    js = T.to_json_bytes(tab)
    assert T.from_json_bytes(js) == tab
    for fmt in ("json", "binary"):
        p = tmp_path / f"t.{fmt}"
        T.save(tab, p, fmt=fmt)
        assert T.load(p) == tab


def test_corruption_detected(tab):
    blob = bytearray(T.to_binary(tab))
    blob[40] ^= 1
    with pytest.raises(FormatError):
        T.from_binary(bytes(blob))
    with pytest.raises(FormatError):
        T.from_binary(b"NOPE" + bytes(blob[4:]))
    doc = json.loads(T.to_json_bytes(tab))
    doc["L_max"] += 1
    with pytest.raises(FormatError):
        T.from_json_bytes(json.dumps(doc).encode())
    with pytest.raises(FormatError):
        T.from_json_bytes(b"[1, 2]")
    with pytest.raises(FormatError):
        T.from_json_bytes(b"{not json")


def test_shipped_files_crc():
    from importlib import resources
    for kind in (T.EXPONENTIAL, T.HALF_NORMAL):
        blob = resources.files("paper_1403_6870_b200").joinpath(
            "data", f"{kind}_256.zigt").read_bytes()
        assert zlib.crc32(blob[:-4]).to_bytes(4, "little") == blob[-4:]


def test_alias_bit_identical_to_reference(golden):
    for kind in (T.EXPONENTIAL, T.HALF_NORMAL):
        a = T.build_alias(T.default_tables(kind).a)
        assert np.array_equal(a.prob.view(np.uint64),
                              hex_to_bits(golden[f"alias_{kind}_prob"]))
        assert a.alias.tolist() == golden[f"alias_{kind}_alias"]


def test_alias_exact_probabilities():
    rng = np.random.default_rng(3)
    for n in (1, 2, 7, 100, 254):
        w = rng.random(n)
        a = T.build_alias(w)
        np.testing.assert_allclose(a.exact_probabilities(), w / w.sum(), rtol=1e-12, atol=1e-15)
    with pytest.raises(EmptyWeights):
        T.build_alias([0.0, 0.0])
    with pytest.raises(ValueError):
        T.build_alias([1.0, -1.0])
    with pytest.raises(ValueError):
        T.build_alias([])


def test_packs_match_oracle(orc):
    hn, ex = orc.packs()
    for kind, op in ((T.EXPONENTIAL, ex), (T.HALF_NORMAL, hn)):
        p = T.make_pack(T.default_tables(kind))
        for name, oname in (("scale", "sx"), ("xlo", "xlo"), ("xw", "xw"), ("flo", "flo"),
                            ("fh", "fh"), ("prob", "prob"), ("alias", "alias")):
            assert np.array_equal(np.asarray(getattr(p, name)), getattr(op, oname)), (kind, name)
        assert p.tail_x == op.c.tailx and p.eps == op.c.eps and p.l_max == op.c.lmax


def test_unknown_kind():
    with pytest.raises(ValueError):
        T.default_tables("cauchy")
