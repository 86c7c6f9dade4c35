"""File formats: CMFR cache and text COO, byte-compatible with the
reference (data.py:142-202, :305-345).  Pinned by tests/golden/io_cases.npz,
which holds the bytes the reference itself wrote (make_golden.py io)."""

import io
import os

import numpy as np
import pytest

import paper_1808_03843_b200 as cmfb
from paper_1808_03843_b200.errors import DataError, FormatError, ParseError

GOLD = os.path.join(os.path.dirname(__file__), "golden", "io_cases.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(GOLD)


def _write(tmp_path, name, data: bytes):
    p = tmp_path / name
    p.write_bytes(data)
    return str(p)


def test_cache_roundtrip_bytes(g, tmp_path):
    ref = g["cache_bytes"].tobytes()
    sr = cmfb.load_cache(_write(tmp_path, "ref.cmfr", ref))
    m, n = (int(x) for x in g["dims"])
    assert (sr.m, sr.n) == (m, n)
    assert sr.nnz == int(sr.row_ptr[-1]) == int(sr.col_ptr[-1])
    assert sr.row_ptr.dtype == np.int64 and sr.col_idx.dtype == np.int32 and sr.csr_val.dtype == np.float32
    out = str(tmp_path / "ours.cmfr")
    cmfb.save_cache(out, sr)
    assert open(out, "rb").read() == ref


def test_cache_content_matches_triples(g, tmp_path):
    sr = cmfb.load_cache(_write(tmp_path, "ref.cmfr", g["cache_bytes"].tobytes()))
    # last duplicate wins (data.py:205-249): rebuild the cell map from the triples
    cells = {}
    for u, v, r in zip(g["u"], g["v"], g["r"]):
        cells[(int(u), int(v))] = np.float32(r)
    assert sr.nnz == len(cells)
    t = sr.to_triples()
    got = {(int(u), int(v)): np.float32(r) for u, v, r in zip(t.user, t.item, t.rating)}
    assert got == cells
    # CSC holds the same cells, ordered by (item, user)
    items = np.repeat(np.arange(sr.n), np.diff(sr.col_ptr))
    keys = items * sr.m + sr.row_idx
    assert np.all(np.diff(keys) > 0)
    assert {(int(u), int(v)): np.float32(r) for u, v, r in zip(sr.row_idx, items, sr.csc_val)} == cells


@pytest.mark.parametrize("fmt", ["tsv", "csv"])
def test_save_coo_bytes(g, tmp_path, fmt):
    t = cmfb.Triples(g["u"], g["v"], g["r"])
    out = str(tmp_path / ("x." + fmt))
    cmfb.save_coo(out, t, fmt=fmt)
    assert open(out, "rb").read() == g[fmt + "_bytes"].tobytes()
    back, m, n = cmfb.load_coo(out, fmt=fmt)
    np.testing.assert_array_equal(back.user, g["u"])
    np.testing.assert_array_equal(back.item, g["v"])
    np.testing.assert_array_equal(back.rating, g["r"])  # %.9g round-trips float32
    assert (m, n) == (int(g["u"].max()) + 1, int(g["v"].max()) + 1)


def test_parse_coo_matches_reference(g):
    text = g["parse_text"].tobytes().decode()
    t, m, n = cmfb.parse_coo(io.StringIO(text), fmt="tsv")
    np.testing.assert_array_equal(t.user, g["parse_u"])
    np.testing.assert_array_equal(t.item, g["parse_v"])
    np.testing.assert_array_equal(t.rating, g["parse_r"])
    assert [m, n] == list(g["parse_dims"])
    t2, m2, n2 = cmfb.parse_coo(text.splitlines(), fmt="tsv", m=100, n=50)
    assert (m2, n2) == (100, 50) and len(t2) == len(t)


@pytest.mark.parametrize("line,frag", [
    ("1\t2", "expected 3 fields"),
    ("1\t2\t3\t4", "expected 3 fields"),
    ("a\t2\t3", "invalid literal"),
    ("1\t2\tnan", "non-finite"),
    ("1\t2\tinf", "non-finite"),
    ("-1\t2\t3", "negative index"),
])
def test_parse_errors_name_the_line(line, frag):
    with pytest.raises(ParseError) as ei:
        cmfb.parse_coo(["# c\n", "0\t0\t1\n", line + "\n"], fmt="tsv")
    assert ei.value.line_no == 3 and frag in str(ei.value)


def test_parse_empty_and_bad_format():
    t, m, n = cmfb.parse_coo(["# only a comment\n", "\n"])
    assert len(t) == 0 and (m, n) == (0, 0)
    with pytest.raises(DataError):
        cmfb.parse_coo([], fmt="json")
    with pytest.raises(DataError):
        cmfb.save_coo("/nonexistent/x", cmfb.Triples(np.zeros(0, np.int64), np.zeros(0, np.int64),
                                                     np.zeros(0, np.float32)), fmt="json")


def test_cache_errors(g, tmp_path):
    ref = g["cache_bytes"].tobytes()
    cases = {
        "magic": b"XXXX" + ref[4:],
        "header": ref[:10],
        "version": ref[:4] + (2).to_bytes(4, "little") + ref[8:],
        "payload": ref[:-3],
        "trailing": ref + b"\0",
    }
    msgs = {"magic": "bad magic", "header": "truncated header", "version": "unsupported cache version",
            "payload": "truncated payload", "trailing": "trailing bytes"}
    for k, data in cases.items():
        with pytest.raises(FormatError, match=msgs[k]):
            cmfb.load_cache(_write(tmp_path, k + ".cmfr", data))
