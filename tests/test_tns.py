"""CPU: the parallel .tns reader/writer (csrc/tns.cpp) against the reference's
read_tns/write_tns (tns_io.cpp:41-142): same tensors, same line-numbered
diagnostics.  Host-only entry points of libntcb.so, no device needed."""
import os

import numpy as np
import pytest

import oracle as O
from paper_2109_09534_b200.ntc import parse_tns


def write(path, text):
    with open(path, "w") as f:
        f.write(text)
    return str(path)


def canon(orc, dims, idx, vals):
    return orc.canonicalize(dims, idx, vals)


def check_same(orc, path):
    dims, idx, vals = parse_tns(path)
    ci, cv = canon(orc, dims, idx, vals)
    if O.ref_available():
        rp = O.ref_read_tns(path)
        assert [int(d) for d in rp.dims] == dims
        ri, rv = rp.tensor()
        np.testing.assert_array_equal(ri, ci)
        np.testing.assert_array_equal(rv, cv)
    return dims, ci, cv


def test_header_comments_and_inferred_dims(tmp_path, orc):
    text = ("# a comment\n# dims: 8 6 4\n\n1 1 3 0.81204054259487735\n"
            "  2 3 1 0.5   # trailing comment\n8 6 4 1e-3\n\t3 2 2 7\n")
    dims, ci, cv = check_same(orc, write(tmp_path / "a.tns", text))
    assert dims == [8, 6, 4] and len(cv) == 4
    dims, ci, cv = check_same(orc, write(tmp_path / "b.tns", "1 2 0.5\n3 1 2.5\n2 5 1\n"))
    assert dims == [3, 5]


@pytest.mark.parametrize("text,msg", [
    ("1 2 0.5\n1 x 0.5\n", ":2: bad index 'x'"),
    ("1 2 0.5\n0 1 0.5\n", ":2: indices are 1-based; got 0"),
    ("1 2 0.5\n1 1 abc\n", ":2: bad value 'abc'"),
    ("1 2 0.5\n1 1 -1\n", ":2: negative value"),
    ("1 2 0.5\n1 1 nan\n", ":2: non-finite value"),
    ("1 2 0.5\n1 1 1 0.5\n", ":2: expected 3 fields, got 4"),
    ("1 0.5\n", ":1: expected at least 2 indices and a value"),
    ("# dims: 2 2\n3 1 0.5\n", ":2: index 3 exceeds declared dimension 2"),
    ("1 2 0.5\n# dims: 4 4 4\n", ":2: dims header order disagrees with entries"),
    ("# dims: 4 x\n", ":1: bad dims header"),
    ("# dims: 4 0\n", ":1: non-positive dimension in dims header"),
    ("# dims: 4\n", ":1: dims header needs at least 2 dimensions"),
    ("1 2 0.5\n1 2 0.5\n", "SparseTensor: duplicate index (1,2)"),
])
def test_diagnostics_match_reference(tmp_path, text, msg):
    path = write(tmp_path / "e.tns", text)
    if "duplicate" in msg:
        dims, idx, vals = parse_tns(path)  # duplicates are the tensor's error, not the parser's
        with pytest.raises(ValueError, match=r"duplicate index \(1,2\)"):
            O.Oracle().canonicalize(dims, idx, vals)
    else:
        with pytest.raises(RuntimeError) as e:
            parse_tns(path)
        assert str(e.value) == path + msg
    if O.ref_available():
        with pytest.raises(Exception) as e2:
            O.ref_read_tns(path)
        assert msg in str(e2.value)


def test_empty_file_rules(tmp_path):
    with pytest.raises(RuntimeError, match="has no entries and no dims header"):
        parse_tns(write(tmp_path / "z.tns", "# just a comment\n"))
    dims, idx, vals = parse_tns(write(tmp_path / "h.tns", "# dims: 3 4\n"))
    assert dims == [3, 4] and len(vals) == 0
    with pytest.raises(RuntimeError, match="cannot open"):
        parse_tns(str(tmp_path / "missing.tns"))


def test_large_file_parallel_chunks_and_round_trip(tmp_path, orc):
    rng = np.random.default_rng(3)
    dims = [300, 200, 100]
    nnz = 200_000
    cells = rng.choice(int(np.prod(dims)), nnz, replace=False)
    idx = np.stack(np.unravel_index(cells, dims), 1).astype(np.uint32)
    vals = rng.random(nnz)
    lines = ["# dims: 300 200 100"] + [
        f"{a + 1} {b + 1} {c + 1} {v!r}" + ("  # c" if k % 97 == 0 else "")
        for k, ((a, b, c), v) in enumerate(zip(idx.tolist(), vals.tolist()))]
    path = write(tmp_path / "big.tns", "\n".join(lines) + "\n")
    assert os.path.getsize(path) > (1 << 20)  # > 1 MiB: the multi-threaded path
    d, i2, v2 = parse_tns(path)
    assert d == dims
    np.testing.assert_array_equal(i2, idx)   # file order preserved
    np.testing.assert_array_equal(v2, vals)  # from_chars: exact round trip
    # an error deep inside a later chunk is reported with its global line number
    bad = lines[:]
    bad[150_001] = "1 1"
    pbad = write(tmp_path / "bad.tns", "\n".join(bad) + "\n")
    with pytest.raises(RuntimeError) as e:
        parse_tns(pbad)
    assert str(e.value) == pbad + ":150002: expected 4 fields, got 2"
    if O.ref_available():
        check_same(orc, path)
