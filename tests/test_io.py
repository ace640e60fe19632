"""On-disk formats (io.hpp:80-262): the native loaders in
csrc/host/mtx.cpp against the reference's own load_mtx / save_mtx /
load_features / load_labels / load_mask (oracle/_ref): identical CSR bits on
success, identical exception class, message and line number on failure --
including the multi-threaded chunked parse on files larger than one chunk."""
import os

import numpy as np
import pytest

from oracle import ref
from paper_2403_14853_b200 import graph_io
from paper_2403_14853_b200._lib import ConfigError, IoError, ParseError

needs_ref = pytest.mark.skipif(not ref.available("O2"), reason="oracle/_ref not built")

MTX_CASES = {
    "general_real": "%%MatrixMarket matrix coordinate real general\n% comment\n3 4 4\n1 1 1.5\n3 4 -2\n2 2 0.25\n1 3 7\n",
    "integer": "%%MatrixMarket matrix coordinate integer general\n2 2 2\n1 2 3\n2 1 -4\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n3 3 3\n3 1\n1 2\n2 3\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n4 4 4\n1 1 2\n3 1 0.5\n4 2 -1\n4 4 3\n",
    "upper_banner": "%%MATRIXMARKET MATRIX COORDINATE REAL GENERAL\n2 2 1\n2 2 9\n",
    "no_symmetry_token": "%%MatrixMarket matrix coordinate real\n2 2 1\n1 2 1\n",
    "blank_and_comments": "%%MatrixMarket matrix coordinate real general\n\n%c\n\n2 3 2\n\n% mid\n1 3 1e-3\n\n2 1 +4.5\n% tail\n",
    "crlf": "%%MatrixMarket matrix coordinate real general\r\n2 2 2\r\n1 1 1\r\n2 2 2\r\n",
    "duplicates": "%%MatrixMarket matrix coordinate real general\n2 2 4\n1 1 1\n1 1 2\n2 1 0.5\n1 1 4\n",
    "no_trailing_newline": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 2 2",
    "empty_matrix": "%%MatrixMarket matrix coordinate real general\n5 7 0\n",
    "zero_dims": "%%MatrixMarket matrix coordinate real general\n0 0 0\n",
    "garbage_after_entries": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\nthis is ignored\n9 9 9\n",
    "special_values": "%%MatrixMarket matrix coordinate real general\n1 4 4\n1 1 inf\n1 2 -INF\n1 3 0x1p-3\n1 4 1e39\n",
    "tabs": "%%MatrixMarket matrix coordinate real general\n2\t2\t1\n 2\t 1  \t3.25 \n",
    "symmetric_pattern_diag": "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n1 1\n2 1\n3 3\n",
    # errors
    "empty_file": "",
    "not_banner": "hello world\n1 1 1\n",
    "short_banner": "%%MatrixMarket matrix coordinate\n1 1 0\n",
    "array_format": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "complex_field": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "missing_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n3 3\n",
    "negative_size": "%%MatrixMarket matrix coordinate real general\n3 -3 1\n",
    "float_size": "%%MatrixMarket matrix coordinate real general\n3 3.0 1\n",
    "blank_ws_line": "%%MatrixMarket matrix coordinate real general\n2 2 1\n   \n1 1 1\n",
    "too_few_entries": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1\n2 2 2\n",
    "malformed_entry": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n2 x 2\n",
    "pattern_with_value": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 1 1\n",
    "missing_value": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1\n",
    "out_of_range_row": "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n4 1 1\n",
    "zero_index": "%%MatrixMarket matrix coordinate real general\n3 3 1\n0 1 1\n",
    "value_overflow": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 1e400\n",
    "value_underflow": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 1e-400\n",
    "index_overflow": "%%MatrixMarket matrix coordinate real general\n3 3 1\n99999999999999999999 1 1\n",
    "crlf_blank_line": "%%MatrixMarket matrix coordinate real general\r\n2 2 1\r\n\r\n1 1 1\r\n",
}


def _ours(fn, *a):
    try:
        return ("ok", fn(*a))
    except ParseError as e:
        return ("parse", str(e), e.line)
    except IoError as e:
        return ("io", str(e))


def _theirs(fn, *a):
    try:
        return ("ok", fn(*a))
    except ref.RefError as e:
        return ({6: "parse", 5: "io"}.get(e.status, e.status), e.what) + ((e.line,) if e.status == 6 else ())


def _same_csr(a, b):
    m, n, rp, ci, v = b
    assert (a.n_rows, a.n_cols) == (m, n)
    np.testing.assert_array_equal(a.row_ptr, rp)
    np.testing.assert_array_equal(a.col_idx, ci)
    np.testing.assert_array_equal(a.values.view(np.uint32), v.view(np.uint32))


def _compare_mtx(path, threads=0):
    ours = _ours(graph_io.load_mtx, path, threads)
    theirs = _theirs(ref.load_mtx, path)
    assert ours[0] == theirs[0], (ours, theirs)
    if ours[0] == "ok":
        _same_csr(ours[1], theirs[1])
    else:
        assert ours[1:] == theirs[1:]
    return ours


@needs_ref
@pytest.mark.parametrize("name", sorted(MTX_CASES))
def test_mtx_cases_match_reference(tmp_path, name):
    p = tmp_path / f"{name}.mtx"
    p.write_bytes(MTX_CASES[name].encode())
    _compare_mtx(str(p))


def test_mtx_known_answers(tmp_path):
    """SPEC-style known answers, independent of oracle/_ref."""
    p = tmp_path / "a.mtx"
    p.write_text(MTX_CASES["symmetric"])
    a = graph_io.load_mtx(str(p))
    assert (a.n_rows, a.n_cols, a.nnz) == (4, 4, 6)
    np.testing.assert_array_equal(a.row_ptr, [0, 2, 3, 4, 6])
    np.testing.assert_array_equal(a.col_idx, [0, 2, 3, 0, 1, 3])
    np.testing.assert_array_equal(a.values, np.float32([2, 0.5, -1, 0.5, -1, 3]))
    p.write_text(MTX_CASES["duplicates"])
    a = graph_io.load_mtx(str(p))
    np.testing.assert_array_equal(a.values, np.float32([7, 0.5]))
    p.write_text(MTX_CASES["malformed_entry"])
    with pytest.raises(ParseError, match=r"^line 4: malformed entry '2 x 2'$") as ei:
        graph_io.load_mtx(str(p))
    assert ei.value.line == 4
    with pytest.raises(IoError, match="cannot open"):
        graph_io.load_mtx(str(tmp_path / "missing.mtx"))


def _big_mtx(rng, n, nnz, symmetric=False, comments=True):
    rows = rng.integers(1, n + 1, nnz)
    cols = rng.integers(1, n + 1, nnz)
    vals = rng.standard_normal(nnz).astype(np.float32)
    lines = [f"%%MatrixMarket matrix coordinate real {'symmetric' if symmetric else 'general'}",
             f"{n} {n} {nnz}"]
    for i in range(nnz):
        if comments and i % 997 == 0:
            lines.append("% interleaved comment")
        if comments and i % 1499 == 0:
            lines.append("")
        lines.append(f"{rows[i]} {cols[i]} {float(vals[i])!r}")
    return lines


@needs_ref
@pytest.mark.parametrize("symmetric", [False, True])
def test_mtx_large_multichunk_matches_reference(tmp_path, symmetric):
    rng = np.random.default_rng(11)
    lines = _big_mtx(rng, 5000, 150_000, symmetric)  # ~3.5 MB: several parse chunks
    p = tmp_path / "big.mtx"
    p.write_text("\n".join(lines) + "\n")
    for threads in (1, 3, 8):
        _compare_mtx(str(p), threads)


@needs_ref
def test_mtx_errors_in_late_chunks(tmp_path):
    rng = np.random.default_rng(12)
    lines = _big_mtx(rng, 3000, 120_000, comments=False)
    base = "\n".join(lines) + "\n"
    p = tmp_path / "e.mtx"
    # a malformed entry deep in the file
    bad = lines.copy()
    bad[100_000] = "12 oops 1"
    p.write_text("\n".join(bad) + "\n")
    ours = _compare_mtx(str(p), 8)
    assert ours[0] == "parse" and ours[2] == 100_001
    # garbage beyond the declared entry count is never read
    p.write_text(base + "garbage line\n" * 50_000)
    assert _compare_mtx(str(p), 8)[0] == "ok"
    # fewer entries than declared (count on a late line)
    p.write_text("\n".join(lines[:-10]) + "\n")
    ours = _compare_mtx(str(p), 8)
    assert ours[0] == "parse" and "expected 120000 entries, found 119990" in ours[1]
    # an out-of-range entry in the last chunk
    bad = lines.copy()
    bad[-1] = "3001 1 1"
    p.write_text("\n".join(bad))
    assert _compare_mtx(str(p), 8)[0] == "parse"


@needs_ref
def test_save_mtx_matches_reference_bytes_and_round_trips(tmp_path):
    rng = np.random.default_rng(5)
    m, n = 700, 300
    rp = np.zeros(m + 1, np.uint64)
    rows = []
    for i in range(m):
        k = int(rng.integers(0, 9))
        rows.append(np.sort(rng.choice(n, k, replace=False)).astype(np.uint32))
        rp[i + 1] = rp[i] + k
    ci = np.concatenate(rows)
    v = (rng.standard_normal(len(ci)) * 10.0 ** rng.integers(-30, 30, len(ci))).astype(np.float32)
    v[:3] = [np.float32(1) / 3, -0.0, 1e-45]
    ours, theirs = tmp_path / "o.mtx", tmp_path / "t.mtx"
    graph_io.save_mtx((m, n, rp, ci, v), str(ours), threads=4)
    ref.save_mtx(str(theirs), m, n, rp, ci, v)
    assert ours.read_bytes() == theirs.read_bytes()
    back = graph_io.load_mtx(str(ours))
    np.testing.assert_array_equal(back.row_ptr, rp)
    np.testing.assert_array_equal(back.col_idx, ci)
    np.testing.assert_array_equal(back.values.view(np.uint32), v.view(np.uint32))
    with pytest.raises(IoError, match="for writing"):
        graph_io.save_mtx((m, n, rp, ci, v), str(tmp_path / "no" / "dir.mtx"))
    with pytest.raises(ConfigError):
        graph_io.save_mtx((m, n, rp, ci[:-1], v), str(ours))


FEATURE_CASES = {
    "ok": "2 3\n1 2 3\n-1.5 0 1e-3\n",
    "blank_lines": "2 2\n\n1 2\n\n3 4\nextra ignored\n",
    "zero": "0 4\n",
    "empty": "",
    "bad_header": "2\n1 2\n",
    "neg_header": "-1 2\n",
    "short_row": "2 3\n1 2 3\n1 2\n",
    "non_numeric": "1 2\n1 abc\n",
    "missing_rows": "3 1\n1\n2\n",
    "ws_only_line": "1 1\n  \n",
}


@needs_ref
@pytest.mark.parametrize("name", sorted(FEATURE_CASES))
def test_features_match_reference(tmp_path, name):
    p = tmp_path / "f.txt"
    p.write_text(FEATURE_CASES[name])
    ours = _ours(graph_io.load_features, str(p))
    theirs = _theirs(ref.load_features, str(p))
    assert ours[0] == theirs[0], (ours, theirs)
    if ours[0] == "ok":
        np.testing.assert_array_equal(ours[1].view(np.uint32), theirs[1].view(np.uint32))
    else:
        assert ours[1:] == theirs[1:]


@needs_ref
def test_features_large_matches_reference(tmp_path):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((20000, 24)).astype(np.float32)
    p = tmp_path / "x.txt"
    with open(p, "w") as f:
        f.write("20000 24\n")
        for i, row in enumerate(x):
            if i % 777 == 0:
                f.write("\n")
            f.write(" ".join(repr(float(t)) for t in row) + "\n")
    ours = graph_io.load_features(str(p), threads=8)
    np.testing.assert_array_equal(ours.view(np.uint32), ref.load_features(str(p)).view(np.uint32))
    np.testing.assert_array_equal(ours, x)


INT_CASES = {
    "ok": "4\n0 1\n2\n\n3\n",
    "neg_label": "3\n0 -1 2\n",
    "mask_two": "3\n0 2 1\n",
    "too_many": "2\n1 1 1\n",
    "too_few": "3\n1\n",
    "non_int": "2\n1 x\n",
    "bad_header": "2 3\n1 1\n",
    "empty": "",
}


@needs_ref
@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("name", sorted(INT_CASES))
def test_labels_and_mask_match_reference(tmp_path, kind, name):
    p = tmp_path / "l.txt"
    p.write_text(INT_CASES[name])
    fn = graph_io.load_labels if kind == 0 else graph_io.load_mask
    ours = _ours(fn, str(p))
    theirs = _theirs(ref.load_int_column, str(p), kind)
    assert ours[0] == theirs[0], (ours, theirs)
    if ours[0] == "ok":
        np.testing.assert_array_equal(ours[1].astype(np.uint32), theirs[1])
    else:
        assert ours[1:] == theirs[1:]


def test_io_error_for_missing_files(tmp_path):
    missing = str(tmp_path / "nope")
    for fn in (graph_io.load_mtx, graph_io.load_features, graph_io.load_labels, graph_io.load_mask):
        with pytest.raises(IoError, match=f"cannot open '{missing}'"):
            fn(missing)


@pytest.mark.gpu
def test_mtx_to_device_spmm_matches_reference(cuda, tmp_path):
    """Ingest -> device CSR -> B200 SpMM, against the reference's SpMM on the
    reference's own load of the same file."""
    import torch

    from paper_2403_14853_b200 import ops
    rng = np.random.default_rng(21)
    lines = _big_mtx(rng, 4000, 60_000, symmetric=True)
    p = tmp_path / "g.mtx"
    p.write_text("\n".join(lines) + "\n")
    a = graph_io.load_mtx(str(p), device="cuda")
    x = rng.standard_normal((4000, 64)).astype(np.float32)
    got = ops.spmm(a, torch.from_numpy(x).cuda(), "sum").cpu().numpy()
    if ref.available("O2"):
        m, n, rp, ci, v = ref.load_mtx(str(p))
        want = ref.spmm_f32(rp, ci, v, x, n, 0)
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    assert os.path.exists(p)
