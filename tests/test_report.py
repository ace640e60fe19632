"""Report persistence (report.cpp dialect): files written here load in the
reference's own load_report (oracle/_ref), and malformed files fail the same
way (ParseError with a line number)."""
import ctypes as C
from dataclasses import dataclass

import pytest

from paper_2403_14853_b200 import report


@dataclass
class E:
    k: int
    t_trusted_ms: float
    t_specialized_ms: float
    speedup: float


@dataclass
class R:
    entries: list
    best_k: int
    profile: dict
    graph_id: str
    skipped: list
    plans: dict


def _rep():
    plans = {32: {"lanes": 8, "vec": 1, "unroll": 8, "path_items": 64, "split_rows_over": 256, "k_tile": 32,
                  "block": 128, "scalar": 0, "occupancy": 5}}
    return R([E(16, 0.5, 0.25, 2.0), E(32, 0.9, 0.3, 3.0)], 32, {"sm_count": 148, "description": "NVIDIA B200"},
             "rmat18", [48], plans)


def test_roundtrip(tmp_path):
    p = tmp_path / "rep.csv"
    report.save_report(_rep(), p)
    back = report.load_report(p)
    assert back.best_k == 32 and back.graph_id == "rmat18" and back.skipped == [48]
    assert [(e.k, e.t_trusted_ms, e.t_specialized_ms, e.speedup) for e in back.entries] == [(16, 0.5, 0.25, 2.0), (32, 0.9, 0.3, 3.0)]
    assert back.profile["cores"] == 148 and back.profile["description"] == "NVIDIA B200"
    assert back.plans[32]["occupancy"] == 5


def test_reference_loader_reads_our_file(tmp_path):
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    p = tmp_path / "rep.csv"
    report.save_report(_rep(), p)
    L = ref.lib()
    L.ref_load_report.argtypes = [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
    bk, ne, ns = C.c_uint32(), C.c_uint32(), C.c_uint32()
    assert L.ref_load_report(str(p).encode(), C.byref(bk), C.byref(ne), C.byref(ns)) == 0
    assert (bk.value, ne.value, ns.value) == (32, 2, 1)
    # and a malformed one is a ParseError in both loaders
    bad = tmp_path / "bad.csv"
    bad.write_text("k,t_trusted_ms,t_specialized_ms,speedup\n32,1,1,1\nvlen,8\n")
    assert L.ref_load_report(str(bad).encode(), C.byref(bk), C.byref(ne), C.byref(ns)) == 6
    with pytest.raises(report.ParseError, match="missing best_k"):
        report.load_report(bad)


@pytest.mark.parametrize("text,msg", [
    ("", "empty report file"),
    ("k,t,s\n16,1,1,1\n", "expected header"),
    ("k,t_trusted_ms,t_specialized_ms,speedup\nbest_k,32\nvlen,8\n", "no data lines"),
    ("k,t_trusted_ms,t_specialized_ms,speedup\n16,1,1,1\nbest_k,32\nvlen,8\n", "best_k does not match"),
    ("k,t_trusted_ms,t_specialized_ms,speedup\n16,1,-1,1\nbest_k,16\nvlen,8\n", "positive"),
    ("k,t_trusted_ms,t_specialized_ms,speedup\n16,1,1,1\nbest_k,x\nvlen,8\n", "malformed best_k"),
])
def test_parse_errors(tmp_path, text, msg):
    p = tmp_path / "r.csv"
    p.write_text(text)
    with pytest.raises(report.ParseError, match=msg):
        report.load_report(p)
