"""Tuning-report persistence in the reference's CSV dialect (report.cpp:12-145)
plus a sidecar of the tuned B200 plans, so tuned launch geometries can be
reused across runs.

  <path>            exactly report.cpp's format: header
                    `k,t_trusted_ms,t_specialized_ms,speedup`, one line per K,
                    footers best_k / vlen / simd_bits / cores / description /
                    graph_id / skipped -- readable by the reference's own
                    load_report (tests check that through oracle/_ref).
                    The GPU profile maps onto the footers as: vlen = 32 (warp
                    lanes), simd_bits = 1024, cores = SM count,
                    description = device name.
  <path>.plans.csv  `k,lanes,vec,unroll,path_items,split_rows_over,k_tile,block,scalar,occupancy`
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

HEADER = "k,t_trusted_ms,t_specialized_ms,speedup"
PLAN_FIELDS = ("lanes", "vec", "unroll", "path_items", "split_rows_over", "k_tile", "block", "scalar",
               "occupancy")


from ._lib import IoError, ParseError  # noqa: E402  (error.hpp:40-55)


@dataclass
class LoadedEntry:
    k: int
    t_trusted_ms: float
    t_specialized_ms: float
    speedup: float


@dataclass
class LoadedReport:
    entries: list
    best_k: int
    profile: dict
    graph_id: str
    skipped: list
    plans: dict = field(default_factory=dict)  # K -> plan params


def _fmt(v: float) -> str:
    return f"{v:.9g}"  # report.cpp:14-18 ("%.9g")


def save_report(rep, path) -> None:
    """save_report (report.cpp:59-74) + the plans sidecar."""
    path = os.fspath(path)
    prof = getattr(rep, "profile", {}) or {}
    with open(path, "w") as f:
        f.write(HEADER + "\n")
        for e in rep.entries:
            f.write(f"{e.k},{_fmt(e.t_trusted_ms)},{_fmt(e.t_specialized_ms)},{_fmt(e.speedup)}\n")
        f.write(f"best_k,{rep.best_k}\n")
        f.write("vlen,32\n")
        f.write("simd_bits,1024\n")
        f.write(f"cores,{int(prof.get('sm_count', 0))}\n")
        f.write(f"description,{prof.get('description', 'cuda')}\n")
        f.write(f"graph_id,{rep.graph_id}\n")
        for k in rep.skipped:
            f.write(f"skipped,{k}\n")
    plans = getattr(rep, "plans", {}) or {}
    with open(path + ".plans.csv", "w") as f:
        f.write("k," + ",".join(PLAN_FIELDS) + "\n")
        for k in sorted(plans):
            p = plans[k].params if hasattr(plans[k], "params") else plans[k]
            f.write(f"{k}," + ",".join(str(int(p[name])) for name in PLAN_FIELDS) + "\n")


def load_report(path) -> LoadedReport:
    """load_report (report.cpp:76-145) with the same validation and messages."""
    path = os.fspath(path)
    try:
        lines = open(path).read().split("\n")
    except OSError as ex:
        raise IoError(f"cannot open '{path}'") from ex
    if not lines or lines[0] == "" and len(lines) == 1:
        raise ParseError("empty report file", 1)
    if lines[0] != HEADER:
        raise ParseError(f"expected header '{HEADER}'", 1)
    rep = LoadedReport([], 0, {"vlen": 8, "simd_bits": 256, "cores": 1, "description": "fallback"}, "", [])
    saw_best, saw_vlen = False, False

    def u32(s):
        if not s.isdigit() or int(s) > 0xFFFFFFFF:
            raise ValueError
        return int(s)

    n = 1
    for n, line in enumerate(lines[1:], start=2):
        if not line:
            continue
        fields = line.split(",")
        key = fields[0]
        try:
            if key == "best_k":
                if len(fields) != 2:
                    raise ValueError
                rep.best_k, saw_best = u32(fields[1]), True
            elif key == "vlen":
                if len(fields) != 2:
                    raise ValueError
                rep.profile["vlen"] = u32(fields[1])
                rep.profile["simd_bits"] = rep.profile["vlen"] * 32
                saw_vlen = True
            elif key in ("simd_bits", "cores"):
                if len(fields) != 2:
                    raise ValueError
                rep.profile[key] = u32(fields[1])
            elif key == "description":
                rep.profile["description"] = line[len(key) + 1:]
            elif key == "graph_id":
                rep.graph_id = line[len(key) + 1:]
            elif key == "skipped":
                if len(fields) != 2:
                    raise ValueError
                rep.skipped.append(u32(fields[1]))
            else:
                if len(fields) != 4:
                    raise ParseError(f"malformed data line '{line}'", n)
                e = LoadedEntry(u32(fields[0]), float(fields[1]), float(fields[2]), float(fields[3]))
                if e.t_trusted_ms <= 0 or e.t_specialized_ms <= 0 or e.speedup <= 0:
                    raise ParseError("times and speedup must be positive", n)
                rep.entries.append(e)
        except ParseError:
            raise
        except ValueError:
            raise ParseError(f"malformed {key} footer" if key in ("best_k", "vlen", "simd_bits", "cores", "skipped")
                             else f"malformed data line '{line}'", n) from None
    if not rep.entries:
        raise ParseError("report has no data lines", n + 1)
    if not saw_best:
        raise ParseError("missing best_k footer", n + 1)
    if not saw_vlen:
        raise ParseError("missing vlen footer", n + 1)
    if not any(e.k == rep.best_k for e in rep.entries):
        raise ParseError("best_k does not match any data line", n + 1)
    side = path + ".plans.csv"
    if os.path.exists(side):
        rows = open(side).read().strip().split("\n")
        for row in rows[1:]:
            if row:
                vals = [int(t) for t in row.split(",")]
                rep.plans[vals[0]] = dict(zip(PLAN_FIELDS, vals[1:]))
    return rep
