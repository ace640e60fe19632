"""Summarise ncu output for profiles/: a --set full capture (.ncu-rep) and/or
a launch list (--metrics gpu__time_duration.sum --csv log).

  python scripts/ncu_summary.py --rep gpurun_out/prof.ncu-rep --out profiles/r01_x.json
  python scripts/ncu_summary.py --launches gpurun_out/launches.csv --out profiles/r01_launches.json
"""
import argparse
import collections
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__cycles_elapsed.avg",
    "launch__occupancy_limit_registers",
]

SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "usecond": 1e-3, "msecond": 1.0,
         "nsecond": 1e-6, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0}


def num(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    if unit in SCALE:
        x *= SCALE[unit]
    return x


def rep_summary(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[2:]:
        d = {"kernel": r[idx["Kernel Name"]]}
        for k in KEYS:
            if k in idx:
                u = units[idx[k]]
                key = k + (" [ms]" if "duration" in k else " [bytes]" if "bytes" in k else "")
                d[key] = num(r[idx[k]], u)
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        d["top_stalls_per_issue"] = {n: round(v, 3) for v, n in sorted(stalls, reverse=True)[:6]}
        rb = d.get("dram__bytes_read.sum [bytes]", 0) or 0
        wb = d.get("dram__bytes_write.sum [bytes]", 0) or 0
        d["dram_bytes_per_launch"] = rb + wb
        ms = d.get("gpu__time_duration.sum [ms]")
        if ms:
            d["dram_GBps"] = round((rb + wb) / ms / 1e6, 1)
        out.append(d)
    return out


def launches_summary(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        t = num(r["Metric Value"], r.get("Metric Unit", ""))
        a = agg.setdefault(name, {"launches": 0, "total_ms": 0.0})
        a["launches"] += 1
        a["total_ms"] += t
    total = sum(a["total_ms"] for a in agg.values()) or 1.0
    for a in agg.values():
        a["share"] = round(a["total_ms"] / total, 4)
        a["total_ms"] = round(a["total_ms"], 4)
    return {"kernels": agg, "total_ms": round(total, 4), "note": "ncu per-launch durations are cold-cache and serialised; compare shares"}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rep")
    p.add_argument("--launches")
    p.add_argument("--out", required=True)
    p.add_argument("--note", default="")
    a = p.parse_args()
    out = {"note": a.note}
    if a.rep:
        out["full_set"] = rep_summary(a.rep)
    if a.launches:
        out["launch_list"] = launches_summary(a.launches)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
