"""Per-CUDA-source-line instruction counts and stall samples from an ncu
report (--page source --print-source cuda,sass):
python scripts/ncu_lines.py REPORT [function-substring] [top]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn, hdr, seen = None, None, set()
per_fn = {}


def _f(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or want not in (fn or ""):
        continue
    si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    per_fn.setdefault(fn, {})[(int(r[0]), r[1].strip()[:90])] = (_f(r[ii]), _f(r[si]))
for fn, lines in per_fn.items():
    if fn in seen:
        continue
    seen.add(fn)
    ti = sum(v[0] for v in lines.values()) or 1
    ts = sum(v[1] for v in lines.values()) or 1
    print(f"== {fn[:100]}  inst {ti:.3g}  samples {ts:.0f}")
    for (ln, src), (i, s) in sorted(lines.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% stall  L{ln} {src}")
