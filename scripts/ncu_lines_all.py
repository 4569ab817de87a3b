"""Per-source-line stall samples of an ncu report across ALL source files (file-qualified):
usage: ncu_lines_all.py REPORT [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, fname, ie, ii = [], "?", None, None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "File Name":
        fname = r[1].split("/")[-1] if len(r) > 1 else "?"
        continue
    if r and r[0] == "Line No":
        ie = r.index("Warp Stall Sampling (All Samples)")
        ii = r.index("Instructions Executed")
        continue
    if ie is None or len(r) <= max(ie, ii) or not r[0].strip().isdigit():
        continue
    try:
        agg.append((float(r[ie] or 0), float(r[ii] or 0), fname, r[0], r[1]))
    except ValueError:
        pass
ts = sum(a[0] for a in agg) or 1
ti = sum(a[1] for a in agg) or 1
byf = {}
for a in agg:
    byf[a[2]] = byf.get(a[2], 0) + a[0]
print("samples by file:", {k: f"{v / ts * 100:.1f}%" for k, v in sorted(byf.items(), key=lambda kv: -kv[1])})
for a in sorted(agg, key=lambda a: -a[0])[:top]:
    print(f"{a[2][:14]:>14}:{a[3]:>4} samp {a[0] / ts * 100:5.1f}% inst {a[1] / ti * 100:5.1f}% {a[4].strip()[:90]}")
