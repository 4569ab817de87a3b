"""Per-CUDA-source-line warp-stall samples of an ncu report (all files), top N lines.
usage: ncu_lines.py REPORT [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
agg, tot, path = {}, 0.0, ""
ie = None
for r in rows:
    if r and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        ie = r.index("Warp Stall Sampling (All Samples)")
        continue
    if ie is None or len(r) <= ie or r[0] in ("", "Function Name"):
        continue
    try:
        v = float(r[ie])
    except ValueError:
        continue
    tot += v
    key = (path, r[0], r[1][:100])
    agg[key] = agg.get(key, 0.0) + v
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    print(f"{v / tot * 100:5.1f}% {k[0]}:{k[1]} {k[2]}")
