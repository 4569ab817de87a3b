"""Summarise an ncu report: key raw metrics, stall reasons, per-source-line hot spots."""
import csv, io, re, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
def g(name):
    return vals[hdr.index(name)] if name in hdr else None
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_bytes.sum", "launch__occupancy_limit_registers", "smsp__thread_inst_executed_per_inst_executed.ratio"]
for k in keys:
    print(f"{k:70s} {g(k)} {units[hdr.index(k)] if k in hdr else ''}")
items = []
for i, h in enumerate(hdr):
    if re.search(r"smsp__pcsamp_warps_issue_stalled_\w+$", h) and not h.endswith("not_issued"):
        try:
            items.append((float(vals[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(v for v, _ in items)
print("stalls:", ", ".join(f"{h} {v / tot * 100:.1f}%" for v, h in sorted(items, reverse=True)[:10]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
hdr = rows[h]
ie = hdr.index("Warp Stall Sampling (All Samples)"); ii = hdr.index("Instructions Executed")
agg = []
for r in rows[h + 1:]:
    if len(r) <= ii or r[0] == "" or r[0] == "Line No":
        if r and r[0] == "Line No":
            break
        continue
    try:
        agg.append((float(r[ie]), float(r[ii]), r[0], r[1]))
    except ValueError:
        pass
ts = sum(a[0] for a in agg) or 1; ti = sum(a[1] for a in agg) or 1
print(f"total warp-inst {ti:.3g}")
for a in sorted(agg, key=lambda a: -a[0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"L{a[2]:>4} samp {a[0] / ts * 100:5.1f}% inst {a[1] / ti * 100:5.1f}% {a[3][:90]}")
