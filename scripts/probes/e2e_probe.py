"""Where the e2e time goes (fullsky): device-resident solve per step vs kron_cg_solve_host_many with
n = 2, 5, 10, 20 steps (slope = per-step cost, intercept = pipeline fill / drain); plus the bare
H2D / D2H copy times.  usage: e2e_probe.py"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth import make_config
from synth.problems import stack

ps = make_config("fullsky")
st = stack(ps)
dev = torch.device("cuda:0")
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], device=dev, host_staging=2)
Y = torch.from_numpy(st["Y"]).to(dev)
mu = torch.empty(ctx.shape_mu, dtype=torch.float64, device=dev)
Yh = torch.from_numpy(st["Y"]).pin_memory()
mh = [torch.empty(ctx.shape_mu, dtype=torch.float64).pin_memory() for _ in range(2)]
s = torch.cuda.current_stream()

def ev_time(fn, reps=1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)

out = {}
for _ in range(3):
    ctx.solve(Y, mu, tol=1e-10)
out["device_ms_per_step"] = ev_time(lambda: ctx.solve(Y, mu, tol=1e-10), 10) / 10
loops = []
for _ in range(10):
    _, r = ctx.solve(Y, mu, tol=1e-10)
    loops.append(r["loop_time_s"] * 1e3)
out["loop_ms"] = float(np.median(loops))
out["wall_ms_report"] = r["wall_time_s"] * 1e3
out["h2d_ms"] = ev_time(lambda: Y.copy_(Yh, non_blocking=True), 3) / 3
out["d2h_ms"] = ev_time(lambda: mh[0].copy_(mu, non_blocking=True), 3) / 3
for n in (2, 5, 10, 20):
    ctx.solve_host_many([Yh] * n, [mh[i & 1] for i in range(n)], tol=1e-10)
    t = ev_time(lambda: ctx.solve_host_many([Yh] * n, [mh[i & 1] for i in range(n)], tol=1e-10))
    out[f"host_many_{n}_ms"] = t
    out[f"host_many_{n}_ms_per_step"] = t / n
# host-side gap: wall clock per device-resident step
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    ctx.solve(Y, mu, tol=1e-10)
torch.cuda.synchronize()
out["host_wall_ms_per_step"] = (time.perf_counter() - t0) * 100
print(json.dumps({k: round(v, 3) for k, v in out.items()}))

# interference: the device-resident solve while another stream streams H2D copies of Y (and D2H of mu)
side = torch.cuda.Stream()
Yb = torch.empty_like(Y)
mb = torch.empty_like(mu)
def busy(nc):
    with torch.cuda.stream(side):
        for i in range(nc):
            Yb.copy_(Yh, non_blocking=True)
            mh[i & 1].copy_(mb, non_blocking=True)
res = {}
for nc in (0, 1, 3):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        busy(nc)
        ts.append(ev_time(lambda: ctx.solve(Y, mu, tol=1e-10)))
        torch.cuda.synchronize()
    res[f"solve_ms_with_{nc}_copy_pairs"] = round(float(np.median(ts)), 3)
print(json.dumps(res))

# serial paths: one host_many step (H2D + solve + D2H, nothing to overlap) and the blocking host entry
res = {}
for _ in range(2):
    ctx.solve_host_many([Yh], [mh[0]], tol=1e-10)
res["host_many_1_ms"] = round(float(np.median([ev_time(lambda: ctx.solve_host_many([Yh], [mh[0]], tol=1e-10)) for _ in range(3)])), 3)
res["solve_host_ms"] = round(float(np.median([ev_time(lambda: ctx.solve_host(Yh, mh[0], tol=1e-10)) for _ in range(3)])), 3)
reps = ctx.solve_host_many([Yh] * 4, [mh[i & 1] for i in range(4)], tol=1e-10)
res["host_many_4_loop_ms"] = [round(r["loop_time_s"] * 1e3, 3) for r in reps]
res["host_many_4_wall_ms"] = [round(r["wall_time_s"] * 1e3, 3) for r in reps]
print(json.dumps(res))
