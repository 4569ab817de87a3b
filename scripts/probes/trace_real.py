"""Per-iteration time of the persistent CG kernel during a REAL fullsky solve (tol 1e-10) versus the
number of faces still active (KCG_TRACE=1 build).  usage: KCG_LIB_PATH=... trace_real.py [config]"""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from synth import make_config
from synth.problems import stack
from paper_2204_08057_b200 import kroncg
from paper_2204_08057_b200.kroncg import KronCG

cfg = sys.argv[1] if len(sys.argv) > 1 else "fullsky"
ps = make_config(cfg)
st = stack(ps)
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"])
Y = torch.from_numpy(st["Y"]).cuda()
for _ in range(2):
    _, rep = ctx.solve(Y, tol=1e-10)
its = np.array(rep["iterations_per"])
f = kroncg._lib.kcg_debug_trace
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((1024, 160), dtype=np.int64)
n = int(its.max()) + 1
f(ctx._ctx, buf.ctypes.data, n)
T = buf[:n].astype(np.float64) / 1e3
dt = T[1:n, 0] - T[:n - 1, 0]                 # pass q -> q+1 start-to-start
tiles = T[:n - 1, 3:3 + 148]
work = tiles.max(1) - T[:n - 1, 0]
wmin = tiles.min(1) - T[:n - 1, 0]
wmed = np.median(tiles, 1) - T[:n - 1, 0]
active = np.array([(its >= q).sum() for q in range(n - 1)])
out = {"cfg": cfg, "loop_ms": rep["loop_time_s"] * 1e3, "sum_dt_ms": float(dt.sum() / 1e3)}
for a in sorted(set(active.tolist()), reverse=True):
    m = active == a
    out[f"active{a}"] = {"passes": int(m.sum()), "us_per_pass": round(float(np.median(dt[m])), 1),
                          "us_per_face_pass": round(float(np.median(dt[m])) / max(a, 1), 1),
                          "work_us_min_med_max": [round(float(np.median(x[m])), 1) for x in (wmin, wmed, work)]}
print(json.dumps(out))
