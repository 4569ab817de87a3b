"""Per-pass phase breakdown of the slab CG kernel (KCG_TRACE=1 build), planck face split G ways."""
import ctypes, os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from synth import make_config
from synth.problems import stack
from paper_2204_08057_b200 import kroncg
from paper_2204_08057_b200.kroncg import KronCGSlab, split_rows
G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = make_config("planck")[0]
st = stack([p])
Y = split_rows(torch.from_numpy(st["Y"]).cuda(), G)
ctx = KronCGSlab(p.level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], G, emulate=True)
for _ in range(2):
    ctx.solve(Y, tol=1e-300, max_iter=100)
_, rep = ctx.solve(Y, tol=1e-300, max_iter=100)
f = kroncg._lib.kcg_debug_trace
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
n = 101
buf = np.zeros((1024, 160), dtype=np.int64)
f(ctx._ctx, buf.ctypes.data, n)
T = buf[:n].astype(np.float64) / 1e3
ncta = ctx.launch_config()["grid_kron"]
t0, tflag, tred = T[:, 0], T[:, 1], T[:, 2]
tiles = T[:, 3:3 + ncta]
it = np.arange(5, n - 1)
med = lambda x: round(float(np.median(x)), 2)
print(json.dumps({"G": G, "ctas_per_rank": ncta, "us_per_pass": rep["loop_time_s"] / 101 * 1e6,
                  "work_min_med_max": [med(tiles[it].min(1) - t0[it]), med(np.median(tiles[it] - t0[it][:, None], 1)), med(tiles[it].max(1) - t0[it])],
                  "flags_after_last_tile": med(tflag[it] - tiles[it].max(1)), "update": med(tred[it] - tflag[it]),
                  "to_next": med(t0[it + 1] - tred[it]), "pass": med(t0[it + 1] - t0[it])}))
