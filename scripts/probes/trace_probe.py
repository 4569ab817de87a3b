"""Per-iteration phase breakdown of the persistent CG kernel (needs a KCG_TRACE=1 build).
usage: KCG_LIB_PATH=.../trace.so python scripts/trace_probe.py [config] [iters] [route]"""
import ctypes, os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from synth import make_config
from synth.problems import stack
from paper_2204_08057_b200 import kroncg
from paper_2204_08057_b200.kroncg import KronCG

cfg = sys.argv[1] if len(sys.argv) > 1 else "planck"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
route = sys.argv[3] if len(sys.argv) > 3 else "kron"
ps = make_config(cfg)
st = stack(ps)
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"])
Y = torch.from_numpy(st["Y"]).cuda()
fn = ctx.solve if route == "kron" else ctx.sylvester
for _ in range(2):
    fn(Y, tol=1e-300, max_iter=iters)
_, rep = fn(Y, tol=1e-300, max_iter=iters)
f = kroncg._lib.kcg_debug_trace
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
n = min(iters + 1, 1024)
buf = np.zeros((1024, 160), dtype=np.int64)
cols = f(ctx._ctx, buf.ctypes.data, n)
T = buf[:n].astype(np.float64) / 1e3  # us
t0, tsync, tred = T[:, 0], T[:, 1], T[:, 2]
tiles = T[:, 3:3 + 148]
it = np.arange(5, n - 1)
work_min = (tiles[it].min(1) - t0[it]); work_med = np.median(tiles[it] - t0[it][:, None], 1); work_max = tiles[it].max(1) - t0[it]
sync = tsync[it] - tiles[it].max(1)
red = tred[it] - tsync[it]
nxt = t0[it + 1] - tred[it]
tot = t0[it + 1] - t0[it]
print(json.dumps({"cfg": cfg, "route": route, "loop_us_per_iter": rep["loop_time_s"] / (iters + 1) * 1e6,
                  "iter_us": round(float(np.median(tot)), 2),
                  "work_us_min_med_max": [round(float(np.median(x)), 2) for x in (work_min, work_med, work_max)],
                  "sync_after_last_cta_us": round(float(np.median(sync)), 2),
                  "reduce_us": round(float(np.median(red)), 2), "to_next_start_us": round(float(np.median(nxt)), 2)}))
