"""Per-pass phase breakdown of the shared-memory-resident CG kernel (needs a KCG_TRACE=1 build):
usage: KCG_LIB_PATH=.../trace.so python scripts/probes/res_trace_probe.py [config] [iters]"""
import ctypes, os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from synth import make_config
from synth.problems import stack
from paper_2204_08057_b200 import kroncg
from paper_2204_08057_b200.kroncg import KronCG

cfg = sys.argv[1] if len(sys.argv) > 1 else "medium"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
ps = make_config(cfg)
st = stack(ps)
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"])
Y = torch.from_numpy(st["Y"]).cuda()
for _ in range(2):
    ctx.solve(Y, tol=1e-300, max_iter=iters)
_, rep = ctx.solve(Y, tol=1e-300, max_iter=iters)
f = kroncg._lib.kcg_debug_trace
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
n = min(iters + 1, 1024)
buf = np.zeros((1024, 160), dtype=np.int64)
f(ctx._ctx, buf.ctypes.data, n)
T = buf[:n].astype(np.float64) / 1e3  # us
q = np.arange(5, n - 1)
cfgd = ctx.launch_config()
ncta = int(cfgd.get("resident_kron", 0))
arr = T[q][:, 6:6 + max(ncta, 1)]
med = lambda x: round(float(np.median(x)), 2)
print(json.dumps({"cfg": cfg, "strips": ncta, "env_rs": os.environ.get("KCG_RES_RS"),
                  "loop_us_per_iter": rep["loop_time_s"] / (iters + 1) * 1e6,
                  "pass_us": med(T[q + 1, 0] - T[q, 0]), "A": med(T[q, 1] - T[q, 0]), "B": med(T[q, 2] - T[q, 1]),
                  "C+publish": med(T[q, 3] - T[q, 2]),
                  "cta_arrive_spread": med(arr.max(1) - arr.min(1)), "sync_after_last": med(T[q, 4] - arr.max(1)),
                  "reduce+halo": med(T[q, 5] - T[q, 4]), "tail_to_next": med(T[q + 1, 0] - T[q, 5])}))
