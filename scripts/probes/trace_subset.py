"""Per-pass CG time for fixed batches of fullsky faces (KCG_TRACE=1 build), max_iter capped so every
face stays active: separates a batch-composition effect from a pass-index / value effect.
usage: KCG_LIB_PATH=.../trace1.so trace_subset.py"""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from synth import make_config
from synth.problems import stack
from paper_2204_08057_b200 import kroncg
from paper_2204_08057_b200.kroncg import KronCG

ps_all = make_config("fullsky")
f = kroncg._lib.kcg_debug_trace
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
subsets = {"all12": list(range(12)), "0-10": list(range(11)), "1-11": list(range(1, 12)),
           "0-7": list(range(8)), "4-11": list(range(4, 12)), "0-8": list(range(9)), "face0": [0],
           "face0x12": [0] * 12, "face0x11": [0] * 11}
cap = int(sys.argv[1]) if len(sys.argv) > 1 else 80
for name, idx in subsets.items():
    ps = [ps_all[i] for i in idx]
    st = stack(ps)
    ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"])
    Y = torch.from_numpy(st["Y"]).cuda()
    for _ in range(2):
        _, rep = ctx.solve(Y, tol=1e-10, max_iter=cap)
    buf = np.zeros((1024, 160), dtype=np.int64)
    n = cap + 1
    f(ctx._ctx, buf.ctypes.data, n)
    T = buf[:n].astype(np.float64) / 1e3
    dt = T[1:n, 0] - T[:n - 1, 0]
    dt = dt[2:]
    out = {"subset": name, "faces": len(idx), "loop_ms": round(rep["loop_time_s"] * 1e3, 3),
           "us_per_pass_med": round(float(np.median(dt)), 1),
           "us_per_face_pass": round(float(np.median(dt)) / len(idx), 2),
           "first10": [round(float(v), 1) for v in dt[:10]], "last10": [round(float(v), 1) for v in dt[-10:]]}
    print(json.dumps(out), flush=True)
    del ctx
    torch.cuda.empty_cache()
