"""Per-pass phase breakdown of the block-Lanczos kernel (needs a KCG_TRACE=1 build).
usage: KCG_LIB_PATH=.../trace.so python scripts/lz_trace_probe.py [config] [store]"""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from synth import make_config
from synth.problems import stack
from paper_2204_08057_b200 import kroncg
from paper_2204_08057_b200.kroncg import KronCG

cfg = sys.argv[1] if len(sys.argv) > 1 else "planck"
store = len(sys.argv) > 2 and sys.argv[2] == "store"
ps = make_config(cfg)
st = stack(ps)
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], lanczos_cap=320, lanczos_store=store)
Y = torch.from_numpy(st["Y"]).cuda()
for _ in range(3):
    _, rep = ctx.lanczos(Y, tol=1e-10)
f = kroncg._lib.kcg_debug_trace
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((1024, 160), dtype=np.int64)
n = max(rep["iterations_per"]) + 1
f(ctx._ctx, buf.ctypes.data, n)
T = buf[:n].astype(np.float64) / 1e3
tiles = T[:, 5:5 + 148]
q = np.arange(2, n - 1)
out = {"cfg": cfg, "store": store, "steps": rep["iterations_per"], "loop_ms": rep["loop_time_s"] * 1e3,
       "pass_us": float(np.median(T[q + 1, 0] - T[q, 0])),
       "tiles_min_us": float(np.median(tiles[q].min(1) - T[q, 0])),
       "tiles_med_us": float(np.median(np.median(tiles[q], 1) - T[q, 0])),
       "tiles_max_us": float(np.median(tiles[q].max(1) - T[q, 0])),
       "sync1_us": float(np.median(T[q, 2] - tiles[q].max(1))),
       "reduce_us": float(np.median(T[q, 3] - T[q, 2])),
       "sync2_us": float(np.median(T[q, 4] - T[q, 3])),
       "next_us": float(np.median(T[q + 1, 0] - T[q, 4])),
       "red_partials_us": float(np.median(T[q, 153] - T[q, 2])),
       "red_chol_us": float(np.median(T[q, 154] - T[q, 153])),
       "red_shifts_us": float(np.median(T[q, 155] - T[q, 154])),
       "red_tail_us": float(np.median(T[q, 3] - T[q, 155])),
       "tail_ms": float((T[n - 1, 4] - T[0, 0]) / 1e3)}
print(json.dumps(out))
