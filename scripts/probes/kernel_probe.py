"""Steady-state CG-kernel bandwidth probe: fixed iteration count (tol 1e-300), all systems active.
usage: KCG_LIB_PATH=... python scripts/kernel_probe.py [config] [iters] [route]"""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from synth import make_config
from synth.problems import stack
from paper_2204_08057_b200.kroncg import KronCG

cfg = sys.argv[1] if len(sys.argv) > 1 else "fullsky"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
route = sys.argv[3] if len(sys.argv) > 3 else "kron"
ps = make_config(cfg)
st = stack(ps)
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"])
Y = torch.from_numpy(st["Y"]).cuda()
fn = ctx.solve if route == "kron" else ctx.sylvester
for _ in range(2):
    fn(Y, tol=1e-300, max_iter=iters)
res = []
for _ in range(3):
    _, r = fn(Y, tol=1e-300, max_iter=iters)
    res.append(r["loop_bytes"] / r["loop_time_s"] / 1e9)
lib = os.path.basename(os.environ.get("KCG_LIB_PATH", "default"))
print(json.dumps({"lib": lib, "cfg": cfg, "route": route, "iters": iters, "GBps": [round(x) for x in res],
                  "frac": round(max(res) / 6550.7, 3), "us_per_iter": round(r["loop_time_s"] / (iters + 1) * 1e6, 2)}))
