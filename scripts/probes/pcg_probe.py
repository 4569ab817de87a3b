import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth import make_config
from synth.problems import stack
ps = make_config(sys.argv[1] if len(sys.argv) > 1 else "fullsky")
st = stack(ps)
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], precond="block_jacobi")
Y = torch.from_numpy(st["Y"]).cuda()
ts = []
for _ in range(5):
    mu, r = ctx.solve(Y, tol=1e-10)
    ts.append(r["loop_time_s"] * 1e3)
print(json.dumps({"lib": os.environ.get("KCG_LIB_PATH", "default"), "loop_ms": sorted(ts)[2], "its": r["system_iterations"]}))
