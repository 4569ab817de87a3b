"""us per CG iteration of the streaming tile kernel (KCG_RESIDENT=0) on the tiny and medium configs
(k = 3), best of 20 solves after warm-up.  usage: small_probe.py"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ["KCG_RESIDENT"] = "0"
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth import make_config
from synth.problems import stack
out = {}
for cfg in ("tiny", "medium"):
    ps = make_config(cfg)
    st = stack(ps)
    ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"])
    Y = torch.from_numpy(st["Y"]).cuda()
    ts = []
    for i in range(25):
        _, r = ctx.solve(Y, tol=1e-10)
        if i >= 5:
            ts.append(r["loop_time_s"] * 1e6 / (r["iterations"] + 1))
    out[cfg] = {"us_per_iter": round(min(ts), 2), "iters": r["iterations"], "rel_true": r["rel_residual_true"]}
print(json.dumps(out))
