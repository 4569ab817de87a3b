"""Kron-CG loop time with k = 3 on large faces (level 10: one face, and 12 faces), for the K = 2, 3 tile
geometry A/B.  usage: k3_large_probe.py"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth import make_patch
from synth.problems import stack
out = {}
for name, nf in (("L10x1", 1), ("L10x12", 12), ("L9x4", 4)):
    lv = 9 if name == "L9x4" else 10
    ps = [make_patch(lv, 9, 3, seed=700 + i, tau="loguniform") for i in range(nf)]
    st = stack(ps)
    ctx = KronCG(lv, st["A"], st["noise_prec"], st["tau"], st["kappa2"])
    Y = torch.from_numpy(st["Y"]).cuda()
    ts = []
    for i in range(6):
        _, r = ctx.solve(Y, tol=1e-10)
        if i >= 1:
            ts.append(r["loop_time_s"] * 1e3)
    out[name] = {"loop_ms": round(min(ts), 3), "face_iters": r["system_iterations"],
                 "us_per_face_iter": round(min(ts) * 1e3 / r["system_iterations"], 2)}
    del ctx
print(json.dumps(out))
