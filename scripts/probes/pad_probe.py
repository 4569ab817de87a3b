import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth import make_config
from synth.problems import stack
cfg = sys.argv[1] if len(sys.argv) > 1 else "fullsky"
ps = make_config(cfg)
st = stack(ps)
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"])
Y = torch.from_numpy(st["Y"]).cuda()
ts = []
for _ in range(5):
    _, r = ctx.solve(Y, tol=1e-10)
    ts.append(r["loop_time_s"] * 1e3)
print(json.dumps({"cfg": cfg, "pad_kb": os.environ.get("KCG_PAD_KB", "0"), "loop_ms": sorted(ts)[2],
                  "frac_bytes": r["loop_bytes"] / (sorted(ts)[2] * 1e-3) / 1e9 / 6456.8}))
