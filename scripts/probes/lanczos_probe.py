"""Time the block-Lanczos route (sylvester_lanczos_solve) on a BASELINE config: steps, kernel time,
algorithmic bytes / kernel time vs the measured HBM peak.  usage: lanczos_probe.py CONFIG [store]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2204_08057_b200.kroncg import KronCG  # noqa: E402
from synth import make_config  # noqa: E402
from synth.problems import stack  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "planck"
store = "store" in sys.argv[2:]
prior = "d2" if "d2" in sys.argv[2:] else "laplacian"
ps = make_config(name, prior=prior)
st = stack(ps)
cap = 320
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"], lanczos_cap=cap, lanczos_store=store,
             prior=prior)
Y = torch.from_numpy(st["Y"]).cuda()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.7) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6550.7
for rep_i in range(4):
    mu, r = ctx.lanczos(Y, tol=1e-10)
print(json.dumps(dict(config=name, store=store, prior=prior, steps=r["iterations_per"], status=r["status_name"],
                      wall_ms=r["wall_time_s"] * 1e3, loop_ms=r["loop_time_s"] * 1e3,
                      loop_GBs=r["loop_bytes"] / r["loop_time_s"] / 1e9, frac=r["loop_bytes"] / r["loop_time_s"] / 1e9 / peak,
                      rel_true=r["rel_residual_true"], solves_per_s=1.0 / r["wall_time_s"])))
