"""Sample SM / memory clocks, power and throttle reasons (nvidia-smi, 20 ms) during back-to-back
fullsky Kron-CG solves; print per-solve loop time next to the samples."""
import json, os, subprocess, sys, threading, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
from paper_2204_08057_b200.kroncg import KronCG
from synth import make_config
from synth.problems import stack
ps = make_config("fullsky")
st = stack(ps)
ctx = KronCG(ps[0].level, st["A"], st["noise_prec"], st["tau"], st["kappa2"])
Y = torch.from_numpy(st["Y"]).cuda()
samples, stop = [], [False]
def sampler():
    q = "clocks.sm,clocks.mem,power.draw,clocks_throttle_reasons.sw_power_cap,clocks_throttle_reasons.hw_slowdown"
    p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "20"],
                         stdout=subprocess.PIPE, text=True)
    while not stop[0]:
        line = p.stdout.readline()
        if line:
            samples.append((time.time(), line.strip()))
    p.terminate()
th = threading.Thread(target=sampler); th.start()
time.sleep(0.5)
ts = []
for _ in range(30):
    _, r = ctx.solve(Y, tol=1e-10)
    ts.append(round(r["loop_time_s"] * 1e3, 2))
time.sleep(0.2)
stop[0] = True; th.join(timeout=2)
print(json.dumps({"loop_ms": ts}))
for t, l in samples[::5]:
    print(l)
