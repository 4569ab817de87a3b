import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import numpy as np
from gpu_util import make_ctx
from synth import make_patch
L, k, P, store = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ps = [make_patch(L, 9, k, seed=300 + s, tau="loguniform", prior="d2") for s in range(P)]
ctx, Y = make_ctx(ps, lanczos_cap=400, lanczos_store=bool(store), prior="d2")
print(ctx.launch_config())
mu, rep = ctx.lanczos(Y, tol=1e-10)
print("OK", L, k, P, store, rep["iterations_per"])
