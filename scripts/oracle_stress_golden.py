"""Write the stress-config oracle golden data (BASELINE configs[4]: L = 11, k = 6, seed 3).

Calls only oracle/ and synth/ (never the CUDA path).  The oracle's full solution (4,194,304 x 6
doubles = 201 MB) is too large to commit, so this stores what a GPU test needs to compare with it
element by element and in norm:

* `tests/golden/oracle_iterations.json["stress"]`: oracle HS-CG iteration count (textbook CG,
  P:L225-241, readings R7/R8) and the Sylvester-route per-column counts (Lemma 2);
* `tests/golden/stress_oracle_sample.npz`: the oracle iterate x_or at 16384 seeded sample indices
  (PCG64(20250) without replacement over the k*N entries, component-major vec), ||x_or||_2, and
  rel(x_or, x_dct) where x_dct is the exact DCT-II solve (oracle/exact.py).

The GPU test then checks (i) the sampled entries element by element, (ii) |it_gpu - it_or| <= 2,
and (iii) the triangle bound rel(x_gpu, x_or) <= rel(x_gpu, x_dct)*|x_dct|/|x_or| + rel(x_or, x_dct)
*|x_dct|/|x_or|, evaluated against a full-size DCT-exact solve it recomputes (not stored).

Run time: about 20-40 CPU-minutes (one literal sparse assembly of a 25M x 25M G, ~1450 SpMVs).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import make_config  # noqa: E402
from oracle import cg, exact, model, sylvester  # noqa: E402

SAMPLE_SEED = 20250
N_SAMPLE = 16384

t0 = time.time()
p = make_config("stress")[0]
G, b = model.problem_system(p)
print("assembled", G.shape, G.nnz, f"{time.time() - t0:.0f}s", flush=True)
r = cg.cg_hs(G, b, tol=1e-10, max_iter=100000)
print("cg_hs", r.iterations, r.converged, r.rel_residual, f"{time.time() - t0:.0f}s", flush=True)
assert r.converged
true_res = float(np.linalg.norm(b - G @ r.x) / np.linalg.norm(b))
del G
xd = exact.problem_dct_exact(p)
rel_or_dct = float(np.linalg.norm(r.x - xd) / np.linalg.norm(xd))
print("rel(x_or, x_dct)", rel_or_dct, "true residual", true_res, flush=True)
rng = np.random.Generator(np.random.PCG64(SAMPLE_SEED))
idx = np.sort(rng.choice(r.x.size, size=N_SAMPLE, replace=False))
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "stress_oracle_sample.npz"),
                    idx=idx.astype(np.int64), x=r.x[idx], x_norm=np.linalg.norm(r.x),
                    dct_norm=np.linalg.norm(xd), rel_or_dct=rel_or_dct,
                    iterations=r.iterations, true_residual=true_res)
s = sylvester.problem_solve(p, tol=1e-10)
print("sylvester", s.iterations, f"{time.time() - t0:.0f}s", flush=True)

out_path = os.path.join(ROOT, "tests", "golden", "oracle_iterations.json")
res = json.load(open(out_path))
ent = res.get("stress", {})
ent.update({"kron_cg_iterations": [int(r.iterations)],
            "sylvester_iterations": [[int(v) for v in s.iterations]], "tol": 1e-10,
            "_source": "scripts/oracle_stress_golden.py (oracle.cg.cg_hs / oracle.sylvester.solve)",
            "rel_oracle_vs_dct_exact": rel_or_dct, "oracle_true_residual": true_res})
res["stress"] = ent
json.dump(res, open(out_path, "w"), indent=1)
print("done", f"{time.time() - t0:.0f}s", flush=True)
