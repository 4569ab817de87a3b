"""Add the ORACLE block-Lanczos step counts (oracle.lanczos, Alg. SylvSolver, tol 1e-10) per face to
tests/golden/oracle_iterations.json ("lanczos_iterations").  Calls only oracle/ and synth/; used
by the GPU parity tests at sizes where re-running the oracle would be slow (planck, fullsky)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import CONFIGS, make_config  # noqa: E402
from oracle import lanczos  # noqa: E402

out_path = os.path.join(ROOT, "tests", "golden", "oracle_iterations.json")
names = sys.argv[1:] or ["tiny", "medium", "planck", "fullsky"]
for name in names:
    t0 = time.time()
    its = []
    for i in range(len(CONFIGS[name]["seeds"])):
        p = make_config(name, patches=[i])[0]
        r = lanczos.problem_solve(p, tol=1e-10)
        its.append(r.iterations)
        print(name, i, r.iterations, f"{time.time() - t0:.0f}s", flush=True)
    res = json.load(open(out_path))
    res.setdefault(name, {})["lanczos_iterations"] = its
    res[name]["_source_lanczos"] = "scripts/oracle_lanczos_iterations.py (oracle.lanczos.solve)"
    json.dump(res, open(out_path, "w"), indent=1)
