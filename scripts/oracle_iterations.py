"""Write tests/golden/oracle_iterations.json: per-face iteration counts of the ORACLE (textbook
HS-CG on the literal assembled system, tol 1e-10) for the BASELINE configs.  Calls only oracle/
and synth/; used by bench.py --impl reference to extrapolate a bounded oracle sample to a full
solve, and as context for the GPU parity tests."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import CONFIGS, make_config  # noqa: E402
from oracle import cg, model, sylvester  # noqa: E402

out_path = os.path.join(ROOT, "tests", "golden", "oracle_iterations.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
names = sys.argv[1:] or ["tiny", "medium", "planck", "fullsky", "stress"]
for name in names:
    t0 = time.time()
    its, syl = [], []
    for i in range(len(CONFIGS[name]["seeds"])):
        p = make_config(name, patches=[i])[0]
        G, b = model.problem_system(p)
        r = cg.cg_hs(G, b, tol=1e-10, max_iter=100000)
        its.append(r.iterations)
        del G
        s = sylvester.problem_solve(p, tol=1e-10)
        syl.append(s.iterations)
        print(name, i, r.iterations, s.iterations, f"{time.time() - t0:.0f}s", flush=True)
    res[name] = {"kron_cg_iterations": its, "sylvester_iterations": syl, "tol": 1e-10,
                 "_source": "scripts/oracle_iterations.py (oracle.cg.cg_hs / oracle.sylvester.solve)"}
    json.dump(res, open(out_path, "w"), indent=1)
