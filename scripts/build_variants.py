"""Build experimental variants of libkroncg (compile-time tile/thread/M-placement knobs)."""
import os, sys
from concurrent.futures import ThreadPoolExecutor
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2204_08057_b200 import build

VARIANTS = {
    "trace": ["KCG_TRACE=1"],
}
names = sys.argv[1:] or list(VARIANTS)
out = os.path.join(ROOT, "paper_2204_08057_b200", "lib", "variants")
with ThreadPoolExecutor(len(names)) as ex:
    futs = {n: ex.submit(build.build, True, False, tuple(VARIANTS[n]), os.path.join(out, n + ".so")) for n in names}
    for n, f in futs.items():
        print(n, f.result())
