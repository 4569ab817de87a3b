"""Build experimental variants of libkroncg (compile-time tile/thread/M-placement knobs)."""
import os, sys
from concurrent.futures import ThreadPoolExecutor
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2204_08057_b200 import build

VARIANTS = {
    "a16x256": [],
    "b8x256x2": ["KCG_TY4=8", "KCG_MINB4=2"],
    "c8x128x2": ["KCG_TY4=8", "KCG_NT4=128", "KCG_MINB4=2"],
    "d16x128": ["KCG_NT4=128"],
    # D2 row march, K = 4: two face columns per lane (64-column boxes, 56 output columns)
    "m4c2k2g4": ["KCG_MKP4=2", "KCG_MCP4=2", "KCG_MG4=4"],
    "m4c2k1g3": ["KCG_MKP4=1", "KCG_MCP4=2", "KCG_MG4W=3"],
    "m4c2k1g4": ["KCG_MKP4=1", "KCG_MCP4=2", "KCG_MG4W=4"],
    # after the change: K = 4 with hits (two planes per warp), groups per CTA
    "m4hg5": ["KCG_MG4=5"],
    "m4hg3": ["KCG_MG4=3"],
    "m4hs8g3": ["KCG_MG4=3", "KCG_MST4=8"],
    # K = 4 with hits, one column per lane (24-column strips): more, thinner warps
    "m4hc1k2g6": ["KCG_MCP4=1", "KCG_MKP4H=2", "KCG_MG4=6"],
    "m4hc1k2g7": ["KCG_MCP4=1", "KCG_MKP4H=2", "KCG_MG4=7"],
    "m4hc1k2g8": ["KCG_MCP4=1", "KCG_MKP4H=2", "KCG_MG4=8"],
    "m4hc1k4g8": ["KCG_MCP4=1", "KCG_MKP4H=4", "KCG_MG4Q=8"],
    "mint": ["KCG_MINT=1"],
    "apty8": ["KCG_AP_TYD2=8"],
    "apty4": ["KCG_AP_TYD2=4"],
    "m4hc1k4g9": ["KCG_MCP4=1", "KCG_MKP4H=4", "KCG_MG4Q=9"],
}
names = sys.argv[1:] or list(VARIANTS)
out = os.path.join(ROOT, "paper_2204_08057_b200", "lib", "variants")
with ThreadPoolExecutor(len(names)) as ex:
    futs = {n: ex.submit(build.build, True, False, tuple(VARIANTS[n]), os.path.join(out, n + ".so")) for n in names}
    for n, f in futs.items():
        print(n, f.result())
