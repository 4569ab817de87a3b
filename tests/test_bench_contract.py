"""The bench.py JSON-line contract, checked on the committed round-end line (profiles/r01) and on
the argument parser (CPU only; the GPU run itself is the driver's)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINE = os.path.join(ROOT, "profiles", "r01", "bench_fullsky_v20.json")


def test_committed_bench_line_has_every_contract_key():
    d = json.load(open(LINE))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks",
              "cpu_baseline"):
        assert k in d, k
    assert d["config"]["workload"] == "fullsky" and d["dtype"] == "f64" and d["higher_is_better"] is True
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and r["traffic"] > 0
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and 0 < e["value"] <= d["value"]
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["sample"] and 0 < c["value"] < d["value"]
    assert d["gpu_launches"] == 5 * d["steps"]
    assert d["clocks"]["sm_mhz"] > 0 and "reasons" in d["clocks"]
    # every further route / row reports its own value and roofline
    for k in ("sylvester", "lanczos", "kohler", "pcg_block_jacobi", "posterior_variance"):
        assert d[k]["value"] > 0 and 0 < d[k]["roofline"]["frac"] < 1, k
    assert d["lanczos"]["cpu_baseline"]["kind"] == "oracle"
    assert set(d["paper_workload"]) >= {"kron", "sylvester", "lanczos"}


def test_bench_cli_flags():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--config", "--no-lanczos", "--no-paper",
                 "--no-variance", "--no-pcg", "--no-kohler"):
        assert flag in out.stdout, flag
