# D2 march with the per-pass segment plan: D2-touching tests, then the paper workload / fullsky-d2 / planck-d2 probes
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_d2.py tests/test_gpu_paper.py tests/test_gpu_warm.py tests/test_gpu_variance.py tests/test_gpu_kohler.py tests/test_gpu_nested.py -x -q > gpurun_out/mseg_auto_tests.txt 2>&1
tail -2 gpurun_out/mseg_auto_tests.txt
for r in 1 2; do
  timeout 300 python scripts/probes/paper_routes_probe.py 2>&1 | sed "s/^/paper /"
  for cfg in fullsky planck; do timeout 300 python scripts/probes/d2_cg_probe.py $cfg 2>&1 | sed "s/^/$cfg /"; done
done > gpurun_out/mseg_auto.txt 2>&1
cat gpurun_out/mseg_auto.txt
