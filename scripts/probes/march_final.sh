# D2 march after a geometry change: D2-touching GPU tests, then the paper workload and fullsky / planck d2 probes
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_d2.py tests/test_gpu_paper.py tests/test_gpu_warm.py tests/test_gpu_variance.py tests/test_gpu_kohler.py tests/test_gpu_hs.py tests/test_gpu_nested.py tests/test_gpu_args.py -x -q > gpurun_out/march_final_tests.txt 2>&1
tail -2 gpurun_out/march_final_tests.txt
for r in 1 2; do
  timeout 300 python scripts/probes/paper_routes_probe.py 2>&1 | sed "s/^/paper /"
  for cfg in fullsky planck; do timeout 300 python scripts/probes/d2_cg_probe.py $cfg 2>&1 | sed "s/^/$cfg /"; done
done > gpurun_out/march_final.txt 2>&1
cat gpurun_out/march_final.txt
