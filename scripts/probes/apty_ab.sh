# D2 apply / residual kernel tile rows (KCG_AP_TYD2 = 4 vs 8 (main)): paper workload wall - loop, then the D2 / paper GPU tests on the variant
mkdir -p gpurun_out
V=$PWD/paper_2204_08057_b200/lib/variants/apty4.so
for r in 1 2; do
  for v in main apty4; do
    if [ $v = main ]; then L=""; else L=$V; fi
    KCG_LIB_PATH=$L timeout 300 python scripts/probes/paper_routes_probe.py 2>&1 | grep -E "kron|sylv|lanc" | sed "s/^/$v paper /"
  done
done > gpurun_out/apty_ab.txt 2>&1
KCG_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_d2.py tests/test_gpu_paper.py -q -m gpu > gpurun_out/apty_pytest.log 2>&1; echo pytest rc $? >> gpurun_out/apty_ab.txt
cat gpurun_out/apty_ab.txt; tail -3 gpurun_out/apty_pytest.log
