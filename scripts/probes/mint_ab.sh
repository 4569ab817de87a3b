# D2 march interior-unit step (KCG_MINT=1) vs main: paper workload twice, then the D2 / paper GPU tests on the variant
mkdir -p gpurun_out
V=$PWD/paper_2204_08057_b200/lib/variants/mint.so
for r in 1 2; do
  for v in main mint; do
    if [ $v = main ]; then L=""; else L=$V; fi
    KCG_LIB_PATH=$L timeout 300 python scripts/probes/paper_routes_probe.py 2>&1 | grep -E "kron|sylv" | sed "s/^/$v paper /"
  done
done > gpurun_out/mint_ab.txt 2>&1
for v in main mint; do
  if [ $v = main ]; then L=""; else L=$V; fi
  KCG_LIB_PATH=$L timeout 300 python scripts/probes/d2_cg_probe.py 2>&1 | grep -E "kron" | sed "s/^/$v /"
done >> gpurun_out/mint_ab.txt 2>&1
KCG_LIB_PATH=$V timeout 900 python -m pytest tests/test_gpu_d2.py tests/test_gpu_paper.py -q -m gpu > gpurun_out/mint_pytest.log 2>&1; echo pytest rc $? >> gpurun_out/mint_ab.txt
cat gpurun_out/mint_ab.txt; tail -3 gpurun_out/mint_pytest.log
