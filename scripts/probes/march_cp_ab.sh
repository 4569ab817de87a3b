# D2 row march, K = 4, columns per lane: D2 / paper tests on each variant, then the paper workload
# (paper_routes_probe) and fullsky-d2 / planck-d2 (d2_cg_probe) for main and every variant, twice.
# usage: march_cp_ab.sh VARIANT...
mkdir -p gpurun_out
for v in "$@"; do
  L=$PWD/paper_2204_08057_b200/lib/variants/$v.so
  echo "== tests $v"; KCG_LIB_PATH=$L timeout 900 python -m pytest tests/test_gpu_d2.py tests/test_gpu_paper.py -x -q 2>&1 | tail -2
done > gpurun_out/march_cp_tests.txt 2>&1
for r in 1 2; do
  for v in main "$@"; do
    if [ $v = main ]; then L=""; else L=$PWD/paper_2204_08057_b200/lib/variants/$v.so; fi
    KCG_LIB_PATH=$L timeout 300 python scripts/probes/paper_routes_probe.py 2>&1 | sed "s/^/$v paper /"
    for cfg in fullsky planck; do KCG_LIB_PATH=$L timeout 300 python scripts/probes/d2_cg_probe.py $cfg 2>&1 | grep kron | sed "s/^/$v $cfg /"; done
  done
done > gpurun_out/march_cp_ab.txt 2>&1
cat gpurun_out/march_cp_tests.txt gpurun_out/march_cp_ab.txt
