# D2 march: tests on the main build, then d2_cg_probe planck / fullsky for main and a variant (usage: d2ab.sh VARIANT)
V=$1
timeout 900 python -m pytest tests/test_gpu_d2.py tests/test_gpu_paper.py tests/test_gpu_warm.py -x -q 2>&1 | tail -2
for v in main $V; do
  if [ $v = main ]; then L=""; else L=$PWD/paper_2204_08057_b200/lib/variants/$V.so; fi
  for cfg in planck fullsky; do KCG_LIB_PATH=$L timeout 300 python scripts/probes/d2_cg_probe.py $cfg | sed "s/^/$v /"; done
done > gpurun_out/d2ab_$V.txt 2>&1
cat gpurun_out/d2ab_$V.txt
