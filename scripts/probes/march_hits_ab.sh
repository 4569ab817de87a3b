# D2 march K = 4 with hits: groups per CTA / stages (paper workload), main vs variants, twice; usage: march_hits_ab.sh VARIANT...
mkdir -p gpurun_out
for r in 1 2; do
  for v in main "$@"; do
    if [ $v = main ]; then L=""; else L=$PWD/paper_2204_08057_b200/lib/variants/$v.so; fi
    KCG_LIB_PATH=$L timeout 300 python scripts/probes/paper_routes_probe.py 2>&1 | grep kron | sed "s/^/$v paper /"
  done
done > gpurun_out/march_hits_ab.txt 2>&1
cat gpurun_out/march_hits_ab.txt
