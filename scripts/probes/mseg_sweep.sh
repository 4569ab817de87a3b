# D2 march: segment rows (KCG_MSEG override) on the paper workload, fullsky-d2 and planck-d2 (Kronecker route)
mkdir -p gpurun_out
for sg in model 96 128 160 208 256 352; do
  if [ $sg = model ]; then unset KCG_MSEG; else export KCG_MSEG=$sg; fi
  timeout 300 python scripts/probes/paper_routes_probe.py 2>&1 | grep kron | sed "s/^/seg=$sg paper /"
done > gpurun_out/mseg_sweep.txt 2>&1
for sg in model 32 48 64 80 112 160; do
  if [ $sg = model ]; then unset KCG_MSEG; else export KCG_MSEG=$sg; fi
  for cfg in fullsky planck; do timeout 300 python scripts/probes/d2_cg_probe.py $cfg 2>&1 | grep kron | sed "s/^/seg=$sg $cfg /"; done
done >> gpurun_out/mseg_sweep.txt 2>&1
cat gpurun_out/mseg_sweep.txt
