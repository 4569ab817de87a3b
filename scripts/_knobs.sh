mkdir -p gpurun_out
for r in 1 2; do for v in default xtma4 xpf0 serp0 dyn0; do
  L=paper_2204_08057_b200/lib/libkroncg.so; [ $v != default ] && L=paper_2204_08057_b200/lib/libkroncg_$v.so
  echo -n "$v "; KCG_LIB_PATH=$L timeout 200 python scripts/pad_probe.py fullsky 2>&1 | tail -1
done; done > gpurun_out/knobs.txt 2>&1
