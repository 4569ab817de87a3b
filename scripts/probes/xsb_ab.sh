# A/B of the single x buffer (K = 4 CG tile): main lib vs -DKCG_XSB=0, fullsky and planck, twice each
F="--no-cpu-baseline --no-slab-probe --no-lanczos --no-paper --no-variance --no-pcg --no-kohler --no-hs --no-planck --no-small --e2e-steps 1"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "fullsky or planck or medium or tiny or edge" > gpurun_out/ab_pytest.log 2>&1; tail -2 gpurun_out/ab_pytest.log
for r in 1 2; do
for v in main xsb0; do
  if [ $v = main ]; then L=""; else L=$PWD/paper_2204_08057_b200/lib/variants/xsb0.so; fi
  for cfg in fullsky planck; do
    KCG_LIB_PATH=$L timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 $F 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', '$cfg', round(d['value'],3), round(d['ms_per_step'],3), d['roofline']['frac'], d['clocks']['sm_mhz'])"
  done
done
done > gpurun_out/ab_xsb.txt 2>&1
cat gpurun_out/ab_xsb.txt
