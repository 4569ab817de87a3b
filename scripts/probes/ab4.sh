# A/B of build variants against the main lib, Kronecker and Sylvester routes: fullsky and planck, twice each
# (usage: ab4.sh NAME1 NAME2 ...)
F="--no-cpu-baseline --no-slab-probe --no-lanczos --no-paper --no-variance --no-pcg --no-kohler --no-hs --no-planck --no-small --e2e-steps 1"
OUT=gpurun_out/ab4_$(echo "$@" | tr ' ' '_').txt
cat > /tmp/ab4_fmt.py <<'PY'
import json, sys
d = json.loads(sys.stdin.readline())
print(sys.argv[1], sys.argv[2], "kron", round(d["value"], 3), "syl", round(d["sylvester"]["value"], 3),
      round(d["ms_per_step"], 3), round(d["roofline"]["frac"], 4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
for r in 1 2; do
for v in main "$@"; do
  if [ $v = main ]; then L=""; else L=$PWD/paper_2204_08057_b200/lib/variants/$v.so; fi
  for cfg in fullsky planck; do
    KCG_LIB_PATH=$L timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 $F 2>/dev/null | python /tmp/ab4_fmt.py $v $cfg
  done
done
done > $OUT 2>&1
cat $OUT
