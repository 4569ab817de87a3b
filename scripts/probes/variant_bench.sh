# usage: bash scripts/variant_bench.sh <config> [variants...]
cfg=$1; shift
for v in "$@"; do
  r=$(KCG_LIB_PATH=paper_2204_08057_b200/lib/variants/$v.so timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 5 --e2e-steps 1 2>&1 | tail -1)
  echo "$v $cfg $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],3), round(d["roofline"]["achieved"]), round(d["roofline"]["frac"],3), "syl", round(d["sylvester"]["roofline"]["frac"],3))' 2>&1)"
done
