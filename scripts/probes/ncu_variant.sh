# usage: bash scripts/ncu_variant.sh <variant> <config> <tag>
v=$1; cfg=$2; tag=$3
export KCG_LIB_PATH=paper_2204_08057_b200/lib/variants/$v.so
B="python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 300 $B > gpurun_out/plain_$tag.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cg_(persistent|march)" -s 3 -c 1 -o gpurun_out/prof_$tag $B > gpurun_out/ncu_$tag.log 2>&1; echo ncu rc $?
