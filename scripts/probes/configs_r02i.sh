# bench lines on the other BASELINE configs at the final round-2 code
mkdir -p gpurun_out
for c in stress planck medium; do
  timeout 700 python bench.py --config $c --no-cpu-baseline --no-slab-probe --no-paper --no-small --no-planck > gpurun_out/r2i_bench_$c.json 2> gpurun_out/r2i_bench_$c.err; echo $c rc $?
done
