#!/bin/bash
# Round-2 evidence (f): GPU tests, smoke, the default bench, the ncu launch list of the bench command,
# one full capture of the dominant CG tile kernel (fullsky).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2f_pytest_gpu.log 2>&1; echo pytest rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo bench rc $?
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-slab-probe --e2e-steps 1"
timeout 900 $B > gpurun_out/r2f_bench_short.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches.csv $B > gpurun_out/r2f_ncu_launch.log 2>&1; echo launches rc $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cg_persistent" -s 3 -c 1 -o gpurun_out/r2f_prof_fullsky $B > gpurun_out/r2f_ncu_full.log 2>&1; echo ncu full rc $?
tail -3 gpurun_out/r2f_pytest_gpu.log
