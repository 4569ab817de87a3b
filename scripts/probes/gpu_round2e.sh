#!/bin/bash
# Round-2 evidence (e): GPU tests, smoke, the default bench, the ncu launch list of the bench command.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2e_pytest_gpu.log 2>&1; echo pytest rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo bench rc $?
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-slab-probe --e2e-steps 1"
timeout 900 $B > gpurun_out/r2e_bench_short.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_launches.csv $B > gpurun_out/r2e_ncu_launch.log 2>&1; echo launches rc $?
tail -3 gpurun_out/r2e_pytest_gpu.log
