#!/bin/bash
# One gpurun call: GPU parity tests, the default bench, ncu launch list and one full capture of the CG kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-slab-probe --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches rc $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cg_persistent -s 3 -c 1 -o gpurun_out/prof_fullsky $B > gpurun_out/ncu_full.log 2>&1; echo full rc $?
ls -la gpurun_out
