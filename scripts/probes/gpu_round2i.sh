#!/bin/bash
# Round-2 evidence (i), final code (8-row D2 apply tiles, one-predicate march stores): GPU tests, smoke, the default bench,
# the ncu launch list of the bench command, full captures of the CG tile kernel (fullsky) and of the
# D2 row-march kernel (paper workload).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2i_pytest_gpu.log 2>&1; echo pytest rc $?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo bench rc $?
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-slab-probe --e2e-steps 1"
timeout 900 $B > gpurun_out/r2i_bench_short.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_launches.csv $B > gpurun_out/r2i_ncu_launch.log 2>&1; echo launches rc $?
timeout 900 python scripts/probes/paper_kron_one.py > gpurun_out/r2i_paper_kron_one.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march -s 0 -c 1 -o gpurun_out/r2i_prof_march_paper python scripts/probes/paper_kron_one.py > gpurun_out/r2i_ncu_march.log 2>&1; echo march rc $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cg_persistent" -s 3 -c 1 -o gpurun_out/r2i_prof_fullsky $B > gpurun_out/r2i_ncu_full.log 2>&1; echo ncu full rc $?
tail -3 gpurun_out/r2i_pytest_gpu.log
