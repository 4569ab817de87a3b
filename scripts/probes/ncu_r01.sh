set -x
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches rc $?
timeout 300 $B > gpurun_out/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cg_persistent -s 3 -c 1 -o gpurun_out/prof_fullsky $B > gpurun_out/ncu_full.log 2>&1; echo full rc $?
ls -la gpurun_out
