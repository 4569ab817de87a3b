# Round-end evidence: GPU tests, smoke, bench line, ncu launch list of the bench command, ncu full
# captures of the CG kernel (fullsky) and the block-Lanczos kernel (fullsky, store mode).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $? >> gpurun_out/pytest_gpu.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc $? >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $? >> gpurun_out/bench.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-slab-probe --e2e-steps 1 --no-paper"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches rc $? >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cg_persistent -s 3 -c 1 -o gpurun_out/prof_fullsky $B --no-lanczos --no-pcg --no-kohler --no-variance > gpurun_out/ncu_full.log 2>&1; echo full rc $? >> gpurun_out/ncu_full.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lanczos_kernel -s 2 -c 1 -o gpurun_out/prof_lz_fullsky python scripts/lanczos_probe.py fullsky store > gpurun_out/ncu_lz.log 2>&1; echo lz rc $? >> gpurun_out/ncu_lz.log
ls -la gpurun_out
