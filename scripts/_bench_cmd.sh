mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $? >> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lanczos_kernel -s 2 -c 1 -o gpurun_out/prof_lz_fullsky python scripts/lanczos_probe.py fullsky store > gpurun_out/ncu_lz.log 2>&1; echo rc $? >> gpurun_out/ncu_lz.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lz.csv python scripts/lanczos_probe.py fullsky store > gpurun_out/ncu_lz2.log 2>&1; echo rc $? >> gpurun_out/ncu_lz2.log
