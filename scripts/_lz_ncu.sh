mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lanczos_kernel -s 2 -c 1 -o gpurun_out/prof_lz_planck python scripts/lanczos_probe.py planck store > gpurun_out/ncu_lz.log 2>&1; echo rc $? >> gpurun_out/ncu_lz.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lanczos_kernel -s 1 -c 1 -o gpurun_out/prof_lz_fullsky python scripts/lanczos_probe.py fullsky store > gpurun_out/ncu_lz2.log 2>&1; echo rc $? >> gpurun_out/ncu_lz2.log
