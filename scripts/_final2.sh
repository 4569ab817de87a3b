mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $? >> gpurun_out/pytest_gpu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_persistent -s 2 -c 1 -o gpurun_out/prof_pcg python scripts/pcg_probe.py fullsky > gpurun_out/ncu_pcg.log 2>&1; echo rc $? >> gpurun_out/ncu_pcg.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_persistent -s 2 -c 1 -o gpurun_out/prof_syl python scripts/resid_probe.py > gpurun_out/ncu_syl.log 2>&1; echo rc $? >> gpurun_out/ncu_syl.log
