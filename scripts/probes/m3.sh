timeout 600 python -m pytest tests/test_gpu_d2.py tests/test_gpu_paper.py -x -q > gpurun_out/m6_pytest.log 2>&1
timeout 120 python scripts/probes/d2_cg_probe.py planck > gpurun_out/m6_probe.log 2>&1
timeout 200 python scripts/probes/d2_cg_probe.py fullsky >> gpurun_out/m6_probe.log 2>&1
timeout 60 python scripts/probes/d2_one.py planck kron > gpurun_out/m6_plain.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:march -s 0 -c 1 -o gpurun_out/prof_march6_k4 python scripts/probes/d2_one.py planck kron 10 > gpurun_out/m6_ncu.log 2>&1
tail -3 gpurun_out/m6_pytest.log
