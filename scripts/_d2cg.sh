mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_d2.py tests/test_gpu_paper.py -q > gpurun_out/pytest_d2.log 2>&1; echo rc $? >> gpurun_out/pytest_d2.log
timeout 300 python scripts/d2_cg_probe.py planck > gpurun_out/d2cg.txt 2>&1
