mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nested.py -q -x > gpurun_out/pytest_nested.log 2>&1; echo rc $? >> gpurun_out/pytest_nested.log
