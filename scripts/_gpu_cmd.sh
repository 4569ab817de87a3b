mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $? >> gpurun_out/pytest_gpu.log
for c in "planck 200 kron" "fullsky 40 kron" "fullsky 40 sylvester"; do
    timeout 200 python scripts/kernel_probe.py $c 2>&1 | tail -1
done > gpurun_out/probe.txt 2>&1
