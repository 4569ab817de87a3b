mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $? >> gpurun_out/pytest_gpu.log
for r in 1 2; do for v in xpf noxpf; do for c in "planck 200 kron" "planck 100 sylvester" "fullsky 40 kron" "fullsky 40 sylvester" "stress 60 kron"; do
    KCG_LIB_PATH=paper_2204_08057_b200/lib/variants/$v.so timeout 200 python scripts/kernel_probe.py $c 2>&1 | tail -1
done; done; done > gpurun_out/probe.txt 2>&1
