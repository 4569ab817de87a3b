mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lanczos.py tests/test_gpu_paper.py -q -x > gpurun_out/pytest_lz.log 2>&1; echo pytest rc $? >> gpurun_out/pytest_lz.log
for c in "planck store" "fullsky store" "stress store" "medium store"; do timeout 300 python scripts/lanczos_probe.py $c 2>&1 | tail -1; done > gpurun_out/lz_probe.txt
for c in "planck store" "fullsky store"; do KCG_LIB_PATH=paper_2204_08057_b200/lib/libkroncg_trace.so timeout 300 python scripts/lz_trace_probe.py $c 2>&1 | tail -2; done > gpurun_out/lz_trace.txt
