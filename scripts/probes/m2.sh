set -x
timeout 60 python scripts/probes/d2_one.py planck kron > gpurun_out/m2_plain.log 2>&1 && \
timeout 60 python scripts/probes/d2_one.py planck sylvester >> gpurun_out/m2_plain.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:march -s 0 -c 1 -o gpurun_out/prof_march_k4 python scripts/probes/d2_one.py planck kron 10 > gpurun_out/m2_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:march -s 0 -c 1 -o gpurun_out/prof_march_k1 python scripts/probes/d2_one.py planck sylvester 10 >> gpurun_out/m2_ncu.log 2>&1
tail -3 gpurun_out/m2_ncu.log
for rs in 2 4 8; do KCG_LIB_PATH=$PWD/paper_2204_08057_b200/lib/libkroncg_trace.so KCG_RES_RS=$rs timeout 60 python scripts/probes/res_trace_probe.py medium 100; done > gpurun_out/m2_res_trace.log 2>&1
KCG_LIB_PATH=$PWD/paper_2204_08057_b200/lib/libkroncg_trace.so timeout 60 python scripts/probes/res_trace_probe.py tiny 100 >> gpurun_out/m2_res_trace.log 2>&1
timeout 300 python -m pytest tests/test_gpu_resident.py -x -q > gpurun_out/m2_pytest.log 2>&1
