mkdir -p gpurun_out
for G in 2 8; do KCG_LIB_PATH=paper_2204_08057_b200/lib/variants/trace.so timeout 300 python scripts/trace_slab.py $G; done > gpurun_out/trace_slab.txt 2>&1
KCG_LIB_PATH=paper_2204_08057_b200/lib/variants/trace.so timeout 300 python scripts/trace_probe.py planck 100 kron >> gpurun_out/trace_slab.txt 2>&1
