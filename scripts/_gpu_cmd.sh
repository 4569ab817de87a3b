mkdir -p gpurun_out
for r in 1 2; do for v in n512 n256; do for c in "planck 200 kron" "fullsky 40 kron"; do
    KCG_LIB_PATH=paper_2204_08057_b200/lib/variants/$v.so timeout 200 python scripts/kernel_probe.py $c 2>&1 | tail -1
done; done; done > gpurun_out/probe.txt 2>&1
