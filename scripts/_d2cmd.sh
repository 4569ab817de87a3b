mkdir -p gpurun_out
for c in "6 1 2 0" "8 2 1 1"; do CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/_d2case.py $c 2>&1 | grep -E "OK|Error" | tail -1; echo "case $c done"; done > gpurun_out/d2cases.txt 2>&1
