# full ncu captures on the stress config (L = 11, k = 6) at the final round-2 code: the CG tile kernel (second launch of the
# Kronecker leg) and the block-Lanczos kernel (ncu's -k matches the base name, without template arguments)
mkdir -p gpurun_out
B="python bench.py --config stress --steps 1 --warmup 3 --no-cpu-baseline --no-slab-probe --no-paper --no-small --no-planck --no-variance --no-pcg --no-kohler --no-hs --e2e-steps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cg_persistent" -s 1 -c 1 -o gpurun_out/r2i_prof_stress_cg $B > gpurun_out/r2i_ncu_stress_cg.log 2>&1; echo cg rc $?
if [ "$1" = all ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lanczos_kernel" -s 1 -c 1 -o gpurun_out/r2i_prof_stress_lz $B > gpurun_out/r2i_ncu_stress_lz.log 2>&1; echo lz rc $?
fi
