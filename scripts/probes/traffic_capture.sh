# DRAM bytes per launch of the dominant kernels of each bench leg (ncu, DRAM metrics only, the profiled
# solve of scripts/probes/solve_once.py); csv per leg under gpurun_out/traffic_*.csv
set -x
mkdir -p gpurun_out
for cr in "planck kron" "planck sylvester" "planck lanczos" "fullsky hs" "fullsky kohler" "fullsky variance" "fullsky lanczos" "paper sylvester" "fullsky pcg" "fullsky sylvester"; do
  set -- $cr
  timeout 300 python scripts/probes/solve_once.py $1 $2 > gpurun_out/traffic_$1_$2.plain 2>&1 || continue
  timeout 900 ncu --profile-from-start off --clock-control none -k regex:"cg_|march|lanczos|lz_" \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    python scripts/probes/solve_once.py $1 $2 > gpurun_out/traffic_$1_$2.csv 2> gpurun_out/traffic_$1_$2.err
done
ls -la gpurun_out | grep traffic
