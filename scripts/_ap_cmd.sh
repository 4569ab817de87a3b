mkdir -p gpurun_out
for v in 1 3 4; do
  L=paper_2204_08057_b200/lib/libkroncg.so; [ $v != 1 ] && L=paper_2204_08057_b200/lib/libkroncg_ap$v.so
  KCG_LIB_PATH=$L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ap$v.csv python scripts/resid_probe.py > /dev/null 2>&1
  echo "minb $v"; python scripts/launch_summary.py gpurun_out/launches_ap$v.csv | grep apply
done > gpurun_out/ap.txt 2>&1
