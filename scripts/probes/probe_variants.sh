for v in "$@"; do
  for c in "fullsky 60" "planck 200"; do
    KCG_LIB_PATH=paper_2204_08057_b200/lib/variants/$v.so timeout 200 python scripts/kernel_probe.py $c kron 2>&1 | tail -1
  done
  KCG_LIB_PATH=paper_2204_08057_b200/lib/variants/$v.so timeout 200 python scripts/kernel_probe.py fullsky 60 sylvester 2>&1 | tail -1
done
