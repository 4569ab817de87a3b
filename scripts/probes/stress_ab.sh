F="--no-cpu-baseline --no-slab-probe --no-lanczos --no-paper --no-variance --no-pcg --no-kohler --no-hs --no-planck --no-small --e2e-steps 1"
for r in 1 2; do for v in main fuse0; do if [ $v = main ]; then L=""; else L=$PWD/paper_2204_08057_b200/lib/variants/$v.so; fi
KCG_LIB_PATH=$L timeout 300 python bench.py --config stress --steps 3 --warmup 3 $F 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print('$v', 'stress', round(d['value'],4), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done; done
