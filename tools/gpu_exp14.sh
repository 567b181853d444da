# physics column kernel: occupancy / batch depth A/B (bench physics workload, IJK mode 0)
for i in 1 2; do for v in head minb6 b16 b16m4 b4m8; do
  HFTW_LIBRARY=$PWD/tools/exp/$v.so timeout 200 python bench.py --workload physics --physics-mode 0 --steps 100 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,1), 'us frac', round(d['roofline']['frac'],3))"
done; done
