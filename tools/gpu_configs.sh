# BASELINE configs 2 and 3 through bench.py (stencil 256^2x64 L2-cold; physics IJK / KIJ)
mkdir -p gpurun_out
for args in "--workload stencil" "--workload physics --physics-mode 0" "--workload physics --layout kij --physics-mode 1" "--workload physics --layout kij --physics-mode 0"; do
  timeout 300 python bench.py $args --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$args', round(d['ms_per_step']*1e3,2), 'us', '%.3e' % d['value'], 'frac', round(d['roofline']['frac'],3), 'achieved', round(d['roofline']['achieved']), 'launches', d.get('gpu_launches'))"
done
