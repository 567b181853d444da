# The round's bench lines: default (AUTO), pair kernel, single-step launches, KIJ,
# configs (2) and (3), and the reference arm.
mkdir -p gpurun_out
TAG=${1:-r01c}
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; head -c 600 gpurun_out/bench_default_$TAG.json; echo
for args in "--kernel fused_pair" "--kernel fused_tma --steps 1" "--layout kij" "--kernel split" "--workload stencil" "--workload physics --physics-mode 0" "--workload physics --layout kij --physics-mode 1"; do
  echo "== $args"; timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({k: d[k] for k in ('value','ms_per_step','gpu_launches')}), json.dumps(d['roofline']['frac']), d['roofline']['kernel'], json.dumps(d.get('kernels')))"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 | head -c 600; echo
