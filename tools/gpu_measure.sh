# Measurement pass: default bench line, the config sweep, a 2-rank protocol check,
# and the ncu launch list of the default bench command.
TAG=${1:-m}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; cat gpurun_out/bench_default_$TAG.json | head -c 3000; echo
for args in "--workload physics --layout ijk --physics-mode 0" "--workload physics --layout kij --physics-mode 0" "--workload physics --layout kij --physics-mode 1" "--workload physics --layout ijk --physics-mode 1" "--workload stencil --layout ijk" "--workload stencil --layout kij" "--kernel split" "--kernel fused_cell" "--layout kij"; do
  echo "== $args"; timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline $args | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({k: d[k] for k in ('value','ms_per_step')}), json.dumps(d['roofline']['frac']), d['config']['kernel'])"
done
echo "== 2 ranks on one GPU (protocol check, timing meaningless)"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --e2e-steps 1 2>&1 | tail -2 | head -c 2000; echo
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; wc -l gpurun_out/launches_$TAG.csv
