# Full check: smoke, GPU tests, default bench line, reference arm.
TAG=${1:-chk}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 | cut -c1-300
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; head -c 4000 gpurun_out/bench_default_$TAG.json; echo; tail -3 gpurun_out/bench_default_$TAG.err
