# Session re-entry check: smoke, GPU tests, default bench line, launch list.
TAG=${1:-chk}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; head -c 3000 gpurun_out/bench_default_$TAG.json; echo
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 | head -c 1500; echo
