# Round evidence in one call: smoke, GPU tests, default bench line, reference arm,
# a 2-rank torchrun bench (protocol check on one GPU: ranks time-slice it), the launch
# list of the exact default bench command and one ncu --set full capture of the pair kernel.
TAG=${1:-r01g}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; echo bench=$?; head -c 600 gpurun_out/bench_default_$TAG.json; echo
timeout 300 python bench.py --impl reference > gpurun_out/bench_reference_$TAG.json 2>&1; echo ref=$?; tail -c 300 gpurun_out/bench_reference_$TAG.json; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2_$TAG.json 2> gpurun_out/bench_n2_$TAG.err; echo n2=$?; head -c 400 gpurun_out/bench_n2_$TAG.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py > gpurun_out/bench_under_ncu_$TAG.json 2>&1; echo launches=$?; wc -l gpurun_out/launches_$TAG.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_pair -s 4 -c 1 -o gpurun_out/prof_pair_$TAG python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pair_$TAG.log 2>&1; echo ncu=$?
