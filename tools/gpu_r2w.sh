#!/bin/bash
# torchrun protocol check on one GPU (2 ranks time-slice it), group bench, C++ adapter tests
cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2_r2w.json 2> gpurun_out/bench_n2_r2w.err; echo "torchrun n2 rc $?"; head -c 300 gpurun_out/bench_n2_r2w.json; echo
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_g2_r2w.json 2> gpurun_out/bench_g2_r2w.err; echo "group n2 rc $? (expected: fails loudly with 1 GPU)"; tail -2 gpurun_out/bench_g2_r2w.err
timeout 600 python bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_ref_g2_r2w.json 2>&1; echo "ref n2 rc $?"; head -c 300 gpurun_out/bench_ref_g2_r2w.json; echo
timeout 900 python -m pytest tests/test_cpp_adapter.py tests/test_emit_gpu.py tests/test_no_fallback.py -q -p no:cacheprovider 2>&1 | tail -2
