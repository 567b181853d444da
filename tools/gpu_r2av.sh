#!/bin/bash
# torchrun protocol check (2 ranks time-slicing one GPU) with the weak companion
cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 6 --warmup 3 > gpurun_out/bench_n2_r2av.json 2> gpurun_out/bench_n2_r2av.err; echo "torchrun n2 rc $?"
python -c "import json; d=json.load(open('gpurun_out/bench_n2_r2av.json')); print(d['n_gpus'], d['scaling'], d['ms_per_step'], d['config']['workload']); print(d.get('weak_companion'))"
tail -3 gpurun_out/bench_n2_r2av.err
