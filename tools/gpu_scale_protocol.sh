# bench.py under torchrun with 2/4/8 ranks on ONE GPU (time-sliced): protocol check that every
# rank count produces its JSON line (numbers are not scaling results), strong and weak
mkdir -p gpurun_out
for n in 2 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 6 --warmup 3 > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err; echo "n=$n rc=$?"; tail -c 300 gpurun_out/scale_n$n.json; echo
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus 2 --steps 4 --warmup 3 --scaling weak > gpurun_out/scale_weak2.json 2> gpurun_out/scale_weak2.err; echo "weak2 rc=$?"; tail -c 300 gpurun_out/scale_weak2.json; echo
