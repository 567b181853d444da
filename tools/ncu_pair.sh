# one ncu --set full capture of the pair kernel at ASUCA size
mkdir -p gpurun_out
TAG=${1:-pair}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_pair -s 2 -c 1 -o gpurun_out/prof_$TAG python tools/pair_time.py > gpurun_out/ncu_$TAG.log 2>&1; tail -3 gpurun_out/ncu_$TAG.log
