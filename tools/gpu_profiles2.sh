# ncu --set full of the config (2)/(3) kernels and the KIJ full step (one launch each)
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none -k regex:physics_column -s 3 -c 1 -o gpurun_out/prof_phys_ijk $B --workload physics --physics-mode 0 > /dev/null 2>&1; echo a=$?
timeout 600 ncu --set full --clock-control none -k regex:physics_kij_stream -s 3 -c 1 -o gpurun_out/prof_phys_kij $B --workload physics --layout kij --physics-mode 1 > /dev/null 2>&1; echo b=$?
timeout 600 ncu --set full --clock-control none -k regex:step_tma -s 8 -c 1 -o gpurun_out/prof_stencil $B --workload stencil > /dev/null 2>&1; echo c=$?
timeout 600 ncu --set full --clock-control none -k regex:step_tma -s 3 -c 1 -o gpurun_out/prof_kij_full $B --layout kij --kernel fused_tma > /dev/null 2>&1; echo d=$?
