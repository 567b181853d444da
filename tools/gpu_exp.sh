run() { echo -n "$* $EXTRA : "; env "$@" timeout 120 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline $EXTRA | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f ms  frac %.3f %s' % (d['ms_per_step'], d['roofline']['frac'], d['config']['kernel']))"; }
for f in hftw torch none; do EXTRA="--workload stencil --flush $f"; run X=1; done
for ch in 4 7 8 16; do EXTRA="--workload stencil"; run HFTW_CHUNK=$ch HFTW_TX=32; done
EXTRA="--workload stencil"; run HFTW_NS=4
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,gpc__cycles_elapsed.max,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/stencil_launches.csv python bench.py --workload stencil --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
grep step_tma gpurun_out/stencil_launches.csv | tail -8 | cut -c1-20,150-400
