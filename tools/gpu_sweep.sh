# Tile / pipeline sweep of the TMA kernel (env knobs HFTW_TX, HFTW_NS, HFTW_CHUNK).
run() { echo -n "$* : "; env "$@" timeout 120 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline $EXTRA | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f ms  frac %.3f' % (d['ms_per_step'], d['roofline']['frac']))"; }
EXTRA=""
for tx in 64 32; do for ns in 5 7 8 12; do for ch in 16 32 64; do run HFTW_TX=$tx HFTW_NS=$ns HFTW_CHUNK=$ch; done; done; done
EXTRA="--workload stencil"
for tx in 64 32; do for ch in 2 4 8 16; do run HFTW_TX=$tx HFTW_CHUNK=$ch; done; done
