timeout 120 python tools/pair_small.py 100 37 58 >/dev/null 2>&1; echo small=$?
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "pair" 2>&1 | tail -1 | cut -c1-200
for c2 in 16 8 4; do echo "== chunk2 $c2"; HFTW_PAIR_CHUNK2=$c2 timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"; done
