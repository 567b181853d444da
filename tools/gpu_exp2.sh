timeout 120 python tools/pair_small.py 100 37 58; echo small=$?
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "pair or golden or random" 2>&1 | tail -1 | cut -c1-200
echo "== pconv"; timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"
echo "== no pconv"; HFTW_LIBRARY=$PWD/tools/exp/nopconv.so timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"
