echo "== kg4"; HFTW_LIBRARY=$PWD/tools/exp/kg4.so timeout 300 python tools/pair_time.py 2>&1 | grep "kind 1"
echo "== kg4 chunk 24"; HFTW_PAIR_CHUNK=24 HFTW_LIBRARY=$PWD/tools/exp/kg4.so timeout 300 python tools/pair_time.py 2>&1 | grep "kind 1"
