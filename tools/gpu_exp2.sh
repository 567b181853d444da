for ch in 8 12 16 20; do echo "== chunk $ch"; HFTW_PAIR_CHUNK=$ch timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"; done
