#!/bin/bash
# die-aware unit order: each die's SMs take the units of one half of the strips first
cd $GRAFT_REPO_ROOT
HFTW_LIBRARY=tools/exp/dies.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "pair or headline" 2>&1 | tail -1
for v in base dies base dies base dies; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300; done
for v in base dies; do
  HFTW_LIBRARY=tools/exp/$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_ltcfabric.sum --clock-control none -k regex:step_pair -s 2 -c 1 python tools/ab_step.py 20 2>/dev/null | grep -E "duration|dram__bytes|hit_rate|fabric" | awk -v c="$v" '{print c ": " $1 " " $(NF-1) " " $NF}'
done
