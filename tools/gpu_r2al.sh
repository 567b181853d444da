#!/bin/bash
# DRAM bytes of a pair pass vs unit height (how much of the read excess is j-restart re-reads)
cd $GRAFT_REPO_ROOT
for c in "24 12" "48 24" "96 48" "12 6"; do set -- $c
  HFTW_LIBRARY=tools/exp/tune.so HFTW_PAIR_CHUNK=$1 HFTW_PAIR_CHUNK2=$2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:step_pair -s 2 -c 1 python tools/ab_step.py 20 2>/dev/null | grep -E "duration|dram__bytes|hit_rate" | awk -v c="$1" '{print "chunk " c ": " $1 " " $(NF-1) " " $NF}'
done
