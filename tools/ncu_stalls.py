"""Headline metrics and warp-stall ratios of the kernels in an ncu report.
usage: ncu_stalls.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
WANT = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sector_hit_rate.pct"]
for v in rows[2:]:
    d = dict(zip(h, v))
    print(d.get("Kernel Name", "")[:90])
    for k in WANT:
        print(f"  {k} {d.get(k)}")
    st = [(float(x), k) for k, x in d.items()
          if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")
          and x not in ("", "n/a")]
    for x, k in sorted(st, reverse=True)[:8]:
        print(f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {x:.3f}")
