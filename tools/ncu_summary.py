#!/usr/bin/env python3
"""Summarise an ncu report into profiles/: key metrics as JSON + markdown.

usage: python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep profiles/<name> \
           [--key full/ijk/fused_tma] [--alg-bytes N]
Also records dram read+write bytes per launch in profiles/ncu_traffic.json
under --key so bench.py can report roofline.traffic.
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpc__cycles_elapsed.max",
    "sm__cycles_active.avg", "sm__cycles_active.max", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors_srcunit_ltcfabric.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (u, v)
        launches.append(d)
    return launches


def num(d, k):
    if k not in d:
        return None
    u, v = d[k]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * UNIT_SCALE.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--key")
    ap.add_argument("--alg-bytes", type=float)
    ap.add_argument("--note", default="")
    ap.add_argument("--steps-per-launch", type=float, default=1.0,
                    help="a multi-step launch: ncu_traffic.json stores the traffic per step")
    a = ap.parse_args()
    L = raw(a.rep)
    summ = []
    for d in L:
        s = {"kernel": d.get("Kernel Name", ("", ""))[1][:160]}
        for k in KEYS:
            s[k] = num(d, k)
        rd, wr, t = s["dram__bytes_read.sum"], s["dram__bytes_write.sum"], s["gpu__time_duration.sum"]
        if rd is not None and wr is not None:
            s["dram_bytes_total"] = rd + wr
            if t:
                s["dram_GBps"] = (rd + wr) / t / 1e9
        if a.alg_bytes:
            s["algorithmic_bytes"] = a.alg_bytes
            if t:
                s["algorithmic_GBps"] = a.alg_bytes / t / 1e9
            if rd is not None:
                s["traffic_over_algorithmic"] = (rd + wr) / a.alg_bytes
        summ.append(s)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out + ".json", "w") as f:
        json.dump({"report": os.path.basename(a.rep), "note": a.note, "launches": summ}, f, indent=1)
    with open(a.out + ".md", "w") as f:
        f.write(f"# {os.path.basename(a.out)}\n\n{a.note}\n\n")
        for s in summ:
            f.write(f"## {s['kernel']}\n\n| metric | value |\n|---|---|\n")
            for k, v in s.items():
                if k != "kernel":
                    f.write(f"| {k} | {v:.6g} |\n" if isinstance(v, float) else f"| {k} | {v} |\n")
            f.write("\n")
    if a.key and summ and summ[0].get("dram_bytes_total"):
        path = os.path.join(os.path.dirname(a.out) or ".", "ncu_traffic.json")
        d = json.load(open(path)) if os.path.exists(path) else {}
        d[a.key] = summ[0]["dram_bytes_total"] / a.steps_per_launch
        json.dump(d, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(summ[0], indent=1))


if __name__ == "__main__":
    main()
