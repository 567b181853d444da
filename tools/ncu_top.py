"""Summarise an ncu report: headline metrics, stall reasons, top source lines."""
import csv, subprocess, sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ('Duration', 'DRAM Throughput', 'Issue Slots Busy', 'Registers Per Thread', 'Executed Instructions',
        'Eligible Warps Per Scheduler', 'Warp Cycles Per Issued Instruction', 'L2 Hit Rate',
        'Achieved Active Warps Per SM', 'Dynamic Shared Memory Per Block')
for row in csv.reader(det.splitlines()):
    if len(row) > 4 and row[-4] in want:
        print(row[-4], row[-3], row[-2])
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
st = [(a.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), float(c))
      for a, c in zip(raw[0], raw[2]) if 'smsp__average_warps_issue_stalled' in a and 'per_issue_active' in a]
print("stalls:", ", ".join(f"{n} {v:.2f}" for n, v in sorted(st, key=lambda x: -x[1])[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
out = []
for r in csv.reader(src.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split('/')[-1]
        continue
    if r[0].isdigit():
        try:
            out.append((int(r[4]), int(r[7]), cur, r[0], r[1][:96]))
        except ValueError:
            pass
tw = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"-- top stall lines (samples {tw}) --")
for o in sorted(out, key=lambda x: -x[0])[:n]:
    print(f"{o[0] / tw * 100:5.1f}% {o[1] / ti * 100:5.1f}%i {o[2]}:{o[3]} {o[4]}")
