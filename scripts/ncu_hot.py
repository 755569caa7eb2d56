"""Summarise an ncu report's SASS source page: hottest instructions by warp-stall
samples, instruction mix and executed warp-instructions (usage: ncu_hot.py rep [N])."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
tot_s = sum(int(d["Warp Stall Sampling (All Samples)"]) for d in data)
tot_i = sum(int(d["Instructions Executed"]) for d in data)
print(f"samples {tot_s}  warp-instructions executed {tot_i}")
mix = collections.Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    mix[op.split(".")[0]] += int(d["Instructions Executed"])
print("instruction mix (warp-instr):", ", ".join(f"{k}:{v}" for k, v in mix.most_common(25)))
print("hottest:")
for i, d in enumerate(sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"]))[:n]):
    print(f'{d["Warp Stall Sampling (All Samples)"]:>7} {d["Instructions Executed"]:>10}  {d["Address"][-5:]} {d["Source"].strip()[:90]}')
