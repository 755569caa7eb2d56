"""Per-CUDA-source-line aggregation of an ncu report (needs -lineinfo):
warp-instructions executed and stall samples per file:line, per warp-row (32 texels).
usage: ncu_lines.py report.ncu-rep [texels]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
items = (float(sys.argv[2]) if len(sys.argv) > 2 else 402653184) / 32
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout.splitlines()
cur_file = None
cur_line = None
agg = collections.defaultdict(lambda: [0, 0])
src = {}
for line in out:
    row = next(csv.reader([line]))
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if row[0] == "Line No" or row[0] == "Function Name":
        continue
    if row[0] != "":
        try:
            cur_line = int(row[0])
        except ValueError:
            continue
        src[(cur_file, cur_line)] = row[1][:70]
        continue
    if len(row) < 8 or not row[2].startswith("0x"):
        continue
    key = (cur_file, cur_line)
    agg[key][0] += int(row[7] or 0)
    agg[key][1] += int(row[4] or 0)
tot_i = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instr per warp-row {tot_i / items:.1f}; samples {tot_s}")
for key, (ni, ns) in sorted(agg.items(), key=lambda x: -x[1][0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 45]:
    print(f"{ni / items:7.2f} instr/wr  {ns / tot_s * 100:5.1f}% stall  {key[0]}:{key[1]}  {src.get(key, '').strip()}")
