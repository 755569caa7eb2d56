"""Per-step SASS region accounting of the fused kernel's hot loop from an ncu
source page (sass): instructions executed once or more per step, cut at the
TMEM / barrier / MUFU / store markers.
usage: ncu -i rep --page source --csv --print-source sass > x.csv; ncu_regions.py x.csv [texels] [items_per_step]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))[2:]
texels = float(sys.argv[2]) if len(sys.argv) > 2 else 402653184
S = int(sys.argv[3]) if len(sys.argv) > 3 else 2
steps = texels / 32 / S
tot = seg = 0.0
marks = ("BAR.SYNC", "STTM", "LDTM", "UTCBAR", "STG", "TRYWAIT", "LDS.128")
for r in rows:
    if len(r) < 6 or not r[0].startswith("0x"):
        continue
    ex = int(r[5] or 0)
    if ex < steps * 0.9:
        continue
    k = ex / steps
    tot += k
    seg += k
    op = r[1].strip()
    if any(m in op for m in marks):
        print(f"{r[0][-5:]} {op[:56]:56s} seg {seg:6.1f} cum {tot:6.1f}")
        seg = 0.0
print(f"hot instructions per step {tot:.1f}, per warp-row {tot / S:.1f}")
