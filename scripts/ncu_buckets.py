"""Buckets the fused kernel's executed warp-instructions by how often each SASS
instruction runs (per step / per chunk / per unit / once) from an ncu source
page (sass) CSV; prints per-texel counts and the opcode mix of each bucket.
usage: ncu_buckets.py src.csv[.gz] [evaluated_texels] [items_per_step]"""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
hdr = rows[1]
ix = hdr.index("Instructions Executed")
samp = hdr.index("Warp Stall Sampling (All Samples)")
texels = float(sys.argv[2]) if len(sys.argv) > 2 else 402653184
S = int(sys.argv[3]) if len(sys.argv) > 3 else 2
warp_items = texels / 32
steps = warp_items / S
buckets = collections.OrderedDict((k, collections.Counter()) for k in ("step", "sub-step", "chunk", "unit", "rare"))
samples = collections.Counter()
total = 0
for r in rows[2:]:
    if len(r) <= ix or not r[0].startswith("0x"):
        continue
    ex = int(r[ix] or 0)
    if ex == 0:
        continue
    total += ex
    op = r[1].split()[0] if r[1].split() else "?"
    if op.startswith("@"):
        op = r[1].split()[1]
    op = op.split(".")[0]
    k = ex / steps
    b = "step" if k >= 0.9 else ("sub-step" if k >= 0.3 else ("chunk" if k >= 0.05 else ("unit" if k >= 0.004 else "rare")))
    buckets[b][op] += ex
    samples[b] += int(r[samp] or 0)
print(f"total warp-instructions {total:.4g} = {total / warp_items:.1f} per texel (per thread-item)")
ts = sum(samples.values()) or 1
for b, c in buckets.items():
    n = sum(c.values())
    mix = ", ".join(f"{o} {v / warp_items:.1f}" for o, v in c.most_common(14))
    print(f"[{b}] {n / warp_items:.1f} per texel, stall samples {100 * samples[b] / ts:.1f}%: {mix}")
