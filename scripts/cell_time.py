"""Gtexel/s of config-5 cells (decode_full_batch, 24 t, RGBA8, L2 flushed), median of 10."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import statistics  # noqa: E402

import torch  # noqa: E402

import ndgi_synth as S  # noqa: E402
import paper_2604_12625_b200 as ndgi  # noqa: E402

TS = [i / 24 for i in range(24)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
for cell in sys.argv[1].split(","):
    lay, seed = S.config(cell) if cell != "c2" else S.config("c2")
    ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, seed)), 0)
    out = torch.empty((24, ctx.full_texels() * 4), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ndgi.ndgi_decode_full_batch(ctx, TS, out)
    ms = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ndgi.ndgi_decode_full_batch(ctx, TS, out)
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    res.append(f"{cell} {ctx.full_texels() * 24 / (statistics.median(ms) * 1e-3) / 1e9:.2f}")
    del ctx
print("  ".join(res))
