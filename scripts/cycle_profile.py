"""Cycle accounting of the fused kernel (needs a -DNDGI_PROFILE=1 build in NDGI_LIB)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ndgi_synth as S  # noqa: E402
import paper_2604_12625_b200 as ndgi  # noqa: E402

lay, seed = S.config("c2")
ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, seed)), 0)
TS = [i / 24 for i in range(24)]
out = torch.empty((24, ctx.full_texels() * 4), dtype=torch.uint8, device="cuda")
for _ in range(3):
    ndgi.ndgi_decode_full_batch(ctx, TS, out)
torch.cuda.synchronize()
buf = np.zeros(12, np.uint64)
ndgi._lib.ndgi_debug_fused_profile(buf.ctypes.data_as(C.c_void_p), 1)
ndgi.ndgi_decode_full_batch(ctx, TS, out)
torch.cuda.synchronize()
ndgi._lib.ndgi_debug_fused_profile(buf.ctypes.data_as(C.c_void_p), 0)
names = ["barrier", "mbar_wait", "epilogue", "gather", "output", "prologue", "total", "steps", "loops", "issue(w0)"]
tot = float(buf[6])
for n, v in zip(names, buf[:10]):
    print(f"{n:10s} {int(v):16d} {v / tot * 100:6.1f}%")
print("max resident CTAs/SM:", int(buf[10]), " mean resident at CTA start:", float(buf[11]) / 1184)
print("warp-0 issue cycles per layer:", float(buf[9]) / (float(buf[7]) / 4) / 3)
print("cycles per warp-step:", {n: round(float(v) / float(buf[7]), 1) for n, v in zip(names[:9], buf[:9]) if n != 'steps'})
