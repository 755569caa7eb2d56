"""Per-CTA residency of the bench launch (diagnostic build libndgi_res.so,
NDGI_RESIDENCY=1): SM id and %globaltimer at entry / after TMEM allocation /
exit of every CTA of one c2 decode_full_batch (24 t) -> how many CTAs each SM
runs concurrently, and when."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NDGI_LIB"] = os.path.join(ROOT, "paper_2604_12625_b200", os.environ.get("RES_LIB", "libndgi_res.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ndgi_synth as S  # noqa: E402
import paper_2604_12625_b200 as ndgi  # noqa: E402

lib = ctypes.CDLL(os.environ["NDGI_LIB"])
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
lay, seed = S.config(cfg)
ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, seed)), 0)
out = torch.empty((24, ctx.full_texels() * 4), dtype=torch.uint8, device="cuda")
for _ in range(3):
    ndgi.ndgi_decode_full_batch(ctx, [i / 24 for i in range(24)], out)
torch.cuda.synchronize()
nb = 1184
buf = (ctypes.c_ulonglong * (nb * 4))()
lib.ndgi_debug_residency(buf, nb)
a = np.array(buf[:], dtype=np.int64).reshape(nb, 4)
sm, t0, t1, t2 = a[:, 0], a[:, 1], a[:, 2], a[:, 3]
base = t0.min()
t0, t1, t2 = (t0 - base) / 1e3, (t1 - base) / 1e3, (t2 - base) / 1e3
print(f"{cfg}: kernel span {t2.max():.1f} us; entry p0/p50/p100 {np.percentile(t0, [0, 50, 100]).round(2)}; "
      f"alloc wait p50/p99/max {np.percentile(t1 - t0, [50, 99, 100]).round(2)}; exit min/p50/max "
      f"{np.percentile(t2, [0, 50, 100]).round(1)}")
ctas = np.bincount(sm, minlength=148)
print("CTAs per SM histogram:", dict(zip(*np.unique(ctas, return_counts=True))))
# concurrency over time per SM
ts = np.linspace(0, t2.max(), 200)
conc = np.zeros((148, len(ts)))
for s_, a_, b_ in zip(sm, t1, t2):
    conc[s_] += (ts >= a_) & (ts < b_)
print("mean CTAs running per SM (after alloc) over time:", conc.mean(0)[::10].round(2))
late = np.argsort(t1)[-10:]
print("latest-starting CTAs (block, sm, entry, after alloc, exit):")
for b in late:
    print(" ", b, sm[b], round(t0[b], 1), round(t1[b], 1), round(t2[b], 1))
