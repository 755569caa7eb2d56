"""Stage timeline of one VT unit (diagnostic build libndgi_tl.so, NDGI_TIMELINE=1):
block 0's %globaltimer stamps for decode_tiles batches of n tiles."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["NDGI_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                      "paper_2604_12625_b200", "libndgi_tl.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ndgi_synth as S  # noqa: E402
import paper_2604_12625_b200 as ndgi  # noqa: E402

lib = ctypes.CDLL(os.environ["NDGI_LIB"])
lay, seed = S.config("c3")
ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, seed)), 0)
names = ["start", "tmem+bar", "unit start", "weights", "prologue", "chunk start", "chunk decoded",
         "step 1", "step 2", "step 3", "step 4", "end"]
for n in (8, 32, 512):
    cache = torch.empty((n, 136, 136, 4), dtype=torch.uint8, device="cuda")
    rows = []
    for f, (ids, t) in enumerate(S.vt_batches(lay["num_tiles"], n, 12, seed)):
        ndgi.ndgi_decode_tiles(ctx, torch.from_numpy(ids.astype(np.int32)).cuda(), None, n, n, t, cache)
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * 16)()
        lib.ndgi_debug_timeline(buf)
        v = np.array(buf[:12], dtype=np.int64)
        if f >= 4:
            rows.append(v - v[0])
    m = np.median(np.array(rows), 0)
    print(n, "  ".join(f"{nm} {x / 1000:.2f}" for nm, x in zip(names, m) if x >= 0), flush=True)
