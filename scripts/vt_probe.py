"""A few VT batches of config 3 (the kernel that ncu captures in scripts/prof_vt.sh)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import ndgi_synth as S
import paper_2604_12625_b200 as ndgi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
lay, seed = S.config("c3")
ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, seed)), 0)
cache = torch.empty((n, 136, 136, 4), dtype=torch.uint8, device="cuda")
for f, (ids, t) in enumerate(S.vt_batches(lay["num_tiles"], n, 8, seed)):
    ndgi.ndgi_decode_tiles(ctx, torch.from_numpy(ids.astype(np.int32)).cuda(), None, n, n, t, cache, "rgba8", "fast")
torch.cuda.synchronize()
print("ok")
