"""VT batch latency (config 3) per forced strips-per-tile: for tuning choose_strips.
Run once per NDGI_STRIPS value (the library reads it once per process)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ndgi_synth as S  # noqa: E402
import paper_2604_12625_b200 as ndgi  # noqa: E402

lay, seed = S.config("c3")
ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, seed)), 0)
stream = torch.cuda.current_stream()
res = {}
for n in (8, 32, 128, 512):
    batches = S.vt_batches(lay["num_tiles"], n, 16 + 64, seed)
    cache = torch.empty((n, 136, 136, 4), dtype=torch.uint8, device="cuda")
    ids = [torch.from_numpy(b[0].astype(np.int32)).cuda() for b in batches]
    lat = []
    for f, (b, t) in enumerate(batches):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ndgi.ndgi_decode_tiles(ctx, ids[f], None, n, n, t, cache, "rgba8", "fast", stream)
        e1.record(stream)
        e1.synchronize()
        if f >= 16:
            lat.append(e0.elapsed_time(e1) * 1e3)
    lat.sort()
    res[n] = round(lat[len(lat) // 2], 1)
print(json.dumps({"strips": os.environ.get("NDGI_STRIPS", "auto"), "p50_us": res}))
