"""decode_tiles throughput for large VT batches (config 3 scene) vs decode_full on
the same tile count: written Gtexel/s."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ndgi_synth as S  # noqa: E402
import paper_2604_12625_b200 as ndgi  # noqa: E402

lay, seed = S.config("c3")
ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, seed)), 0)
stream = torch.cuda.current_stream()
res = {}
for n in (512, 2048, 8192):
    ids = torch.from_numpy(np.random.default_rng(n).choice(lay["num_tiles"], n, replace=False).astype(np.int32)).cuda()
    cache = torch.empty((n, 136, 136, 4), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ndgi.ndgi_decode_tiles(ctx, ids, None, n, n, 0.37, cache, "rgba8", "fast", stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        ndgi.ndgi_decode_tiles(ctx, ids, None, n, n, 0.37, cache, "rgba8", "fast", stream)
    e1.record(stream)
    e1.synchronize()
    us = e0.elapsed_time(e1) / 10 * 1e3
    res[n] = {"us": round(us, 1), "gtexel_s_written": round(n * 136 * 136 / us / 1e3, 1),
              "gtexel_s_core": round(n * 128 * 128 / us / 1e3, 1)}
print(json.dumps(res))
