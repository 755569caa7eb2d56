"""A fine-tuning step (config 2: 1,024 tiles x 4,096 samples) and a shading frame
(1920x1080 over config-3-like tiles), a few times each: the launches
scripts/prof_aux.sh profiles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ndgi_synth as S  # noqa: E402
import paper_2604_12625_b200 as ndgi  # noqa: E402

what = sys.argv[1]
if what == "train":
    lay, seed = S.config("c2")
    ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, seed)), 0)
    tr = ndgi.Trainer(ctx)
    tiles = list(range(lay["num_tiles"]))
    smp, tgt = S.train_batch(tiles, 4096, 12)
    ids = torch.tensor(tiles, dtype=torch.int32, device="cuda")
    smp_t, tgt_t = torch.from_numpy(smp).cuda(), torch.from_numpy(tgt).cuda()
    for _ in range(5):
        tr.step(ids, smp_t, tgt_t, 1e-3)
    torch.cuda.synchronize()
else:
    lay = S.layout(1, 16, 9, "M")
    cap = 144
    cache = torch.from_numpy(S.page_cache_bytes(cap, 128, 4, 7)).cuda()
    ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, 1)), 0)
    pt = torch.tensor(np.stack([np.arange(144), np.zeros(144)], 1).astype(np.int32)).cuda()
    ys, xs = np.mgrid[0:1080, 0:1920]
    uv = torch.from_numpy(np.stack([(xs.ravel() + 0.5) / 1920, (ys.ravel() + 0.5) / 1080], 1).astype(np.float32)).cuda()
    n = uv.shape[0]
    out = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    g, times, means = S.hdr_params(1, 25, 3)
    hdr = ndgi.make_hdr(g, times, means)
    for _ in range(5):
        ndgi.ndgi_sample_lighting(ctx, pt, 0, cache, cap, uv, None, n, 0.4, hdr, out)
    torch.cuda.synchronize()
print("ok")
