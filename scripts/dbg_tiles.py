import sys; sys.path.insert(0, '.')
import numpy as np, torch
import ndgi_synth as S
import paper_2604_12625_b200 as ndgi
lay, seed = S.config("c1")
th = ndgi.upload_theta(S.make_theta(lay, seed))
ctx = ndgi.ndgi_load(lay, th, 0)
for n in (5, 1, 64, 3000):
    ids = torch.tensor([k % 4 for k in range(n)], dtype=torch.int32, device="cuda")
    for fmt, dt in (("rgba32f", torch.float32), ("rgba8", torch.uint8)):
        out = torch.zeros((n, 136, 136, 4), dtype=dt, device="cuda")
        try:
            ndgi.ndgi_decode_tiles(ctx, ids, None, n, n, 0.3, out, fmt, "fast")
            torch.cuda.synchronize()
            print(n, fmt, "ok")
        except Exception as e:
            print(n, fmt, "FAIL", e)
