"""Small fused-kernel launches for compute-sanitizer (memcheck / racecheck /
synccheck): config 1 decode_full RGBA8 (FULL8), decode_tiles n = 1 (4-row
strips, TILES8) and n = 4, the H profile (windowed F_uvt) through both, and a
wide border (both mirrors).  usage: compute-sanitizer --tool X python scripts/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ndgi_synth as S  # noqa: E402
import paper_2604_12625_b200 as ndgi  # noqa: E402

for name, lay in (("c1-M", S.config("c1")[0]), ("c1-H", S.layout(1, 2, 2, "H", uvt_depth=4, line_t=4)),
                  ("c1-M-B64", S.layout(1, 2, 2, "M", border=64, uvt_depth=4, line_t=4))):
    ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, 3, "mixed")), 0)
    C = lay["core"]
    P = C + 2 * lay["border"]
    out = torch.zeros((1, 2 * C, 2 * C, 4), dtype=torch.uint8, device="cuda")
    ndgi.ndgi_decode_full(ctx, 0.3, out, "rgba8", "fast")
    for n in (1, 4):
        ids = torch.arange(n, dtype=torch.int32, device="cuda")
        cache = torch.zeros((n, P, P, 4), dtype=torch.uint8, device="cuda")
        ndgi.ndgi_decode_tiles(ctx, ids, None, n, n, 0.6, cache, "rgba8", "fast")
        c32 = torch.zeros((n, P, P, 4), dtype=torch.float32, device="cuda")
        ndgi.ndgi_decode_tiles(ctx, ids, None, n, n, 0.6, c32, "rgba32f", "fast")
    torch.cuda.synchronize()
    assert ndgi.ndgi_device_error(ctx) == 0
    print(name, "ok", flush=True)
