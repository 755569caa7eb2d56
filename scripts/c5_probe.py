"""decode_full_batch of one config-5 cell (c2's 1,024-tile atlas, 24 times,
RGBA8) a few times: the launch scripts/round_capture.sh profiles for H / M.64."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ndgi_synth as S  # noqa: E402
import paper_2604_12625_b200 as ndgi  # noqa: E402

lay, seed = S.config(sys.argv[1])
ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, seed)), 0)
out = torch.empty((24, ctx.full_texels() * 4), dtype=torch.uint8, device="cuda")
for _ in range(5):
    ndgi.ndgi_decode_full_batch(ctx, [i / 24 for i in range(24)], out)
torch.cuda.synchronize()
print("ok")
