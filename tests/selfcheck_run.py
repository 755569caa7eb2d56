"""Runs the self-check decode cases with whichever libndgi the environment
selects (NDGI_LIB) and saves every output: tests/test_gpu_selfcheck.py runs it
in a subprocess with the checked build and compares with the product build."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ndgi_synth as S  # noqa: E402
import paper_2604_12625_b200 as ndgi  # noqa: E402

CASES = {
    "M-mixed": (S.config("c1")[0], "mixed"),
    "M-smooth": (S.config("c1")[0], "smooth"),
    "H-mixed": (S.layout(1, 2, 2, "H", uvt_depth=4, line_t=4), "mixed"),          # windowed F_uvt
    "M-B64": (S.layout(1, 2, 2, "M", border=64, uvt_depth=4, line_t=4), "smooth"),  # both mirrors
    "L-u8": (S.layout(1, 2, 2, "L", uvt_depth=4, line_t=4, fmt_uv="u8", fmt_uvt="u8"), "smooth"),
    "M64": (S.layout(1, 2, 1, "M64", uvt_depth=4, line_t=4), "mixed"),
    "C256": (S.layout(1, 1, 1, "M", core=256, uv_res=256, uvt_depth=4, line_t=4), "smooth"),
    "bc3": (S.layout(1, 2, 1, "M", uvt_depth=4, line_t=8, fmt_uv="bc3", fmt_uvt="bc3", fmt_line="bc5"), "mixed"),
    "ring-R3=40-u8": (S.layout(1, 2, 1, "M", uvt_res=40, uvt_depth=4, line_t=4, fmt_uv="u8", fmt_uvt="u8"), "smooth"),
    "ring-R3=56-bc1": (S.layout(1, 2, 1, "M", uvt_res=56, uvt_depth=4, line_t=8, fmt_uv="bc1", fmt_uvt="bc1",
                                fmt_line="bc5"), "mixed"),
}


def run(out_path):
    res = {}
    for name, (lay, payload) in CASES.items():
        ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, 9, payload)), 0)
        C, P = lay["core"], lay["core"] + 2 * lay["border"]
        full = torch.zeros((2, lay["atlases"], lay["tiles_y"] * C, lay["tiles_x"] * C, 4), dtype=torch.uint8,
                           device="cuda")
        ndgi.ndgi_decode_full_batch(ctx, [0.3, 0.8], full, "rgba8", "fast")
        res[name + "/full8"] = full
        f32 = torch.zeros((1, lay["atlases"], lay["tiles_y"] * C, lay["tiles_x"] * C, 4), dtype=torch.float32,
                          device="cuda")
        ndgi.ndgi_decode_full(ctx, 0.55, f32, "rgba32f", "fast")
        res[name + "/full32"] = f32
        nt = lay["num_tiles"]
        for n in (1, 3, 600):                          # 4-row strips, 8/16-row strips, whole tiles
            ids = torch.tensor([(7 * i + 1) % nt for i in range(n)], dtype=torch.int32, device="cuda")
            cache = torch.zeros((n, P, P, 4), dtype=torch.uint8, device="cuda")
            ndgi.ndgi_decode_tiles(ctx, ids, None, n, n, 0.6, cache, "rgba8", "fast")
            res[f"{name}/tiles8-{n}"] = cache[:4]
        c32 = torch.zeros((2, P, P, 4), dtype=torch.float32, device="cuda")
        ndgi.ndgi_decode_tiles(ctx, torch.tensor([nt - 1, 0], dtype=torch.int32, device="cuda"), None, 2, 2, 0.15,
                               c32, "rgba32f", "fast")
        res[name + "/tiles32"] = c32
        torch.cuda.synchronize()
        assert ndgi.ndgi_device_error(ctx) == 0, name
    np.savez(out_path, **{k: v.cpu().numpy() for k, v in res.items()})


if __name__ == "__main__":
    run(sys.argv[1])
