"""Config 5 sweep: decoder width x feature format (BC7, and
BC3 / BC1 with BC5 line maps (R29), u8, f16) on config 2's
atlas (1,024 tiles), decode_full at 24 times per call, RGBA8.  For every cell:
written Gtexel/s, kernel ms, the ALU roofline fraction (2h GELU activations per
texel against the measured rate of the kernel's own GELU epilogue), the HBM fraction of the algorithmic bytes,
and sampled parity against the C oracle.  Prints one JSON object.

    python scripts/sweep.py [--steps K]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import ndgi_synth as S  # noqa: E402
import oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--samples", type=int, default=200)
args = ap.parse_args()

import torch  # noqa: E402

import paper_2604_12625_b200 as ndgi  # noqa: E402

peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
def gelu_roof(h):
    """measured rate of the kernel's own GELU epilogue (its MUFU / FMA split, packing)"""
    m, fp32 = ndgi.ndgi_debug_gelu_split(h)
    ms_g, acts = ndgi.ndgi_debug_gelu_rate(2048, m, fp32)
    return acts / (ms_g * 1e-3), m


ROOF = {h: gelu_roof(h) for h in (16, 64)}
TS = [i / 24 for i in range(24)]
out = {"gelu_rate_act_per_s": {str(h): r for h, (r, _) in ROOF.items()},
       "gelu_mufu_pairs_of_16": {str(h): m for h, (_, m) in ROOF.items()}, "cells": []}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for prof in ("L", "M", "H", "M64"):
    for fmt in ("bc7", "bc3", "bc1", "u8", "f16"):
        lay, seed = S.config(f"c5:{prof}:{fmt}")
        th = S.make_theta(lay, seed)
        ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(th), 0)
        per_t = ctx.full_texels()
        o = torch.empty((24, per_t * 4), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            ndgi.ndgi_decode_full_batch(ctx, TS, o)
        ms = []
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ndgi.ndgi_decode_full_batch(ctx, TS, o)
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        kms = float(np.median(ms))
        texels = per_t * 24
        h = lay["hidden"]
        # sampled parity (RGBA32F) against the oracle, texel by texel
        o32 = torch.empty((1, per_t * 4), dtype=torch.float32, device="cuda")
        ndgi.ndgi_decode_full(ctx, TS[7], o32, "rgba32f")
        y = o32.view(1, 32 * 128, 32 * 128, 4).cpu().numpy()[0]
        M = oracle.Model(lay, th)
        rng = np.random.default_rng(5)
        errs = []
        for _ in range(args.samples):
            k = int(rng.integers(0, 1024))
            i, j = (int(v) for v in rng.integers(0, 128, 2))
            e = M.texel(k, i + 4, j + 4, TS[7])
            errs.append(np.abs(y[(k // 32) * 128 + j, (k % 32) * 128 + i, :3] - e))
        errs = np.array(errs)
        theta_t = S.theta_bytes(lay)
        alg_bytes = 24 * (1024 * (theta_t / lay["uvt_depth"] * 0 + 0) + per_t * 4)
        # Theta bytes read at one t: F_uv + 2 slices + 2x2 line rows + MLP
        def b2(f, rx, ry, nc):
            if f in ("bc7", "bc3", "bc1"):
                return (rx // 4) * (ry // 4) * (8 if f == "bc1" else 16)
            return rx * ry * nc * (1 if f == "u8" else 2)
        # one line-map row: U texels x 2 channels, or (BC5) its whole 4-row block row
        row_b = {"u8": 2 * lay["line_res"], "f16": 4 * lay["line_res"], "bc5": 4 * lay["line_res"]}[lay["fmt_line"]]
        read_t = (b2(lay["fmt_uv"], 128, 128, 4) + 2 * b2(lay["fmt_uvt"], lay["uvt_res"], lay["uvt_res"], 4)
                  + 2 * 2 * row_b + 2 * (16 * h + h + h * h + h + 3 * h + 3))
        alg_bytes = 24 * 1024 * (read_t + 128 * 128 * 4)
        cell = {"profile": prof, "fmt": fmt, "hidden": h, "gtexel_s": texels / (kms * 1e-3) / 1e9, "ms_per_24t": kms,
                "alu_frac": texels * 2 * h / (kms * 1e-3) / ROOF[h][0],
                "hbm_frac": alg_bytes / (kms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                "parity_max_abs": float(errs.max()), "parity_mean_abs": float(errs.mean()),
                "theta_bytes_per_tile": theta_t}
        out["cells"].append(cell)
        print(json.dumps(cell), file=sys.stderr, flush=True)
        del ctx
print(json.dumps(out))
