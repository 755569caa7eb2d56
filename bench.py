"""bench.py -- NDGI temporal-lightmap decode on B200 (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N ... bench.py --gpus N ...   (one rank per GPU)

Workload (BASELINE.json configs[1]): one 4096^2
lightmap atlas = 32 x 32 NDGI tiles of 128^2, profile M (F_uvt 32^2x12x4,
h = 16; Table 1/3), BC7 F_uv / F_uvt, u8 line maps, f16 MLP; synthetic seeded
Theta.  One step = decode_full at the 24 hourly bake times t_i = i/24
= 24 x 16.78 M written texels, RGBA8, in one launch of the fused kernel.
Multi-GPU: weak scaling -- every rank owns 1024 tiles of an N x 1024-tile
scene (tile k on rank k % N) and decodes them with no communication; the
step time is the max over ranks.

Reported: value = written Gtexel/s (whole job); roofline of the fused kernel
(ALU-bound: its GELU activations/s against the measured rate of the same
GELU formulation, plus HBM and tensor fractions); cpu_baseline = the plain C
oracle on this host's cores over a bounded sample; e2e = the same metric
through ndgi_decode_full_host (Theta H2D + decode + RGBA8 D2H in the timed
region); vt_batch_us = per-batch latency of ndgi_decode_tiles for VT batches
of n random tiles of the 16,384-tile config-3 scene.
`--impl reference` times the oracle (the reference arm) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import ndgi_synth as S  # noqa: E402

METRIC = "decoded lightmap Gtexels/s"
UNIT = "Gtexel/s"
N_T = 24
TS = [i / N_T for i in range(N_T)]


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


def _traffic():
    """DRAM bytes per launch of the fused kernel from the committed ncu capture."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))["dram_bytes_per_launch"]
    except Exception:
        return None


def _workload_config(world: int, tiles_per_rank: int, workload: str = "c2") -> dict:
    if workload == "c4":
        desc = ("c4: FarmLand-scale scene, 4 x 8192^2 atlases = 16384 NDGI-M tiles of 128^2 (BC7 F_uv/F_uvt, u8 "
                "lines, f16 MLP h=16) sharded k % N over the GPUs (strong scaling), decoded at 24 times t=i/24 per "
                "step (decode_full into each rank's compact atlas, RGBA8)")
    else:
        desc = ("c2: 4096^2 lightmap atlas (32x32 NDGI-M tiles of 128^2, BC7 F_uv/F_uvt, u8 lines, "
                "f16 MLP h=16) decoded at 24 times t=i/24 per step (decode_full, RGBA8)")
    return {
        "workload": desc,
        "tiles_per_gpu": tiles_per_rank, "times_per_step": N_T, "core": 128, "profile": "M",
        "written_texels_per_step": tiles_per_rank * 128 * 128 * N_T * world,
        "scene_tiles": tiles_per_rank * world, "parallelism": f"tile-sharded x{world} (k % N)",
        "l2": f"flushed between timed steps (256 MiB write); Theta {tiles_per_rank * 36006 / 1e6:.1f} MB/GPU",
    }


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle timing
def cpu_oracle_rate(lay, seed, target_s=12.0, max_tiles=512):
    """The oracle as it stands, all host cores, bounded sample of the same workload
    (about target_s seconds of CPU work, at most max_tiles tiles)."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    th = S.make_theta(lay, seed, tiles=list(range(max_tiles)))
    sub = dict(lay, num_tiles=max_tiles, atlases=1, tiles_x=max_tiles, tiles_y=1)
    M = oracle.Model(sub, th)
    t0 = time.perf_counter()
    M.decode_tiles([0], TS[7], nthreads=cores)           # calibration: one padded tile
    dt = time.perf_counter() - t0
    per_tile = dt
    ntiles = int(max(1, min(max_tiles, target_s / max(per_tile, 1e-6))))
    t0 = time.perf_counter()
    ids = list(range(ntiles))
    M.decode_tiles(ids, TS[13], nthreads=cores)
    dt = time.perf_counter() - t0
    texels = ntiles * 136 * 136
    return {"value": texels / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{ntiles} padded 136^2 tiles of c2 at t=13/24 ({texels} texels), fp64 C oracle, "
                      f"{cores} threads, {dt:.2f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    lay, seed = S.config("c2")
    import oracle
    cores = len(os.sched_getaffinity(0))
    th = S.make_theta(lay, seed, tiles=list(range(8)))
    sub = dict(lay, num_tiles=8, atlases=1, tiles_x=8, tiles_y=1)
    M = oracle.Model(sub, th)
    # each step: one core tile (128^2 written texels) at one of the 24 times
    for w in range(args.warmup):
        M.decode_tiles([w % 8], TS[w % N_T], nthreads=cores)
    t0 = time.perf_counter()
    texels = 0
    for s in range(args.steps):
        M.decode_tiles([s % 8], TS[s % N_T], nthreads=cores)
        texels += 136 * 136
    dt = time.perf_counter() - t0
    v = texels / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": _workload_config(1, 1024),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": "per step one padded 136^2 tile of c2 at one of the 24 times (fp64 C oracle)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args, rank, world, dist):
    import torch

    import paper_2604_12625_b200 as ndgi

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    from paper_2604_12625_b200 import parallel as par
    if args.workload == "c4":
        # strong scaling of config 4: the 16384-tile scene sharded k % N; each
        # rank decodes its shard into a compact 64-tile-wide atlas
        _, seed = S.config("c4")
        scene = 16384
        tiles_per_rank = scene // world
        global_ids = par.shard_tiles(scene, world, rank)
        lay0 = S.layout(1, 64, tiles_per_rank // 64, "M")
    else:
        lay0, seed = S.config("c2")
        tiles_per_rank = lay0["num_tiles"]
        global_ids = par.shard_tiles(tiles_per_rank * world, world, rank)   # tile k on rank k % N
    th_np = S.make_theta(lay0, seed, tiles=global_ids)
    lay = dict(lay0)
    theta = ndgi.upload_theta(th_np, dev)
    ctx = ndgi.ndgi_load(lay, theta, dev)
    per_t = ctx.full_texels()
    out = torch.empty((N_T, per_t * 4), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        ndgi.ndgi_decode_full_batch(ctx, TS, out, "rgba8", "fast", stream)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for i in range(args.steps):
            flush.zero_()                      # L2 flush between timed steps (outside the events)
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    tot_ms = sum(step_ms)
    if dist:
        tot_ms = par.max_over_ranks(tot_ms, dist, "cuda")
    ms_per_step = tot_ms / args.steps
    texels_per_step = per_t * N_T * world
    value = texels_per_step / (ms_per_step * 1e-3) / 1e9

    # ---------------- SURVEY §8(e) verification of a sharded run (off the timed path):
    # the first and last local tile of every rank at t_0 gathered to all ranks
    # (NCCL all_gather) and compared on rank 0 with the oracle's own decode
    verify = None
    if dist is not None:
        try:
            Cc = lay["core"]
            n_loc = lay["num_tiles"]
            img = out[0].view(lay["tiles_y"], Cc, lay["tiles_x"], Cc, 4)
            tiles = img.permute(0, 2, 1, 3, 4).reshape(n_loc, Cc, Cc, 4)
            sid, stl = par.gather_tile_sample(global_ids, tiles, [0, n_loc - 1], dist, "cuda")
            if rank == 0:
                import oracle
                th_s = S.make_theta(lay0, seed, tiles=sid)
                sub = dict(lay0, num_tiles=len(sid), atlases=1, tiles_x=len(sid), tiles_y=1)
                y = oracle.Model(sub, th_s).decode_tiles(list(range(len(sid))), TS[0],
                                                         nthreads=len(os.sched_getaffinity(0)))
                B_ = lay0["border"]
                ref = oracle.quantize_rgba8(np.ascontiguousarray(y[:, B_:B_ + Cc, B_:B_ + Cc]))
                dmax = int(np.abs(ref.astype(int) - stl.astype(int)).max())
                verify = {"tiles": [int(g) for g in sid], "t": TS[0], "max_rgba8_level_diff_vs_oracle": dmax,
                          "ok": dmax <= 1, "how": "NCCL all_gather of 2 decoded tiles per rank, fp64 C oracle"}
        except Exception as exc:  # pragma: no cover - reported, not hidden
            verify = {"ok": False, "error": repr(exc)}

    # ---------------- end-to-end through the host-buffer API (Theta H2D + decode + D2H)
    e2e = None
    try:
        if args.workload == "c4":
            raise RuntimeError("skipped for c4: 24 GiB of pinned host output per step")
        host_theta = {k: v.cpu().pin_memory() for k, v in theta.items()}
        host_out = torch.empty((N_T, per_t * 4), dtype=torch.uint8).pin_memory()
        h2d = sum(v.numel() * v.element_size() for v in host_theta.values()) + 4 * N_T
        d2h = host_out.numel()
        e2e_steps = max(2, min(args.steps, 5))

        def e2e_step():
            for k, v in host_theta.items():
                theta[k].copy_(v, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            ndgi.ndgi_decode_full_host(ctx, TS, host_out, "rgba8", "fast")

        e2e_step()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        if dist:
            e2e_s = par.max_over_ranks(e2e_s, dist, "cuda")
        e2e = {"value": texels_per_step / e2e_s / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
               "path": "ndgi_decode_full_host (pinned host RGBA8 out) + Theta H2D copy per step"}
    except Exception as exc:  # pragma: no cover - reported, not hidden
        e2e = {"value": None, "unit": UNIT, "error": repr(exc)}

    # ---------------- F_uv through the texture unit's BC7 decoder
    texunit = None
    if world == 1 and not args.no_texunit:
        try:
            def tstep():
                ndgi.ndgi_decode_full_batch(ctx, TS, out, "rgba8", "fast_texunit", stream)
            for _ in range(3):
                flush.zero_()
                tstep()
            tms = []
            for _ in range(max(3, min(args.steps, 10))):
                flush.zero_()
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                tstep()
                b_.record(stream)
                b_.synchronize()
                tms.append(a_.elapsed_time(b_))
            t_ms = statistics.median(tms)
            texunit = {"mode": "NDGI_MODE_FAST_TEXUNIT", "value": texels_per_step / (t_ms * 1e-3) / 1e9, "unit": UNIT,
                       "ms_per_step": t_ms, "vs_software_bc7": ms_per_step / t_ms,
                       "note": "same workload and output (bit-identical, tested); F_uv decoded by the texture unit"}
        except Exception as exc:  # pragma: no cover
            texunit = {"error": repr(exc)}

    if rank != 0:
        return
    # ---------------- roofline of the fused kernel (rank 0)
    peaks = _peaks()
    ms_g, acts = ndgi.ndgi_debug_gelu_rate(4096)
    r_gelu = acts / (ms_g * 1e-3)                              # activations/s, same f16x2 GELU
    h = lay["hidden"]
    evaluated = tiles_per_rank * 128 * 128 * N_T               # decode_full: every written texel evaluated
    kern_s = ms_per_step * 1e-3                                 # one fused-kernel launch per step
    achieved_act = evaluated * 2 * h / kern_s
    theta_t_bytes = tiles_per_rank * (16384 + 2 * 1024 + 2 * 2 * 64 * 2 + 595 * 2)   # read at one t
    alg_bytes = N_T * (theta_t_bytes + tiles_per_rank * 128 * 128 * 4)
    flops = evaluated * 2 * (16 * h + (h + 16) * h + (h + 16) * 16)               # tensor work as issued
    roofline = {
        "bound": "alu", "achieved": achieved_act / 1e9, "peak": r_gelu / 1e9, "unit": "Gact/s",
        "frac": achieved_act / r_gelu, "traffic": _traffic(),
        "kernel": "ndgi_fused_kernel<16,BC7>", "per_unit": f"2h = {2 * h} GELU activations per evaluated texel",
        "peak_source": "ndgi_debug_gelu_rate: the kernel's f16x2 tanh-GELU, 148 SMs x 8 CTAs, measured in this run",
        "hbm_frac": alg_bytes / kern_s / 1e9 / peaks["hbm_gbs"],
        "tensor_frac": flops / kern_s / 1e12 / peaks.get("bf16_tflops_sustained", 1375.0),
        "algorithmic_bytes_per_launch": alg_bytes,
    }
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            cpu = cpu_oracle_rate(lay0, seed, args.cpu_seconds)
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "error": repr(exc)}
    vt = None
    if not args.no_vt:
        try:
            vt = vt_latency(ndgi, torch, args)
        except Exception as exc:  # pragma: no cover
            vt = {"error": repr(exc)}
    shading = None
    if not args.no_shading and world == 1:
        try:
            shading = shading_leg(ndgi, torch, args)
        except Exception as exc:  # pragma: no cover
            shading = {"error": repr(exc)}
    encode = None
    if not args.no_encode and world == 1:
        try:
            encode = encode_leg(ndgi, torch, args)
        except Exception as exc:  # pragma: no cover
            encode = {"error": repr(exc)}
    finetune = None
    if not args.no_finetune and world == 1:
        try:
            finetune = finetune_leg(ndgi, torch, args)
        except Exception as exc:  # pragma: no cover
            finetune = {"error": repr(exc)}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f16", "data": "synthetic", "config": _workload_config(world, tiles_per_rank, args.workload),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": args.steps,
        "clocks": clk.summary(), "vt_batch_us": vt, "shading": shading, "texunit": texunit, "bc7_encode": encode, "finetune": finetune,
        "verify": verify,
        "step_ms_p50": statistics.median(step_ms), "step_ms_max": max(step_ms),
    }
    print(json.dumps(line), flush=True)


_C3 = {}


def _c3_context(ndgi, torch):
    """Config 3's scene (16,384 tiles, 590 MB of Theta), built once per process
    for the VT and shading legs."""
    if "ctx" not in _C3:
        lay, seed = S.config("c3")
        th = ndgi.upload_theta(S.make_theta(lay, seed))
        _C3.update(lay=lay, seed=seed, th=th, ctx=ndgi.ndgi_load(lay, th, torch.cuda.current_device()))
    return _C3["lay"], _C3["seed"], _C3["ctx"]


def vt_latency(ndgi, torch, args):
    """Config 3: per-batch latency of ndgi_decode_tiles on a 16,384-tile scene."""
    lay, seed, ctx = _c3_context(ndgi, torch)
    res = {}
    stream = torch.cuda.current_stream()
    for n in (8, 32, 128, 512):
        batches = S.vt_batches(lay["num_tiles"], n, 16 + 64, seed)
        cache = torch.empty((n, 136, 136, 4), dtype=torch.uint8, device="cuda")
        ids = [torch.from_numpy(b[0].astype(np.int32)).cuda() for b in batches]
        lat, host = [], []
        for f, (b, t) in enumerate(batches):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h0 = time.perf_counter()
            ndgi.ndgi_decode_tiles(ctx, ids[f], None, n, n, t, cache, "rgba8", "fast", stream)
            h1 = time.perf_counter()
            e1.record(stream)
            e1.synchronize()
            if f >= 16:
                lat.append(e0.elapsed_time(e1) * 1e3)
                host.append((h1 - h0) * 1e6)
        lat.sort()
        host.sort()
        p50 = lat[len(lat) // 2]
        res[str(n)] = {"p50": p50, "p99": lat[min(len(lat) - 1, int(0.99 * len(lat)))],
                       "gtexel_s": n * 136 * 136 / (p50 * 1e-6) / 1e9, "host_call_us_p50": host[len(host) // 2]}
    return res


def shading_leg(ndgi, torch, args):
    """SURVEY §8(f) NEXT 1, measured: one 1920x1080 frame of coherent shading
    samples over a 16 x 9-tile window of config 3's scene (~1 texel per sample).
    (a) ndgi_sample_lighting alone, inputs resident: Gsample/s and the HBM
    fraction of its algorithmic bytes (8 B uv + 12 B out + 4 B of page cache
    per sample); (b) the VT frame loop -- ndgi_vt_request + ndgi_decode_tiles of
    the jobs + ndgi_vt_upload + sample -- for a frame whose 144 tiles all miss
    (new time bucket) and for a frame that hits."""
    lay, seed, ctx = _c3_context(ndgi, torch)
    stream = torch.cuda.current_stream()
    tx0, ty0, wx, wy = 20, 30, 16, 9
    ids = np.array([(ty0 + j) * lay["tiles_x"] + tx0 + i for j in range(wy) for i in range(wx)], np.uint32)
    cap = 256
    vt = ndgi.VT(lay["num_tiles"], cap, 96)
    cache = torch.zeros((cap, 136, 136, 4), dtype=torch.uint8, device="cuda")
    pt = torch.empty((lay["num_tiles"], 2), dtype=torch.int32, device="cuda")
    g, times, means = S.hdr_params(lay["atlases"], 25, seed)
    hdr = ndgi.make_hdr(g, times, means)
    Wt, Ht = lay["tiles_x"], lay["tiles_y"]
    ys, xs = np.mgrid[0:1080, 0:1920]
    u = (tx0 + wx * (xs.ravel() + 0.5) / 1920) / Wt
    v = (ty0 + wy * (ys.ravel() + 0.5) / 1080) / Ht
    uv = torch.from_numpy(np.stack([u, v], 1).astype(np.float32)).cuda()
    n = uv.shape[0]
    out = torch.empty((n, 3), dtype=torch.float32, device="cuda")

    def frame(t):
        jid, jsl, td, b = vt.request(ids, t)
        if len(jid):
            ndgi.ndgi_decode_tiles(ctx, torch.from_numpy(jid.astype(np.int32)).to("cuda", non_blocking=True),
                                   torch.from_numpy(jsl.astype(np.int32)).to("cuda", non_blocking=True), len(jid),
                                   cap, td, cache, "rgba8", "fast", stream)
        vt.upload(pt, stream)
        ndgi.ndgi_sample_lighting(ctx, pt, b, cache, cap, uv, None, n, t, hdr, out, stream)
        return len(jid), b

    def timed(fn, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    frame(0.40)
    b = vt.bucket(0.40)[0]
    for _ in range(3):
        ndgi.ndgi_sample_lighting(ctx, pt, b, cache, cap, uv, None, n, 0.40, hdr, out, stream)
    ks = timed(lambda: ndgi.ndgi_sample_lighting(ctx, pt, b, cache, cap, uv, None, n, 0.40, hdr, out, stream), 50)
    assert ndgi.ndgi_device_error(ctx, reset=True) == 0
    peaks = _peaks()
    alg = n * (8 + 12 + 4)
    hit_s, miss_s = [], []
    for f in range(12):
        t = 0.40 + 0.5 * f / 96                      # every other frame enters a new bucket
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        jobs, _ = frame(t)
        e1.record(stream)
        e1.synchronize()
        (miss_s if jobs else hit_s).append(e0.elapsed_time(e1) * 1e3)
    res = {
        "workload": "1920x1080 coherent samples over a 16x9-tile window of c3 (144 tiles, ~1 texel/sample), "
                    "cache 256 slots, 96 time buckets",
        "samples": n, "sample_kernel_us": ks * 1e6, "gsample_s": n / ks / 1e9,
        "roofline": {"bound": "hbm", "achieved": alg / ks / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": alg / ks / 1e9 / peaks["hbm_gbs"], "algorithmic_bytes_per_sample": 24},
        "frame_us_all_hit_p50": statistics.median(hit_s) if hit_s else None,
        "frame_us_144_miss_p50": statistics.median(miss_s) if miss_s else None,
        "vt_stats": vt.stats(),
    }
    vt.close()
    return res


def encode_leg(ndgi, torch, args):
    """SURVEY §8(f) NEXT 3, measured: ndgi_bc7_encode_mode6 on an 8192^2 RGBA8
    feature map (a smooth field with noisy rows), inputs resident; Gtexel/s of
    input texels and the HBM fraction of its 5 B/texel (4 in, 1 out)."""
    h = w = 8192
    yy = torch.arange(h, device="cuda", dtype=torch.float32)[:, None] / h
    xx = torch.arange(w, device="cuda", dtype=torch.float32)[None, :] / w
    chans = [torch.clamp(torch.round(255 * (0.5 + 0.3 * torch.sin(2 * np.pi * (a * xx + b * yy) + ph))), 0, 255)
             for a, b, ph in ((1.3, 2.1, 0.3), (0.7, 2.9, 1.1), (2.2, 0.6, 2.0), (1.9, 1.4, 4.0))]
    img = torch.stack(chans, -1).to(torch.uint8).contiguous()
    img[::7] = torch.randint(0, 256, img[::7].shape, device="cuda", dtype=torch.uint8)
    out = torch.empty(((h // 4) * (w // 4), 16), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(3):
        ndgi.ndgi_bc7_encode_mode6(img, out, stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record(stream)
    for _ in range(reps):
        ndgi.ndgi_bc7_encode_mode6(img, out, stream)
    e1.record(stream)
    e1.synchronize()
    s_ = e0.elapsed_time(e1) / reps * 1e-3
    # R31 multi-mode search (mode 6, mode 5 x 4 rotations, mode 7 x 64 partitions) on a 2048^2 crop
    hm = 2048
    crop = img[:hm, :hm].contiguous()
    outm = torch.empty(((hm // 4) * (hm // 4), 16), dtype=torch.uint8, device="cuda")
    ndgi.ndgi_bc7_encode_multi(crop, outm, stream)
    e0.record(stream)
    ndgi.ndgi_bc7_encode_multi(crop, outm, stream)
    e1.record(stream)
    e1.synchronize()
    sm = e0.elapsed_time(e1) * 1e-3
    peaks = _peaks()
    return {"workload": "8192^2 RGBA8 map (smooth field, every 7th row noise) -> BC7 mode 6",
            "multi": {"workload": "2048^2 crop of the same map -> BC7 multi-mode search (R31)", "ms": sm * 1e3,
                      "gtexel_s": hm * hm / sm / 1e9},
            "ms": s_ * 1e3, "gtexel_s": h * w / s_ / 1e9,
            "hbm": {"achieved": 5 * h * w / s_ / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": 5 * h * w / s_ / 1e9 / peaks["hbm_gbs"], "algorithmic_bytes_per_texel": 5}}


def finetune_leg(ndgi, torch, args):
    """SURVEY §8(f) NEXT 4, measured: one fine-tuning step (R27) of all 1,024
    per-tile decoders of config 2, 4,096 samples per tile (the paper's batch of
    2^12): features from the BC7 maps, forward + backward + Adam.
    samples/s, and the fraction of the fp32 FMA peak its MLP arithmetic
    (3 x the forward MACs per sample) would need."""
    lay, seed = S.config("c2")
    th = ndgi.upload_theta(S.make_theta(lay, seed))
    ctx = ndgi.ndgi_load(lay, th, torch.cuda.current_device())
    tr = ndgi.Trainer(ctx)
    tiles = list(range(lay["num_tiles"]))
    Sn = 4096
    smp, tgt = S.train_batch(tiles, Sn, 12)
    ids = torch.tensor(tiles, dtype=torch.int32, device="cuda")
    smp_t, tgt_t = torch.from_numpy(smp).cuda(), torch.from_numpy(tgt).cuda()
    stream = torch.cuda.current_stream()
    for _ in range(2):
        tr.step(ids, smp_t, tgt_t, 1e-3, None, stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record(stream)
    for _ in range(reps):
        tr.step(ids, smp_t, tgt_t, 1e-3, None, stream)
    e1.record(stream)
    e1.synchronize()
    s_ = e0.elapsed_time(e1) / reps * 1e-3
    n = len(tiles) * Sn
    h = lay["hidden"]
    flops = n * 3 * 2 * (16 * h + h * h + 3 * h)
    fma_peak = 148 * 128 * 2 * _peaks().get("sm_max_mhz", 1965.0) * 1e6 / 1e12   # TFLOP/s fp32 (nominal)
    tr.close()
    # the full step (R28): BC-simulated maps + line grids + MLP, Eq. 5 noise, projection
    P = ndgi.train_full_params(lay)
    g = torch.Generator(device="cuda").manual_seed(5)
    init = torch.rand((len(tiles), P), device="cuda", generator=g)
    init[:, :tr.P] = (init[:, :tr.P] - 0.5) * 0.6
    noise = torch.rand((len(tiles), Sn, 12), device="cuda", generator=g) - 0.5
    tf = ndgi.Trainer(ctx, full_init=init)
    for _ in range(2):
        tf.step(ids, smp_t, tgt_t, 1e-3, None, stream, noise)
    e0.record(stream)
    for _ in range(reps):
        tf.step(ids, smp_t, tgt_t, 1e-3, None, stream, noise)
    e1.record(stream)
    e1.synchronize()
    sf = e0.elapsed_time(e1) / reps * 1e-3
    tf.export_full(stream)                                     # R30 export, warm
    e0.record(stream)
    tf.export_full(stream)
    e1.record(stream)
    e1.synchronize()
    sx = e0.elapsed_time(e1) * 1e-3
    tf.close()
    ctx.close()
    return {"workload": "1024 tiles x 4096 samples (c2, BC7 features), forward + backward + Adam, h = 16",
            "ms_per_step": s_ * 1e3, "msample_s": n / s_ / 1e6,
            "mlp_tflops": flops / s_ / 1e12, "fp32_peak_tflops": fma_peak, "frac": flops / s_ / 1e12 / fma_peak,
            "full": {"workload": f"same batch, full step (R28): {P} fp32 parameters per tile "
                                 "(MLP + BC-simulated maps + line grids), Eq. 5 noise, Adam + [0,1] projection",
                     "ms_per_step": sf * 1e3, "msample_s": n / sf / 1e6,
                     "export_ms": sx * 1e3,
                     "export": "R30: Eq. 7 texels -> u8 PTQ -> BC7 mode 6 (F_uv, F_uvt), line grids -> u8, "
                               "MLP -> f16, all 1,024 tiles"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline oracle leg")
    ap.add_argument("--no-vt", action="store_true", help="skip the VT batch-latency leg")
    ap.add_argument("--no-shading", action="store_true", help="skip the shading-side (NEXT 1) leg")
    ap.add_argument("--no-texunit", action="store_true", help="skip the texture-unit F_uv comparator (NEXT 2)")
    ap.add_argument("--no-encode", action="store_true", help="skip the BC7 encoder leg (NEXT 3)")
    ap.add_argument("--no-finetune", action="store_true", help="skip the fine-tuning leg (NEXT 4)")
    ap.add_argument("--workload", default="c2", choices=["c2", "c4"],
                    help="c2: 1,024 tiles per GPU (weak scaling, default); c4: the 16,384-tile scene sharded (strong)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist_mod
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist_mod.init_process_group("nccl")
        dist = dist_mod
    try:
        run_gpu(args, rank, world, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
