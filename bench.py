"""bench.py -- NDGI temporal-lightmap decode on B200 (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    torchrun --nproc-per-node N ... bench.py --gpus N ...   (one rank per GPU)

Workload (BASELINE.json configs[1]): one 4096^2
lightmap atlas = 32 x 32 NDGI tiles of 128^2, profile M (F_uvt 32^2x12x4,
h = 16; Table 1/3), BC7 F_uv / F_uvt, u8 line maps, f16 MLP; synthetic seeded
Theta.  One step = decode_full at the 24 hourly bake times t_i = i/24
= 24 x 16.78 M written texels, RGBA8, in one launch of the fused kernel.
Multi-GPU (--gpus N > 1; spawns N ranks itself when not under torchrun):
config 4 -- the 16,384-tile scene sharded k % N (strong scaling), each rank
decoding its shard with no communication; the step time is the max over
ranks; NCCL verifies every tile's digest against a single-GPU decode off the
timed path; the c2 weak-scaling number (1,024 tiles per rank) is a secondary
key.

Reported: value = written Gtexel/s (whole job); roofline of the fused kernel
(ALU-bound: its GELU activations/s against the measured rate of its own GELU
epilogue -- the compiled MUFU / FMA-pipe split -- plus HBM and tensor
fractions); cpu_baseline = the plain C
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
    """DRAM bytes (read + write) per launch of the bench's fused-kernel launch
    from the committed `ncu --set full` capture (profiles/roofline_traffic.json
    names the summary file it was read from)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
        return {"dram_bytes_per_launch": d["dram_bytes_per_launch"], "source": d["source"]}
    except Exception:
        return None


def _workload_config(world: int, tiles_per_rank: int, workload: str = "c2") -> dict:
    if workload == "c4":
        desc = ("c4: FarmLand-scale scene, 4 x 8192^2 atlases = 16384 NDGI-M tiles of 128^2 (BC7 F_uv/F_uvt, u8 "
                "lines, f16 MLP h=16) sharded k % N over the GPUs (strong scaling), decoded at 24 times t=i/24 per "
                "step (decode_full into each rank's compact atlas, RGBA8)")
    else:
        desc = ("c2: 4096^2 lightmap atlas (32x32 NDGI-M tiles of 128^2, BC7 F_uv/F_uvt, u8 lines, "
                "f16 MLP h=16) decoded at 24 times t=i/24 per step (decode_full, RGBA8)"
                + ("" if world == 1 else f"; weak scaling: {tiles_per_rank} tiles per GPU"))
    return {
        "workload": desc,
        "tiles_per_gpu": tiles_per_rank, "times_per_step": N_T, "core": 128, "profile": "M",
        "written_texels_per_step": (16384 if workload == "c4" else tiles_per_rank * world) * 128 * 128 * N_T,
        "scene_tiles": 16384 if workload == "c4" else tiles_per_rank * world,
        "parallelism": f"tile-sharded x{world} (k % N)",
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
        if self.index < 0:             # no GPU (launcher test)
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # let nvidia-smi start up (its first queries disturb the GPU) before
            # the caller's timed region begins
            t0 = time.time()
            while not self.lines and time.time() - t0 < 2.0:
                time.sleep(0.01)
            time.sleep(0.05)
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
def cpu_oracle_rate(lay, seed, target_s=8.0, max_tiles=512):
    """The oracle as it stands on this host's cores: a bounded
    sample of the bench workload (padded c2 tiles at one time, ~target_s s) on
    all threads and a smaller one on 1 thread, plus config 1 decoded in full
    ("CPU oracle in seconds", BASELINE config 1) on all threads and on 1."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    th = S.make_theta(lay, seed, tiles=list(range(max_tiles)))
    sub = dict(lay, num_tiles=max_tiles, atlases=1, tiles_x=max_tiles, tiles_y=1)
    M = oracle.Model(sub, th)
    t0 = time.perf_counter()
    M.decode_tiles([0], TS[7], nthreads=1)                # calibration: one padded tile, 1 thread
    per_tile_1 = time.perf_counter() - t0
    ntiles = int(max(cores, min(max_tiles, target_s * cores / max(per_tile_1, 1e-6))))
    t0 = time.perf_counter()
    M.decode_tiles(list(range(ntiles)), TS[13], nthreads=cores)
    dt = time.perf_counter() - t0
    texels = ntiles * 136 * 136
    n1 = int(max(1, min(16, 3.0 / max(per_tile_1, 1e-6))))
    t0 = time.perf_counter()
    M.decode_tiles(list(range(n1)), TS[13], nthreads=1)
    dt1 = time.perf_counter() - t0
    lay1, seed1 = S.config("c1")
    M1 = oracle.Model(lay1, S.make_theta(lay1, seed1))
    t0 = time.perf_counter()
    M1.decode_full(0.3, nthreads=cores)
    c1_n = time.perf_counter() - t0
    t0 = time.perf_counter()
    M1.decode_full(0.3, nthreads=1)
    c1_1 = time.perf_counter() - t0
    c1_texels = lay1["num_tiles"] * 128 * 128
    return {"value": texels / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{ntiles} padded 136^2 tiles of c2 at t=13/24 ({texels} texels), fp64 C oracle, "
                      f"{cores} threads, {dt:.2f} s",
            "value_1thread": n1 * 136 * 136 / dt1 / 1e9,
            "sample_1thread": f"{n1} padded tiles of c2 at t=13/24, 1 thread, {dt1:.2f} s",
            "config1_full": {"texels": c1_texels, "t": 0.3, "seconds": c1_n, "threads": cores,
                             "seconds_1thread": c1_1, "gtexel_s": c1_texels / c1_n / 1e9,
                             "gtexel_s_1thread": c1_texels / c1_1 / 1e9,
                             "what": "config 1 (256^2 lightmap, 2x2 tiles, D=T=4) decode_full at t=0.3, in full"}}


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
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _workload_config(1, 1024) if world == 1 else _workload_config(world, 16384 // world, "c4"),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": "per step one padded 136^2 tile of c2 at one of the 24 times (fp64 C oracle)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- decoders
class NdgiDecoder:
    """The product path: libndgi.so through the Python binding (C ABI)."""
    stub = False

    def __init__(self, dev):
        import torch

        import paper_2604_12625_b200 as ndgi
        self.torch, self.ndgi, self.dev = torch, ndgi, dev
        torch.cuda.set_device(dev)
        self.device = torch.device("cuda", dev)
        self.stream = torch.cuda.current_stream()

    def load(self, lay, seed, ids):
        theta = self.ndgi.upload_theta(S.make_theta(lay, seed, tiles=ids), self.dev)
        return self.ndgi.ndgi_load(lay, theta, self.dev), theta

    def decode(self, ctx, ts, out):
        self.ndgi.ndgi_decode_full_batch(ctx, ts, out, "rgba8", "fast", self.stream)

    def sync(self):
        self.torch.cuda.synchronize()

    def timer(self):
        torch = self.torch
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        return (lambda: a.record(self.stream)), (lambda: b.record(self.stream)), (lambda: a.elapsed_time(b))


class StubDecoder:
    """CPU stand-in for the launcher / sharding test (tests/test_bench_launcher.py):
    deterministic bytes per (global tile id, t), no CUDA.  Not a product path."""
    stub = True

    def __init__(self, dev):
        import torch
        self.torch, self.dev, self.device = torch, dev, torch.device("cpu")

    def load(self, lay, seed, ids):
        return {"lay": lay, "ids": np.asarray(ids, np.int64), "seed": seed}, None

    def decode(self, ctx, ts, out):
        torch = self.torch
        lay, ids = ctx["lay"], torch.from_numpy(ctx["ids"])
        C = lay["core"]
        tx, ty = lay["tiles_x"], lay["tiles_y"] * lay["atlases"]
        pix = torch.arange(C * C * 4, dtype=torch.int64)
        for i, t in enumerate(ts):
            tiles = ((ids[:, None] * 2654435761 + pix[None, :] * 40503 + int(t * 1e6) + ctx["seed"]) >> 7) & 255
            img = tiles.to(torch.uint8).view(ty, tx, C, C, 4).permute(0, 2, 1, 3, 4).reshape(-1)
            out[i].copy_(img)

    def sync(self):
        pass

    def timer(self):
        box = {}
        return (lambda: box.__setitem__("a", time.perf_counter())), \
               (lambda: box.__setitem__("b", time.perf_counter())), (lambda: (box["b"] - box["a"]) * 1e3)


def _local_layout(n_loc: int) -> dict:
    """Compact atlas for a rank's shard: 64 tiles wide when the shard allows it."""
    tx = 64 if n_loc % 64 == 0 else n_loc
    return S.layout(1, tx, n_loc // tx, "M")


def _tiles_of(img, lay):
    """[atlas image bytes] -> [tile][C][C][4] in tile-id order of the layout."""
    C = lay["core"]
    return img.view(lay["tiles_y"], C, lay["tiles_x"], C, 4).permute(0, 2, 1, 3, 4).reshape(-1, C, C, 4)


def timed_decode(dec, ctx, out, args, dist, flush):
    """W warm-ups, then K steps each bracketed by device events (L2 flushed in
    between, outside the events); barrier + sync on both sides; MAX over ranks.
    Returns (ms per step, per-step ms list, clocks summary)."""
    for _ in range(args.warmup):
        if flush is not None:
            flush.zero_()
        dec.decode(ctx, TS, out)
    dec.sync()
    timers = [dec.timer() for _ in range(args.steps)]
    if dist:
        dist.barrier()
    dec.sync()
    with ClockSampler(dec.dev if not dec.stub else -1) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()                  # L2 flush between timed steps (outside the events)
            timers[i][0]()
            dec.decode(ctx, TS, out)
            timers[i][1]()
        dec.sync()
    if dist:
        dist.barrier()
    step_ms = [tm[2]() for tm in timers]
    tot = sum(step_ms)
    if dist:
        from paper_2604_12625_b200 import parallel as par
        tot = par.max_over_ranks(tot, dist, dec.device)
    return tot / args.steps, step_ms, clk.summary()


def comm_check(dist, dec, world):
    """NCCL plumbing checks off the timed path: the communicator spans every
    rank (all_reduce of ones == N) and every rank drives a distinct GPU."""
    import torch
    one = torch.ones(1, dtype=torch.float64, device=dec.device)
    dist.all_reduce(one)
    ident = -1 if dec.stub else torch.cuda.current_device()
    uid = f"{os.uname().nodename}:{ident}:{torch.cuda.get_device_properties(ident).uuid if not dec.stub else os.getpid()}"
    names = [None] * world
    dist.all_gather_object(names, uid)
    return {"comm_nranks_ok": int(one.item()) == world == dist.get_world_size(),
            "gpus_active": len(set(names)), "devices": names}


def verify_sharded(dec, dist, rank, world, lay_loc, ids, out0, scene_lay, seed):
    """SURVEY §8(e) verification, off the timed path: every rank's per-tile
    64-bit digests at t_0 all_gathered (NCCL) into one digest per global tile;
    rank 0 decodes the WHOLE scene on its own GPU and compares every digest
    (bit-exactness across GPUs), and compares the first and last tile of every
    rank (all_gather of the bytes) with the fp64 oracle (<= 1 RGBA8 level)."""
    from paper_2604_12625_b200 import parallel as par
    n_scene = scene_lay["num_tiles"]
    tiles = _tiles_of(out0, lay_loc)
    full = par.gather_digests(ids, par.tile_digests(tiles), n_scene, dist, dec.device)
    sid, stl = par.gather_tile_sample(ids, tiles, [0, len(ids) - 1], dist, dec.device)
    res = None
    if rank == 0:
        torch = dec.torch
        ctx_all, th_all = dec.load(scene_lay, seed, np.arange(n_scene))
        C = scene_lay["core"]
        ref_out = torch.empty((1, n_scene * C * C * 4), dtype=torch.uint8, device=dec.device)
        dec.decode(ctx_all, [TS[0]], ref_out)
        dec.sync()
        ref = par.tile_digests(_tiles_of(ref_out[0], dict(scene_lay, tiles_y=scene_lay["tiles_y"] * scene_lay["atlases"])))
        ref = ref.cpu().numpy()
        mism = int((ref != full).sum())
        res = {"tiles": n_scene, "t": TS[0], "digest_mismatches_vs_single_gpu": mism,
               "how": "NCCL all_gather of per-tile digests of every rank's shard vs rank 0's decode of the whole scene"}
        ok = mism == 0
        if not dec.stub:
            import oracle
            th_s = S.make_theta(S.layout(1, 1, 1, "M"), seed, tiles=sid)
            sub = S.layout(1, len(sid), 1, "M")
            y = oracle.Model(sub, th_s).decode_tiles(list(range(len(sid))), TS[0],
                                                     nthreads=len(os.sched_getaffinity(0)))
            B_ = sub["border"]
            q = oracle.quantize_rgba8(np.ascontiguousarray(y[:, B_:B_ + C, B_:B_ + C]))
            dmax = int(np.abs(q.astype(int) - stl.astype(int)).max())
            res["oracle_sample"] = {"tiles": [int(g) for g in sid], "max_rgba8_level_diff": dmax}
            ok = ok and dmax <= 1
        res["ok"] = ok
        del ctx_all, th_all
    return res


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args, rank, world, dist):
    dev = int(os.environ.get("LOCAL_RANK", "0"))
    dec = StubDecoder(dev) if args.stub else NdgiDecoder(dev)
    torch = dec.torch
    from paper_2604_12625_b200 import parallel as par
    workload = args.workload or ("c2" if world == 1 else "c4")
    if workload == "c4":
        # config 4, strong scaling: the 16,384-tile scene sharded k % N; each
        # rank decodes its shard into a compact 64-tile-wide atlas
        scene_lay, seed = S.config("c4")
        if args.scene_tiles:                   # launcher tests: a small scene of the same kind
            scene_lay = S.layout(1, 8, args.scene_tiles // 8, "M")
        global_ids = par.shard_tiles(scene_lay["num_tiles"], world, rank)
        lay = _local_layout(len(global_ids))
    else:
        # config 2, weak scaling: every rank owns 1,024 tiles of an N x 1,024-tile scene
        lay0, seed = S.config("c2")
        scene_lay = S.layout(world, 32, 32, "M")
        global_ids = par.shard_tiles(lay0["num_tiles"] * world, world, rank)
        lay = lay0
    tiles_per_rank = len(global_ids)
    ctx, theta = dec.load(lay, seed, global_ids)
    per_t = tiles_per_rank * 128 * 128
    out = torch.empty((N_T, per_t * 4), dtype=torch.uint8, device=dec.device)
    flush = None if dec.stub else torch.empty(256 << 20, dtype=torch.uint8, device=dec.device)
    comm = comm_check(dist, dec, world) if dist else None

    ms_per_step, step_ms, clocks = timed_decode(dec, ctx, out, args, dist, flush)
    n_scene = scene_lay["num_tiles"]
    texels_per_step = n_scene * 128 * 128 * N_T           # all ranks' written texels
    value = texels_per_step / (ms_per_step * 1e-3) / 1e9

    verify, weak_c2 = None, None
    if dist is not None:
        try:
            verify = verify_sharded(dec, dist, rank, world, lay, global_ids, out[0], scene_lay, seed)
        except Exception as exc:  # pragma: no cover - reported, not hidden
            verify = {"ok": False, "error": repr(exc)}
        if workload == "c4" and not args.no_weak:
            # secondary key: config 2 weak scaling (1,024 tiles per rank), same timing rules
            lay2, seed2 = S.config("c2")
            ids2 = par.shard_tiles(1024 * world, world, rank)
            ctx2, th2 = dec.load(lay2, seed2, ids2)
            out2 = torch.empty((N_T, 1024 * 128 * 128 * 4), dtype=torch.uint8, device=dec.device)
            a2 = argparse.Namespace(**vars(args))
            a2.steps = max(3, min(args.steps, 10))
            ms2, _, _ = timed_decode(dec, ctx2, out2, a2, dist, flush)
            weak_c2 = {"workload": "c2 weak scaling: 1,024 tiles per rank of an N x 1,024-tile scene",
                       "value": 1024 * world * 128 * 128 * N_T / (ms2 * 1e-3) / 1e9, "unit": UNIT,
                       "ms_per_step": ms2, "steps": a2.steps}
            del ctx2, th2, out2

    vt_sharded = None
    if dist is not None and workload == "c4" and not args.no_vt and not dec.stub and not args.scene_tiles:
        vt_sharded = vt_sharded_leg(dec, dist, rank, world, ctx, scene_lay["num_tiles"])

    # ---------------- end to end through the host-buffer API (Theta H2D + decode + D2H)
    e2e = None
    if not dec.stub:
        try:
            e2e = e2e_leg(dec, ctx, theta, per_t, tiles_per_rank, world, dist, args)
        except Exception as exc:  # pragma: no cover - reported, not hidden
            e2e = {"value": None, "unit": UNIT, "error": repr(exc)}

    texunit = None
    if world == 1 and not args.no_texunit and not dec.stub:
        try:
            texunit = texunit_leg(dec, ctx, out, flush, args, texels_per_step, ms_per_step)
        except Exception as exc:  # pragma: no cover
            texunit = {"error": repr(exc)}

    if rank != 0:
        return
    roofline = None if dec.stub else roofline_leg(dec.ndgi, lay, tiles_per_rank, ms_per_step)
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            cpu = cpu_oracle_rate(S.config("c2")[0], S.config("c2")[1], args.cpu_seconds)
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "error": repr(exc)}
    legs = {}
    if not dec.stub:
        for name, fn, on in (("vt_batch_us", vt_latency, not args.no_vt),
                             ("shading", shading_leg, not args.no_shading and world == 1),
                             ("bc7_encode", encode_leg, not args.no_encode and world == 1),
                             ("finetune", finetune_leg, not args.no_finetune and world == 1)):
            if on:
                try:
                    legs[name] = fn(dec.ndgi, torch, args)
                except Exception as exc:  # pragma: no cover
                    legs[name] = {"error": repr(exc)}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if workload == "c4" else "weak",
        "vs_baseline": None, "dtype": "f16", "data": "synthetic",
        "config": _workload_config(world, tiles_per_rank, workload),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": 0 if dec.stub else args.steps,
        "clocks": clocks, **({"comm": comm} if comm else {}), "verify": verify, "weak_c2": weak_c2,
        "texunit": texunit, **legs, **({"vt_sharded_us": vt_sharded} if vt_sharded else {}),
        "step_ms_p50": statistics.median(step_ms), "step_ms_max": max(step_ms),
    }
    if dec.stub:
        line["stub"] = "StubDecoder (CPU launcher test, not a measurement)"
    print(json.dumps(line), flush=True)


def vt_sharded_leg(dec, dist, rank, world, ctx, n_scene):
    """VT frames served by N GPUs (parallel.split_requests):
    config 3's request stream over config 4's scene, each frame's requests split
    by the owner rule k % N; rank g decodes its share from its shard (local
    index k // N) with one ndgi_decode_tiles call.  Per frame, the device time
    of every rank's call (launches queued back to back, an event pair per
    frame) and the MAX over ranks; p50 / p99 of that max.  Every rank reaches
    the all_reduce even if its decode fails (NaN times, reported)."""
    from paper_2604_12625_b200 import parallel as par
    ndgi, torch = dec.ndgi, dec.torch
    stream = dec.stream
    res = {}
    for n in (8, 32, 128, 512):
        if n > n_scene:
            continue
        frames = S.vt_batches(n_scene, n, 16 + 64, 3000)
        times = np.full(len(frames), np.nan)
        err = None
        try:
            cache = torch.empty((n, 136, 136, 4), dtype=torch.uint8, device=dec.device)
            work = []
            for ids, t in frames:
                _, loc = par.local_requests(ids, world, rank)
                work.append((torch.from_numpy(loc.astype(np.int32)).to(dec.device), len(loc), t))
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(frames) + 1)]
            torch.cuda._sleep(int(2e-3 * 1.9e9))
            for f, (loc, m, t) in enumerate(work):
                evs[f].record(stream)
                if m:
                    ndgi.ndgi_decode_tiles(ctx, loc, None, m, n, t, cache, "rgba8", "fast", stream)
            evs[-1].record(stream)
            evs[-1].synchronize()
            times = np.array([evs[f].elapsed_time(evs[f + 1]) * 1e3 for f in range(len(frames))])
        except Exception as exc:  # pragma: no cover - reported, not hidden
            err = repr(exc)
        mx = np.sort(par.max_over_ranks_vec(times, dist, dec.device)[16:])
        res[str(n)] = {"device_p50": float(mx[len(mx) // 2]), "device_p99": float(mx[min(len(mx) - 1, int(0.99 * len(mx)))]),
                       "requests_per_rank_avg": n / world, **({"error": err} if err else {})}
    res["how"] = ("per frame: max over ranks of the device time of each rank's ndgi_decode_tiles call for its "
                  "k % N share (event pair per frame, launches queued ahead); p50/p99 over 64 frames")
    return res


def e2e_leg(dec, ctx, theta, per_t, tiles_per_rank, world, dist, args):
    """The metric end to end through the public host-buffer call: per step the
    Theta H2D copy from pinned host memory, then ndgi_decode_full_host (decode
    of time i+1 overlapped with the D2H of time i into pinned host RGBA8)."""
    torch, ndgi = dec.torch, dec.ndgi
    from paper_2604_12625_b200 import parallel as par
    n_t = N_T if tiles_per_rank * 128 * 128 * 4 * N_T <= (8 << 30) else 4   # host memory bound for c4 shards
    ts = TS[:: N_T // n_t][:n_t]
    host_theta = {k: v.cpu().pin_memory() for k, v in theta.items()}
    host_out = torch.empty((n_t, per_t * 4), dtype=torch.uint8).pin_memory()
    h2d = sum(v.numel() * v.element_size() for v in host_theta.values()) + 4 * n_t
    d2h = host_out.numel()
    e2e_steps = max(2, min(args.steps, 5))

    def e2e_step():
        for k, v in host_theta.items():
            theta[k].copy_(v, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        ndgi.ndgi_decode_full_host(ctx, ts, host_out, "rgba8", "fast")

    e2e_step()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if dist:
        e2e_s = par.max_over_ranks(e2e_s, dist, dec.device)
    return {"value": tiles_per_rank * world * 128 * 128 * n_t / e2e_s / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": e2e_steps, "times_per_step": n_t,
            "path": "ndgi_decode_full_host (pinned host RGBA8 out) + Theta H2D copy per step"
                    + ("" if n_t == N_T else f"; {n_t} of the 24 times per step (host memory)")}


def texunit_leg(dec, ctx, out, flush, args, texels_per_step, ms_per_step):
    """F_uv through the texture unit's BC7 decoder."""
    torch, ndgi = dec.torch, dec.ndgi
    stream = dec.stream

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
    return {"mode": "NDGI_MODE_FAST_TEXUNIT", "value": texels_per_step / (t_ms * 1e-3) / 1e9, "unit": UNIT,
            "ms_per_step": t_ms, "vs_software_bc7": ms_per_step / t_ms,
            "note": "same workload and output (bit-identical, tested); F_uv decoded by the texture unit"}


def _gelu_rate(ndgi, mufu_pairs, pack, iters=2048):
    ms, acts = ndgi.ndgi_debug_gelu_rate(iters, mufu_pairs, pack)
    return acts / (ms * 1e-3)


def roofline_leg(ndgi, lay, tiles_per_rank, ms_per_step):
    """Roofline of the fused kernel: T_roof = max(T_hbm, T_tc,
    T_alu); the binding one is T_alu = N_eval * 2h / R_gelu with R_gelu the
    measured rate of the kernel's own GELU epilogue (its MUFU / FMA-pipe split
    and fp32 -> f16x2 packing, ndgi_debug_gelu_split).  The step is one launch
    of the fused kernel, so its time is the kernel's average launch time."""
    peaks = _peaks()
    h = lay["hidden"]
    m_kern, fp32acc = ndgi.ndgi_debug_gelu_split(h)
    r_kern = _gelu_rate(ndgi, m_kern, fp32acc)
    r_mufu = _gelu_rate(ndgi, 16, fp32acc)
    sweep = {m: _gelu_rate(ndgi, m, fp32acc, 1024) for m in range(4, 17)}
    m_best = max(sweep, key=sweep.get)
    evaluated = tiles_per_rank * 128 * 128 * N_T               # decode_full: every written texel evaluated
    kern_s = ms_per_step * 1e-3
    achieved_act = evaluated * 2 * h / kern_s
    theta_t_bytes = tiles_per_rank * (16384 + 2 * 1024 + 2 * 2 * 64 * 2 + (16 * h + h * h + 5 * h + 3) * 2)
    alg_bytes = N_T * (theta_t_bytes + tiles_per_rank * 128 * 128 * 4)
    flops_alg = evaluated * 2 * (16 * h + h * h + 3 * h)                      # 1,120 / texel (h = 16)
    flops_issued = evaluated * 2 * (16 * h + (h + 16) * h + (h + 16) * 16)     # N padded to 16, bias chunks
    traffic = _traffic()
    return {
        "bound": "alu", "achieved": achieved_act / 1e9, "peak": r_kern / 1e9, "unit": "Gact/s",
        "frac": achieved_act / r_kern,
        "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
        "traffic_source": traffic["source"] if traffic else None,
        "kernel": f"ndgi_fused_kernel<{h},BC7,128,FULL8>",
        "per_unit": f"2h = {2 * h} GELU activations per evaluated texel; {evaluated} evaluated texels per launch",
        "gelu_formulation": {"mufu_pairs_of_16": m_kern, "fp32_accumulators": fp32acc,
                             "pack_f32_to_f16x2": fp32acc},
        "peak_source": "ndgi_debug_gelu_rate at the kernel's own MUFU/FMA split (+ fp32 packing), "
                       "148 SMs x 2048 threads, measured in this run",
        "peak_mufu_only": r_mufu / 1e9, "frac_vs_mufu_only": achieved_act / r_mufu,
        "peak_best_split": sweep[m_best] / 1e9, "best_split_mufu_pairs_of_16": m_best,
        "frac_vs_best_split": achieved_act / sweep[m_best],
        "gelu_rate_sweep_gact_s": {str(m): v / 1e9 for m, v in sweep.items()},
        "hbm_frac": alg_bytes / kern_s / 1e9 / peaks["hbm_gbs"],
        "algorithmic_bytes_per_launch": alg_bytes,
        "tensor_frac": flops_alg / kern_s / 1e12 / peaks.get("bf16_tflops_sustained", 1375.0),
        "tensor_flop_per_texel": flops_alg // evaluated,
        "tensor_frac_issued": flops_issued / kern_s / 1e12 / peaks.get("bf16_tflops_sustained", 1375.0),
        "tensor_peak": "bf16_tflops_sustained (MEASURED_PEAKS.json); f16 dense = bf16 rate",
    }


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
    # the floor: an empty kernel launched through the same binding + C-ABI path
    fl, fh = [], []
    for f in range(80):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        ndgi.ndgi_debug_null_launch(stream)
        h1 = time.perf_counter()
        e1.record(stream)
        e1.synchronize()
        if f >= 16:
            fl.append(e0.elapsed_time(e1) * 1e3)
            fh.append((h1 - h0) * 1e6)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(65)]
    torch.cuda._sleep(int(2e-3 * 1.9e9))
    for f in range(64):
        evs[f].record(stream)
        ndgi.ndgi_debug_null_launch(stream)
    evs[-1].record(stream)
    evs[-1].synchronize()
    fd = sorted(evs[f].elapsed_time(evs[f + 1]) * 1e3 for f in range(16, 64))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(2e-3 * 1.9e9))
    e0.record(stream)
    for f in range(64):
        ndgi.ndgi_debug_null_launch(stream)
    e1.record(stream)
    e1.synchronize()
    fa = e0.elapsed_time(e1) * 1e3 / 64
    res["floor"] = {"p50": statistics.median(fl), "host_call_us_p50": statistics.median(fh),
                    "device_p50": fd[len(fd) // 2], "device_avg": fa,
                    "what": "empty kernel via ndgi_debug_null_launch, events around the Python call (p50), "
                            "queued ahead with an event pair per launch (device_p50), queued ahead with no events "
                            "in between (device_avg)"}
    for n in (8, 32, 128, 512):
        batches = S.vt_batches(lay["num_tiles"], n, 16 + 64, seed)
        cache = torch.empty((n, 136, 136, 4), dtype=torch.uint8, device="cuda")
        ids = [torch.from_numpy(b[0].astype(np.int32)).cuda() for b in batches]
        # the render loop's buffers: one device id buffer, refilled per frame
        # (device-to-device, outside the timed call), one bound decoder
        idbuf = torch.empty(n, dtype=torch.int32, device="cuda")
        dec = ndgi.TileDecoder(ctx, idbuf, None, n, cache, "rgba8", "fast", stream)
        lat, host = [], []
        for f, (b, t) in enumerate(batches):
            idbuf.copy_(ids[f])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h0 = time.perf_counter()
            dec(n, t)
            h1 = time.perf_counter()
            e1.record(stream)
            e1.synchronize()
            if f >= 16:
                lat.append(e0.elapsed_time(e1) * 1e3)
                host.append((h1 - h0) * 1e6)
        lat.sort()
        host.sort()
        p50 = lat[len(lat) // 2]
        # device time per batch with the host running ahead (the renderer's case):
        # a 2 ms sleep kernel first, so every launch below is queued before the
        # GPU reaches it; events between consecutive launches
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(batches) + 1)]
        torch.cuda._sleep(int(2e-3 * 1.9e9))
        for f, (b, t) in enumerate(batches):
            evs[f].record(stream)
            ndgi.ndgi_decode_tiles(ctx, ids[f], None, n, n, t, cache, "rgba8", "fast", stream)
        evs[-1].record(stream)
        evs[-1].synchronize()
        dev = sorted(evs[f].elapsed_time(evs[f + 1]) * 1e3 for f in range(16, len(batches)))
        # the same stream of batches with no events in between (an event record
        # between launches costs ~4 us of device time itself): average per batch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(2e-3 * 1.9e9))
        e0.record(stream)
        for f, (b, t) in enumerate(batches):
            ndgi.ndgi_decode_tiles(ctx, ids[f], None, n, n, t, cache, "rgba8", "fast", stream)
        e1.record(stream)
        e1.synchronize()
        dev_avg = e0.elapsed_time(e1) * 1e3 / len(batches)
        res[str(n)] = {"p50": p50, "p99": lat[min(len(lat) - 1, int(0.99 * len(lat)))],
                       "gtexel_s": n * 136 * 136 / (p50 * 1e-6) / 1e9, "host_call_us_p50": host[len(host) // 2],
                       "device_p50": dev[len(dev) // 2], "device_p99": dev[min(len(dev) - 1, int(0.99 * len(dev)))],
                       "device_avg": dev_avg}
    res["how"] = ("p50/p99: events around the Python call of ndgi.TileDecoder (ndgi_decode_tiles bound to the "
                  "render loop's fixed id/cache buffers; host enqueue inside the events); device_p50/p99: per-batch "
                  "device time with launches queued ahead of the GPU, an event pair around each (each event record "
                  "adds ~4 us); device_avg: the same batches back to back between two events, per batch")
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


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks (one process per GPU)
    with torch.distributed.run on this node, 127.0.0.1 rendezvous."""
    import socket
    if args.backend == "nccl":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} CUDA devices are visible", file=sys.stderr)
            return 2
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # NCCL's init log (transport, NVLS) stays on, on stderr
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


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
    ap.add_argument("--no-weak", action="store_true", help="N > 1: skip the secondary c2 weak-scaling number")
    ap.add_argument("--workload", default=None, choices=["c2", "c4"],
                    help="default: c2 (1,024 tiles) at N = 1, c4 (the 16,384-tile scene sharded k % N, strong "
                         "scaling) at N > 1")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"], help="gloo: CPU launcher tests only")
    ap.add_argument("--stub", action="store_true", help="CPU stand-in decoder (launcher tests only)")
    ap.add_argument("--scene-tiles", type=int, default=0, help="c4 scene size override (launcher tests only)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world_env = os.environ.get("WORLD_SIZE")
    world = int(world_env or "1")
    rank = int(os.environ.get("RANK", "0"))
    if args.gpus > 1 and world_env is None:
        sys.exit(spawn_ranks(args))
    if world != args.gpus and args.impl != "reference":
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_mod
        if args.backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
            os.environ.setdefault("NCCL_DEBUG", "INFO")    # NCCL's init log (transports, NVLS) on stderr
        dist_mod.init_process_group(args.backend)
        dist = dist_mod
    try:
        run_gpu(args, rank, world, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
