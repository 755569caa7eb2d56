"""Device time per decode_tiles batch vs n (launches queued ahead), and with
every id invalid (units exit at once: the launch + CTA setup cost)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ndgi_synth as S  # noqa: E402
import paper_2604_12625_b200 as ndgi  # noqa: E402

lay, seed = S.config("c3")
ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, seed)), 0)
stream = torch.cuda.current_stream()


def dev_time(n, bad=False, reps=48):
    cache = torch.empty((n, 136, 136, 4), dtype=torch.uint8, device="cuda")
    batches = S.vt_batches(lay["num_tiles"], n, reps, seed)
    ids = [torch.from_numpy((b[0].astype(np.int64) + (10 ** 6 if bad else 0)).astype(np.int32)).cuda() for b in batches]
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    torch.cuda._sleep(int(3e-3 * 1.9e9))
    for f in range(reps):
        evs[f].record(stream)
        ndgi.ndgi_decode_tiles(ctx, ids[f], None, n, n, batches[f][1], cache, "rgba8", "fast", stream)
    evs[-1].record(stream)
    evs[-1].synchronize()
    d = sorted(evs[f].elapsed_time(evs[f + 1]) * 1e3 for f in range(8, reps))
    return round(d[len(d) // 2], 2)


for n in (1, 2, 4, 8, 16, 32):
    print(n, "valid", dev_time(n), "all-invalid", dev_time(n, True), flush=True)
ndgi.ndgi_device_error(ctx, reset=True)


def probe(kind, reps=48):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    torch.cuda._sleep(int(3e-3 * 1.9e9))
    for f in range(reps):
        evs[f].record(stream)
        ndgi.ndgi_debug_launch_probe(kind, stream)
    evs[-1].record(stream)
    evs[-1].synchronize()
    d = sorted(evs[f].elapsed_time(evs[f + 1]) * 1e3 for f in range(8, reps))
    return round(d[len(d) // 2], 2)


for kind, what in ((0, "empty"), (1, "empty + fused param block"), (2, "256 CTAs + 24 KB smem"),
                   (3, "256 CTAs + TMEM alloc")):
    print(what, probe(kind), flush=True)
# and without events between launches: 48 launches between two events
for kind in (0, 1, 2, 3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(3e-3 * 1.9e9))
    e0.record(stream)
    for f in range(48):
        ndgi.ndgi_debug_launch_probe(kind, stream)
    e1.record(stream)
    e1.synchronize()
    print("no events", kind, round(e0.elapsed_time(e1) * 1e3 / 48, 2), flush=True)
