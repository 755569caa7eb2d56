#!/bin/bash
# host-side cost of ndgi_decode_tiles: C harness vs the Python binding
cd "$(dirname "$0")/.."
gcc -O2 scripts/host_overhead.c -Iinclude -I/usr/local/cuda/include -Lpaper_2604_12625_b200 -lndgi \
    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2604_12625_b200 -o /tmp/host_overhead
/tmp/host_overhead
python - <<'PY'
import time, torch, numpy as np, sys
sys.path.insert(0, ".")
import ndgi_synth as S, paper_2604_12625_b200 as ndgi
lay = S.layout(1, 8, 8, "M")
ctx = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, 1)), 0)
ids = torch.tensor([0, 9, 18, 27, 36, 45, 54, 63], dtype=torch.int32, device="cuda")
cache = torch.empty((8, 136, 136, 4), dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()
for _ in range(100):
    ndgi.ndgi_decode_tiles(ctx, ids, None, 8, 8, 0.3, cache, "rgba8", "fast", st)
torch.cuda.synchronize()
N = 5000
host = done = 0.0
for _ in range(N):
    t0 = time.perf_counter()
    ndgi.ndgi_decode_tiles(ctx, ids, None, 8, 8, 0.3, cache, "rgba8", "fast", st)
    t1 = time.perf_counter()
    st.synchronize()
    t2 = time.perf_counter()
    host += t1 - t0
    done += t2 - t0
print({"python_host_us_per_call": host / N * 1e6, "python_call_to_done_us": done / N * 1e6})
PY
