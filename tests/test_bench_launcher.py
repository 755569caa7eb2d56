"""bench.py's multi-GPU entry point on CPU (`--gpus N` must spawn
the ranks itself).

`python bench.py --gpus 2` outside torchrun starts two ranks through
torch.distributed.run (127.0.0.1 rendezvous); here with the gloo backend and
the CPU stand-in decoder (bench.StubDecoder), so the whole sharded flow runs
without a GPU: k % N shard of a config-4-style scene, the timed loop with
barriers and MAX over ranks, the communicator checks, and the verification
(all_gather of every tile's digest vs rank 0's decode of the whole scene).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra, timeout=300):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo", "--stub",
           "--steps", "3", "--warmup", "3", "--scene-tiles", "64", "--no-weak", *extra]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)


def test_bench_spawns_ranks_and_verifies_shards():
    r = _run()
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout               # rank 0 alone prints the line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["comm"]["comm_nranks_ok"] and d["comm"]["gpus_active"] == 2
    assert d["verify"]["ok"] and d["verify"]["digest_mismatches_vs_single_gpu"] == 0
    assert d["verify"]["tiles"] == 64
    assert d["value"] > 0 and d["steps"] == 3


def test_bench_world_mismatch_is_loud():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--stub"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
