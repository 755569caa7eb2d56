"""SURVEY §8(e) VT sharding on one GPU: a frame's requests split by the owner
rule (k % N, parallel.local_requests) and decoded by rank g from its own shard
of Theta give exactly the bytes a single context holding the whole scene gives
for the same tiles; and bench.py's sharded VT leg runs (rank 0 of a simulated
2-rank group, element-wise max = identity)."""
import numpy as np
import pytest

import ndgi_synth as S

pytestmark = pytest.mark.gpu


def test_shard_decode_equals_whole_scene():
    import torch

    import paper_2604_12625_b200 as ndgi
    from paper_2604_12625_b200 import parallel as par
    lay = S.layout(1, 8, 8, "M")
    seed = 4000
    whole = ndgi.ndgi_load(lay, ndgi.upload_theta(S.make_theta(lay, seed)), 0)
    for world in (2, 3):
        for rank in range(world):
            mine = par.shard_tiles(lay["num_tiles"], world, rank)
            sub = dict(lay, num_tiles=len(mine), atlases=1, tiles_x=len(mine), tiles_y=1)
            shard = ndgi.ndgi_load(sub, ndgi.upload_theta(S.make_theta(sub, seed, tiles=mine)), 0)
            for ids, t in S.vt_batches(lay["num_tiles"], 16, 3, seed):
                pos, loc = par.local_requests(ids, world, rank)
                if len(pos) == 0:
                    continue
                got = torch.empty((len(pos), 136, 136, 4), dtype=torch.uint8, device="cuda")
                exp = torch.empty_like(got)
                ndgi.ndgi_decode_tiles(shard, torch.from_numpy(loc.astype(np.int32)).cuda(), None, len(pos), len(pos),
                                       t, got)
                ndgi.ndgi_decode_tiles(whole, torch.from_numpy(ids[pos].astype(np.int32)).cuda(), None, len(pos),
                                       len(pos), t, exp)
                torch.cuda.synchronize()
                assert torch.equal(got, exp), (world, rank, t)


class _OneRankOfTwo:
    """rank 0 of a 2-rank group whose other rank reports the same times"""
    class ReduceOp:
        MAX = "max"

    @staticmethod
    def all_reduce(t, op=None):
        return t


def test_bench_vt_sharded_leg_runs():
    import bench
    from paper_2604_12625_b200 import parallel as par
    lay = S.layout(1, 16, 8, "M")
    dec = bench.NdgiDecoder(0)
    ids = par.shard_tiles(lay["num_tiles"], 2, 0)
    ctx, theta = dec.load(bench._local_layout(len(ids)), 4000, ids)
    res = bench.vt_sharded_leg(dec, _OneRankOfTwo, 0, 2, ctx, lay["num_tiles"])
    for n in ("8", "32"):
        assert "error" not in res[n], res[n]
        assert 0 < res[n]["device_p50"] <= res[n]["device_p99"] < 1e4
    assert "512" not in res                                  # more requests than tiles: skipped
