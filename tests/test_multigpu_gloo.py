"""Multi-rank host logic on CPU (gloo, world_size 2).

Checks the sharding rule (disjoint, complete, balanced), the request split of
a VT frame, the MAX-over-ranks timing reduction and the digest all_gather
used to verify a sharded decode against a single-process decode.  The decode
itself is stood in for by the oracle on a tiny layout (the GPU path is
covered by the -m gpu tests; no GPU is needed here).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ndgi_synth as S
from paper_2604_12625_b200 import parallel as par


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_rule():
    for n, world in ((16384, 8), (1024, 3), (5, 2), (7, 8)):
        shards = [par.shard_tiles(n, world, g) for g in range(world)]
        allids = np.concatenate(shards)
        assert len(allids) == n and len(set(allids.tolist())) == n
        sizes = [len(s) for s in shards]
        assert max(sizes) - min(sizes) <= 1
        for g, s in enumerate(shards):
            assert all(par.owner(k, world) == g for k in s)
    ids = np.array([5, 2, 9, 12, 3])
    parts = par.split_requests(ids, 2)
    assert sorted(np.concatenate(parts).tolist()) == list(range(5))
    assert all((ids[p] % 2 == g).all() for g, p in enumerate(parts))
    # a rank's share of a frame indexes its own shard: shard[k // N] == k
    for world in (2, 3, 8):
        frame = np.random.default_rng(world).choice(16384, 512, replace=False)
        served = []
        for g in range(world):
            pos, loc = par.local_requests(frame, world, g)
            assert (par.shard_tiles(16384, world, g)[loc] == frame[pos]).all()
            served += pos.tolist()
        assert sorted(served) == list(range(512))


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    lay = S.layout(1, 5, 1, "M", core=8, border=2, uvt_res=4, uvt_depth=2, line_res=4, line_t=3, hidden=4)
    mine = par.shard_tiles(lay["num_tiles"], world, rank)
    th = S.make_theta(lay, 77, "mixed", tiles=mine)           # this rank's Theta only
    sub = dict(lay, num_tiles=len(mine), atlases=1, tiles_x=len(mine), tiles_y=1)
    y = oracle.Model(sub, th).decode_tiles(np.arange(len(mine)), 0.4)
    q = torch.from_numpy(oracle.quantize_rgba8(y))
    dg = par.tile_digests(q)
    full = par.gather_digests(mine, dg, lay["num_tiles"], dist)
    sid, stl = par.gather_tile_sample(mine, q, [0, len(mine) - 1], dist)
    t = par.max_over_ranks(1.5 + rank, dist)
    tv = par.max_over_ranks_vec([1.0 + rank, 5.0 - rank, 2.0], dist)
    if rank == 0:
        out.put((full.tolist(), t, sid.tolist(), stl, tv.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_digests_match_single_process():
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, t, sid, stl, tv = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.5                                          # max over ranks
    assert tv == [2.0, 5.0, 2.0]                             # element-wise
    lay = S.layout(1, 5, 1, "M", core=8, border=2, uvt_res=4, uvt_depth=2, line_res=4, line_t=3, hidden=4)
    th = S.make_theta(lay, 77, "mixed")
    y = oracle.Model(lay, th).decode_tiles(np.arange(5), 0.4)
    q8 = oracle.quantize_rgba8(y)
    ref = par.tile_digests(torch.from_numpy(q8)).numpy()
    np.testing.assert_array_equal(np.array(full), ref)
    # the verification sample: first and last tile of each rank, with global ids
    assert sid == [0, 4, 1, 3]
    for g, tile in zip(sid, stl):
        np.testing.assert_array_equal(tile, q8[g])


def test_digest_detects_single_byte_change():
    a = torch.randint(0, 256, (3, 8, 8, 4), dtype=torch.uint8)
    b = a.clone()
    b[1, 3, 4, 2] ^= 1
    da, db = par.tile_digests(a), par.tile_digests(b)
    assert da[0] == db[0] and da[2] == db[2] and da[1] != db[1]
