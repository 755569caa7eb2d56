"""Multi-GPU plumbing for the NDGI decode.

Tiles are independent models, so the path shards with no
exchange step: rank g of G owns the tiles k with k % G == g (interleaving
balances atlases), loads only its shard's Theta and decodes it locally.
torch.distributed (NCCL on the B200 box, gloo in the CPU tests) is used only
outside the hot path: a barrier before timing, MAX-reduction of the per-rank
device times, and an all_gather of per-tile digests to verify a sharded run
against a single-GPU run.  No collective runs inside the timed region.
"""
from __future__ import annotations

import numpy as np


def shard_tiles(num_tiles: int, world: int, rank: int) -> np.ndarray:
    """Global tile ids owned by `rank` (k % world == rank), ascending."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return np.arange(rank, num_tiles, world, dtype=np.int64)


def owner(tile: int, world: int) -> int:
    return int(tile) % world


def split_requests(tile_ids: np.ndarray, world: int) -> list[np.ndarray]:
    """VT streaming: a frame's request list split by the same owner rule;
    returns, per rank, the positions of the requests it serves."""
    tile_ids = np.asarray(tile_ids)
    return [np.nonzero(tile_ids % world == g)[0] for g in range(world)]


def local_requests(tile_ids: np.ndarray, world: int, rank: int) -> tuple[np.ndarray, np.ndarray]:
    """A frame's requests served by `rank`: (positions in the frame, local tile
    indices into the rank's shard).  shard_tiles(n, world, rank)[k // world] == k
    for every k owned by the rank."""
    tile_ids = np.asarray(tile_ids, dtype=np.int64)
    pos = split_requests(tile_ids, world)[rank]
    return pos, tile_ids[pos] // world


def max_over_ranks_vec(values, dist, device=None) -> np.ndarray:
    """Element-wise MAX of a per-rank float vector over the process group."""
    import torch
    t = torch.as_tensor(np.asarray(values, dtype=np.float64), device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy()


def tile_digests(tiles_u8) -> "torch.Tensor":
    """Order-independent 64-bit digest per decoded tile.

    tiles_u8: torch uint8 tensor [n][...] (any device).  The digest is a
    position-weighted sum of the bytes reinterpreted as int32 words, so two
    runs agree iff (with overwhelming probability) the tiles are bit-equal."""
    import torch
    t = tiles_u8.reshape(tiles_u8.shape[0], -1)
    w = t.view(torch.int32).to(torch.int64)
    idx = torch.arange(w.shape[1], device=w.device, dtype=torch.int64)
    mult = (idx * 2654435761 + 97531) % 2147483647
    return (w * mult).sum(dim=1)


def max_over_ranks(value: float, dist, device=None) -> float:
    """MAX of a per-rank scalar (e.g. elapsed device ms) over the process group."""
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_digests(local_ids: np.ndarray, local_digests, num_tiles: int, dist, device=None) -> np.ndarray:
    """all_gather per-rank (tile id, digest) pairs -> digest array indexed by global tile id."""
    import torch
    world = dist.get_world_size()
    n_max = -(-num_tiles // world)
    ids = torch.full((n_max,), -1, dtype=torch.int64, device=device)
    dg = torch.zeros((n_max,), dtype=torch.int64, device=device)
    ids[: len(local_ids)] = torch.as_tensor(np.asarray(local_ids), dtype=torch.int64, device=device)
    dg[: len(local_ids)] = local_digests.to(device=device, dtype=torch.int64)
    all_ids = [torch.empty_like(ids) for _ in range(world)]
    all_dg = [torch.empty_like(dg) for _ in range(world)]
    dist.all_gather(all_ids, ids)
    dist.all_gather(all_dg, dg)
    out = np.zeros(num_tiles, dtype=np.int64)
    seen = np.zeros(num_tiles, dtype=bool)
    for i_t, d_t in zip(all_ids, all_dg):
        i_np, d_np = i_t.cpu().numpy(), d_t.cpu().numpy()
        m = i_np >= 0
        out[i_np[m]] = d_np[m]
        seen[i_np[m]] = True
    if not seen.all():
        raise RuntimeError("some tiles were not decoded by any rank")
    return out


def gather_tile_sample(local_ids: np.ndarray, local_tiles, pick: list[int], dist, device=None):
    """SURVEY §8(e) verification: every rank contributes the decoded tiles at
    local positions `pick` (same count on every rank) with their global ids;
    all ranks receive them (all_gather) -> (global ids [world * len(pick)],
    tiles [world * len(pick)][...]) as numpy arrays."""
    import torch
    world = dist.get_world_size()
    ids = torch.as_tensor(np.asarray(local_ids)[pick], dtype=torch.int64, device=device)
    tl = local_tiles[pick].contiguous().to(device)
    all_ids = [torch.empty_like(ids) for _ in range(world)]
    all_tl = [torch.empty_like(tl) for _ in range(world)]
    dist.all_gather(all_ids, ids)
    dist.all_gather(all_tl, tl)
    return torch.cat(all_ids).cpu().numpy(), torch.cat(all_tl).cpu().numpy()
