"""ndgi_vt (page table + LRU residency, host C++ behind the C-ABI; no GPU
needed) against an independent Python model of the same policy (R24) and the
SPEC runtime invariants: decode-once within a bucket, eviction safety, the
adversarial LRU trace, bucket arithmetic and error atomicity."""
import collections
import math

import numpy as np
import pytest

import paper_2604_12625_b200 as ndgi


class ModelVT:
    """R24 in plain Python: entry = (slot, bucket); fresh slots in increasing
    order, then strict LRU over slots; stale bucket -> re-decode in place."""

    def __init__(self, num_tiles, capacity, nb):
        self.cap, self.nb = capacity, nb
        self.entry = {}                         # tile -> [slot, bucket]
        self.lru = collections.OrderedDict()    # slot -> tile, least recent first
        self.fresh = 0
        self.stats = [0, 0, 0, 0]

    def bucket(self, t):
        return min(int(math.floor(np.float64(np.float32(t)) * self.nb)), self.nb - 1)

    def request(self, ids, t):
        b = self.bucket(t)
        jobs = []
        seen = set()
        for i in ids:
            if i in seen:
                continue
            seen.add(i)
            self.stats[0] += 1
            if i in self.entry:
                slot = self.entry[i][0]
                self.lru.move_to_end(slot)
                if self.entry[i][1] == b:
                    self.stats[1] += 1
                    continue
            else:
                if self.fresh < self.cap:
                    slot = self.fresh
                    self.fresh += 1
                else:
                    slot, old = next(iter(self.lru.items()))
                    del self.lru[slot]
                    del self.entry[old]
                    self.stats[3] += 1
                self.lru[slot] = i
                self.entry[i] = [slot, b]
            self.entry[i][1] = b
            jobs.append((i, slot))
            self.stats[2] += 1
        td = (b + 0.5) / self.nb
        return jobs, td, b

    def table(self, num_tiles):
        pt = np.full((num_tiles, 2), -1, np.int32)
        for k, (s, b) in self.entry.items():
            pt[k] = (s, b)
        return pt


@pytest.mark.parametrize("cap,ntiles,nb", [(4, 9, 4), (16, 40, 96), (64, 64, 24), (7, 300, 2)])
def test_matches_reference_model_on_random_traces(cap, ntiles, nb):
    rng = np.random.default_rng(cap * 1000 + ntiles)
    vt, ref = ndgi.VT(ntiles, cap, nb), ModelVT(ntiles, cap, nb)
    t = 0.0
    for frame in range(300):
        t = min(1.0, t + rng.choice([0.0, 0.0, 0.003, 0.02]))
        if rng.random() < 0.05:
            t = float(rng.uniform(0, 1))
        if rng.random() < 0.1:
            t = float(rng.integers(0, nb + 1)) / nb           # exactly on a bucket edge
        n = int(rng.integers(0, cap + 3))
        ids = rng.integers(0, ntiles, n)
        if len(set(ids.tolist())) > cap:
            ids = ids[:cap]
        jid, jsl, td, b = vt.request(ids, t)
        jobs, td_r, b_r = ref.request(ids.tolist(), t)
        assert list(zip(jid.tolist(), jsl.tolist())) == jobs
        assert b == b_r and td == pytest.approx(td_r, abs=1e-7)
        np.testing.assert_array_equal(vt.page_table(), ref.table(ntiles))
    s = vt.stats()
    assert [s["requests"], s["hits"], s["jobs"], s["evictions"]] == ref.stats


def test_spec_examples():
    vt = ndgi.VT(10, 8, 96)
    jid, _, _, _ = vt.request([3, 5, 7], 0.5)
    assert sorted(jid.tolist()) == [3, 5, 7]                 # empty cache: 3 jobs
    jid, _, _, _ = vt.request([3, 5, 7], 0.5 + 0.001)        # same bucket: cache hit
    assert len(jid) == 0
    b_now = vt.bucket(0.5)[0]
    t_next = (b_now + 1) / 96                                # crossing a bucket boundary
    jid, jsl, td, b = vt.request([3, 5, 7], t_next)
    assert sorted(jid.tolist()) == [3, 5, 7] and b == b_now + 1
    assert sorted(jsl.tolist()) == [0, 1, 2]                 # re-decoded in place
    assert td == pytest.approx((b + 0.5) / 96, abs=1e-7)


def test_decode_once_within_a_bucket():
    rng = np.random.default_rng(1)
    vt = ndgi.VT(500, 500, 96)
    decoded = collections.Counter()
    for f in range(100):
        ids = rng.integers(0, 500, 64)
        jid, _, _, _ = vt.request(ids, 0.40 + f * 1e-5)       # all inside one bucket
        decoded.update(jid.tolist())
    assert all(c == 1 for c in decoded.values())


def test_eviction_safety_invariant():
    rng = np.random.default_rng(2)
    vt = ndgi.VT(200, 32, 48)
    for f in range(400):
        ids = rng.integers(0, 200, int(rng.integers(1, 33)))
        vt.request(ids, float(rng.uniform(0, 1)))
        pt = vt.page_table()
        res = pt[pt[:, 0] >= 0]
        assert len(np.unique(res[:, 0])) == len(res)        # no two entries share a slot
        assert ((res[:, 0] >= 0) & (res[:, 0] < 32)).all()
        assert len(res) <= 32


def test_adversarial_lru_round_robin_always_misses():
    c = 6
    vt = ndgi.VT(c + 1, c, 1)
    for f in range(5 * (c + 1)):
        jid, _, _, _ = vt.request([f % (c + 1)], 0.5)
        assert len(jid) == 1
    s = vt.stats()
    assert s["hits"] == 0 and s["evictions"] == 5 * (c + 1) - c


def test_bucket_arithmetic():
    vt = ndgi.VT(4, 4, 96)
    assert vt.bucket(0.0)[0] == 0
    assert vt.bucket(1.0)[0] == 95                      # t = 1 -> last bucket
    assert vt.bucket(0.5)[0] == 48                      # bucket edges are exact
    assert vt.bucket(0.25)[0] == 24
    assert vt.bucket(np.nextafter(np.float32(0.25), np.float32(0)))[0] == 23
    b, td = vt.bucket(1.0)
    assert td == pytest.approx(95.5 / 96, abs=1e-7)
    assert ndgi.VT(4, 4, 3).bucket(0.7) == (2, pytest.approx(2.5 / 3))


def test_errors_leave_state_unchanged():
    vt = ndgi.VT(10, 3, 2)
    vt.request([1, 2], 0.1)
    before = vt.page_table().copy(), vt.stats()
    with pytest.raises(ndgi.NdgiError) as e:
        vt.request([1, 10], 0.1)                        # unknown tile id
    assert e.value.status == ndgi.ERR_ARG
    with pytest.raises(ndgi.NdgiError) as e:
        vt.request([4, 5, 6, 7], 0.1)                   # more distinct tiles than slots
    assert e.value.status == ndgi.ERR_RANGE
    for bad in (-0.1, 1.5, float("nan")):
        with pytest.raises(ndgi.NdgiError) as e:
            vt.request([1], bad)
        assert e.value.status == ndgi.ERR_RANGE
    np.testing.assert_array_equal(vt.page_table(), before[0])
    assert vt.stats() == before[1]
    jid, _, _, _ = vt.request([1, 1, 1, 2, 2], 0.1)     # duplicates: hits, no jobs
    assert len(jid) == 0
    with pytest.raises(ndgi.NdgiError):
        ndgi.VT(10, 0, 2)
    with pytest.raises(ndgi.NdgiError):
        ndgi.VT(10, 2, 0)
