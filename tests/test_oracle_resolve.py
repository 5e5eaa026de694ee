"""Pins for oracle O6 (resolve / eviction) and O7 (fetch).

The oracle's key-based resolve is checked against independent, textbook,
sequential Python simulators (an OrderedDict two-phase LRU, a set-protected
LFU, a direct-sort lookahead) and against cache invariants (capacity, table /
slot-map bijection, co-residency of the step's selection, no eviction when
the cache holds everything, LRU stack inclusion).
"""
from collections import OrderedDict

import numpy as np
import pytest

import oracle


# --------------------------------------------------------------- references
class RefCache:
    """Sequential textbook simulator of one segment's block cache.

    Per step: (1) look up every selected block; hits are touched in ascending
    id order; (2) misses are admitted in ascending id order, each into the
    lowest free slot, else into the slot of the policy's victim among residents
    that are neither pinned nor selected this step (PAPER.md:449 for LA;
    LRU/LFU as the paper's baselines)."""

    def __init__(self, nb, C, pinned, policy):
        self.policy = policy
        self.pinned = set(np.nonzero(pinned)[0].tolist())
        self.slot_of = {}
        self.free = list(range(C))
        if C >= nb:
            for b in range(nb):
                self.slot_of[b] = b
            self.free = list(range(nb, C))
        else:
            for i, b in enumerate(sorted(self.pinned)):
                self.slot_of[b] = i
            self.free = list(range(len(self.pinned), C))
        self.lru = OrderedDict()           # non-pinned residents, least recent first
        self.count = {}
        self.last = {}
        self.phase = {}
        if C >= nb:
            for b in range(nb):
                if b not in self.pinned:
                    self.lru[b] = None
                    self.count[b], self.last[b], self.phase[b] = 0, 0, 0

    def step(self, S, t, scores):
        S = sorted(S)
        Sset = set(S)
        hits = [b for b in S if b in self.slot_of]
        misses = [b for b in S if b not in self.slot_of]
        for b in hits:
            self.lru.move_to_end(b)
            self.count[b] += 1
            self.last[b], self.phase[b] = t, 0
        assign = []
        for b in misses:
            if self.free:
                s = min(self.free)
                self.free.remove(s)
            else:
                v = self._victim(Sset, scores)
                s = self.slot_of.pop(v)
                del self.lru[v], self.count[v], self.last[v], self.phase[v]
            self.slot_of[b] = s
            self.lru[b] = None
            self.count[b], self.last[b], self.phase[b] = 1, t, 1
            assign.append((b, s))
        return len(hits), assign

    def _victim(self, Sset, scores):
        cands = [b for b in self.lru if b not in Sset]
        if not cands:
            raise RuntimeError("capacity")
        if self.policy == oracle.LRU:
            return cands[0]                          # OrderedDict front = least recent
        if self.policy == oracle.LFU:
            return min(cands, key=lambda b: (self.count[b], self.last[b], self.phase[b], b))
        def la_key(b):                               # lowest score first, NaN lowest, larger id first
            s = float(scores[b])
            return (0, 0.0, -b) if np.isnan(s) else (1, s + 0.0, -b)
        return min(cands, key=la_key)


def _trace(rng, nb, pinned, k, steps, locality):
    """Random selections with temporal locality (keeps a fraction of the last set)."""
    cands = np.nonzero(pinned == 0)[0]
    prev = rng.choice(cands, k, replace=False)
    out = []
    for _ in range(steps):
        keep = prev[rng.random(k) < locality]
        rest = np.setdiff1d(cands, keep)
        new = rng.choice(rest, k - len(keep), replace=False)
        cur = np.sort(np.concatenate([keep, new]))
        out.append(cur.astype(np.int32))
        prev = cur
    return out


def _check_invariants(c, S, attn, pinned_ids, W):
    tb, sbk = c.table, c.slot_block
    res = np.nonzero(tb >= 0)[0]
    assert len(res) <= c.C                                           # capacity
    assert np.all(sbk[tb[res]] == res)                               # bijection
    occ = np.nonzero(sbk >= 0)[0]
    assert np.all(tb[sbk[occ]] == occ)
    need = np.union1d(S, pinned_ids)
    assert np.all(tb[need] >= 0)                                     # co-residency
    valid = attn[attn[:, 0] >= 0]
    assert np.array_equal(valid[:, 0], need)                         # S u pinned, ascending
    assert np.array_equal(valid[:, 1], tb[need])
    assert len(valid) <= W


@pytest.mark.parametrize("policy", [oracle.LRU, oracle.LFU, oracle.LA])
@pytest.mark.parametrize("seed", range(4))
def test_resolve_matches_reference_simulator(policy, seed):
    rng = np.random.default_rng(100 + seed)
    n, P = 16 * int(rng.integers(40, 120)) - int(rng.integers(0, 16)), 16
    nb = (n + P - 1) // P
    pinned = oracle.pinned_blocks(n, P, 4, 64)
    pinned_ids = np.nonzero(pinned)[0]
    k = int(rng.integers(4, 16))
    C = len(pinned_ids) + k + int(rng.integers(0, 3 * k))
    W = k + len(pinned_ids)
    c = oracle.SegmentCache(nb, C, pinned)
    ref = RefCache(nb, C, pinned, policy)
    for t, S in enumerate(_trace(rng, nb, pinned, k, 60, [0.0, 0.5, 0.8, 0.95][seed]), start=1):
        scores = rng.integers(-4, 5, size=nb).astype(np.float32)       # ties exercised
        scores[rng.random(nb) < 0.05] = np.nan
        attn, miss, nm, nh = c.resolve(S, t, policy, scores, W)
        rh, assign = ref.step(S.tolist(), t, scores)
        assert nh == rh and nm == len(assign)
        assert [tuple(x) for x in miss[:nm].tolist()] == assign
        _check_invariants(c, S, attn, pinned_ids, W)
        for b, s in ref.slot_of.items():
            assert c.table[b] == s


def test_fully_resident_never_misses():
    # capacity >= context => nothing evicted, hit rate 1
    rng = np.random.default_rng(5)
    n, P, k = 1024, 16, 12
    nb = n // P
    pinned = oracle.pinned_blocks(n, P, 4, 64)
    c = oracle.SegmentCache(nb, nb, pinned)
    for t, S in enumerate(_trace(rng, nb, pinned, k, 30, 0.3), start=1):
        attn, miss, nm, nh = c.resolve(S, t, oracle.LRU, None, k + 5)
        assert nm == 0 and nh == k
        assert np.array_equal(c.table, np.arange(nb))


def test_capacity_error_when_selection_cannot_be_coresident():
    n, P, k = 1024, 16, 10
    nb = n // P
    pinned = oracle.pinned_blocks(n, P, 4, 64)
    c = oracle.SegmentCache(nb, 5 + k - 1, pinned)            # one slot short
    with pytest.raises(oracle.OracleError) as e:
        c.resolve(np.arange(1, 1 + k, dtype=np.int32), 1, oracle.LRU, None, k + 5)
    assert e.value.code == 3


def test_window_x1_misses_everything_new():
    # C_u = k ("window x1"): only blocks selected in the previous
    # step can hit.
    rng = np.random.default_rng(9)
    n, P, k = 2048, 16, 16
    nb = n // P
    pinned = oracle.pinned_blocks(n, P, 4, 64)
    for policy in (oracle.LRU, oracle.LFU, oracle.LA):
        c = oracle.SegmentCache(nb, 5 + k, pinned)
        prev = set()
        for t, S in enumerate(_trace(rng, nb, pinned, k, 40, 0.6), start=1):
            attn, miss, nm, nh = c.resolve(S, t, policy, rng.random(nb).astype(np.float32), k + 5)
            assert nh == len(prev & set(S.tolist()))
            prev = set(S.tolist())


def test_lru_stack_inclusion_misses_nonincreasing_in_capacity():
    # LRU is a stack algorithm: a larger cache never misses more on the same trace.
    rng = np.random.default_rng(21)
    n, P, k = 4096, 16, 16
    nb = n // P
    pinned = oracle.pinned_blocks(n, P, 4, 64)
    trace = _trace(rng, nb, pinned, k, 80, 0.7)
    total = []
    for C in (5 + k, 5 + 2 * k, 5 + 3 * k, 5 + 5 * k, nb // 2):
        c = oracle.SegmentCache(nb, C, pinned)
        m = 0
        for t, S in enumerate(trace, start=1):
            m += c.resolve(S, t, oracle.LRU, None, k + 5)[2]
        total.append(m)
    assert all(a >= b for a, b in zip(total, total[1:])), total


def test_fetch_keeps_slots_equal_to_host_records():
    # O7 invariant: after every step every resident slot holds its block's record.
    rng = np.random.default_rng(17)
    n, P, k = 1024, 16, 8
    nb = n // P
    pinned = oracle.pinned_blocks(n, P, 4, 64)
    C = 5 + 2 * k
    host = rng.integers(0, 256, size=(nb, 64), dtype=np.uint8)    # small stand-in records
    pool = np.zeros((C, 64), np.uint8)
    c = oracle.SegmentCache(nb, C, pinned)
    for b in np.nonzero(pinned)[0]:                                # initial placement
        pool[c.table[b]] = host[b]
    for t, S in enumerate(_trace(rng, nb, pinned, k, 30, 0.5), start=1):
        attn, miss, nm, nh = c.resolve(S, t, oracle.LA, rng.random(nb).astype(np.float32), k + 5)
        oracle.fetch(host, pool, miss, nm)
        for s in range(C):
            b = c.slot_block[s]
            if b >= 0:
                assert np.array_equal(pool[s], host[b])


def test_admit_evict_spec_rank_order():
    # capacity 2, admit {a,b} then {c} with score(c)>score(a)>score(b) -> b evicted.
    # Map a,b,c to blocks 1,2,3 of an unpinned 4-block segment (sink=local=0).
    nb = 4
    pinned = np.zeros(nb, np.uint8)
    c = oracle.SegmentCache(nb, 2, pinned)
    c.resolve(np.array([1, 2], np.int32), 1, oracle.LA, np.array([0, 2, 1, 0], np.float32), 2)
    scores = np.array([0, 2.0, 1.0, 3.0], np.float32)              # c=3 > a=1 > b=2
    attn, miss, nm, nh = c.resolve(np.array([3], np.int32), 2, oracle.LA, scores, 2)
    assert c.table[2] == -1 and c.table[1] >= 0 and c.table[3] >= 0
