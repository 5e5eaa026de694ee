"""Pins of the oracle's decode-time append (O13): a resident cache grown token by
token equals the cache of the whole prefix loaded at once; a host-backed cache admits a new block
into the lowest free slot, else evicts the argmin of the policy key among the non-pinned residents
(independent Python restatement of the key); the local window slides (pinned set of n + 1)."""
import numpy as np
import pytest

import oracle
import synth


def test_resident_append_equals_prefix_load():
    n0, steps, P = 100, 70, 16
    K, V = synth.segment_kv(5, 0, 0, 0, n0 + steps)
    nbmax = (n0 + steps + P - 1) // P
    Kc, Vc = K[:n0].copy(), V[:n0].copy()
    S = oracle.block_summaries(Kc, P)
    c = oracle.SegmentCache((n0 + P - 1) // P, nbmax, oracle.pinned_blocks(n0, P))
    for t in range(steps):
        Kc, Vc, S, pin = oracle.append_token(c, Kc, Vc, S, n0 + t, P, K[n0 + t], V[n0 + t], t + 1, oracle.LRU, None)
    assert np.array_equal(S, oracle.block_summaries(K, P))
    assert np.array_equal(pin, oracle.pinned_blocks(n0 + steps, P))
    ref = oracle.SegmentCache(nbmax, nbmax, pin)
    assert np.array_equal(c.table, ref.table) and np.array_equal(c.slot_block, ref.slot_block)


def _key(policy, s, c, scores):
    b = int(c.slot_block[s])
    if policy == oracle.LRU:
        return (int(c.last_use[s]), int(c.phase[s]), b)
    if policy == oracle.LFU:
        return (int(c.use_count[s]), int(c.last_use[s]), int(c.phase[s]), b)
    return (float(scores[b]), -b)


@pytest.mark.parametrize("policy", [oracle.LRU, oracle.LFU, oracle.LA])
def test_host_backed_admission_rule(policy):
    n0, P, C, k = 2048, 16, 40, 24
    K, V = synth.segment_kv(6, 0, 0, 0, n0 + 100)
    Kc, Vc = K[:n0].copy(), V[:n0].copy()
    S = oracle.block_summaries(Kc, P)
    c = oracle.SegmentCache(n0 // P, C, oracle.pinned_blocks(n0, P))
    rng = np.random.default_rng(1)
    n, step = n0, 1
    for t in range(100):
        q = synth.queries(6, 0, 0, 0, 4, t0=t, nsteps=1)[0]
        if t % 7 == 0:                                # a decode step between some appends
            ids, scores = oracle.segment_select(q, S, c.is_pinned, k)
            c.resolve(ids, step, policy, scores, k + 8)
            step += 1
        scores = oracle.block_scores(oracle.group_query(q), S)
        before = (c.table.copy(), c.slot_block.copy())
        opens = n % P == 0
        if opens:
            pin_new = oracle.pinned_blocks(n + 1, P).astype(bool)
            free = np.nonzero(before[1] < 0)[0]
            if len(free):
                want = free[0]
            else:
                cand = [s for s in range(C) if before[1][s] >= 0 and not pin_new[before[1][s]]]
                want = min(cand, key=lambda s: _key(policy, s, c, scores))
        Kc, Vc, S, pin = oracle.append_token(c, Kc, Vc, S, n, P, K[n], V[n], step, policy, scores)
        if opens:
            b = n // P
            assert c.table[b] == want and c.slot_block[want] == b
            assert c.last_use[want] == step and c.phase[want] == 1 and c.use_count[want] == 1
            old = before[1][want]
            if old >= 0:
                assert c.table[old] == -1
        else:
            assert np.array_equal(c.slot_block, before[1])
        n += 1
    occupied = c.slot_block[c.slot_block >= 0]
    assert len(set(occupied.tolist())) == len(occupied)   # a block in at most one slot
    assert all(c.table[b] >= 0 for b in np.nonzero(c.is_pinned)[0])   # pinned blocks resident
