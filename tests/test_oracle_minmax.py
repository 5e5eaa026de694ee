"""Pins of the oracle's Quest min/max summaries and scores (O12): the bound
property against exact fp64 per-token dot products, single-token and constant blocks, and an
independent numpy float32 restatement (IEEE single arithmetic step by step)."""
import numpy as np
import pytest

import oracle
import synth


def _f32(b):
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32)


def _scores_numpy(qbar, MN, MX):
    out = np.empty(MN.shape[0], np.float32)
    mn, mx = _f32(MN), _f32(MX)
    for b in range(MN.shape[0]):
        acc = np.float32(0.0)
        for j in range(MN.shape[1]):
            acc = np.float32(acc + np.maximum(np.float32(qbar[j] * mn[b, j]), np.float32(qbar[j] * mx[b, j])))
        out[b] = acc
    return out


@pytest.mark.parametrize("n,P", [(1000, 16), (333, 4), (50, 1)])
def test_minmax_summaries_and_scores(n, P):
    K, _ = synth.segment_kv(9, 0, 0, 0, n)
    MN, MX = oracle.minmax_summaries(K, P)
    Kf = _f32(K).reshape(n, 128)
    nb = (n + P - 1) // P
    for b in range(nb):                              # channel-wise min / max of the valid tokens
        blk = Kf[P * b:min(n, P * b + P)]
        assert np.array_equal(_f32(MN[b]), blk.min(0)) and np.array_equal(_f32(MX[b]), blk.max(0))
    q = synth.queries(9, 0, 0, 0, 4, nsteps=1)[0]
    qb = oracle.group_query(q)
    sc = oracle.minmax_scores(qb, MN, MX)
    assert np.array_equal(sc.view(np.uint32), _scores_numpy(qb, MN, MX).view(np.uint32))
    # upper bound of every token's dot product (fp64 exact), within the fp32 summation error
    dots = Kf.astype(np.float64) @ qb.astype(np.float64)
    for b in range(nb):
        best = dots[P * b:min(n, P * b + P)].max()
        assert sc[b] >= best - 1e-4 * (1 + np.abs(qb).sum() * np.abs(Kf).max())
    if P == 1:                                      # a single token: min = max = the key
        assert np.array_equal(MN, MX) and np.array_equal(MN, K.reshape(n, 128))


def test_constant_block_bound_is_tight():
    K = np.tile(_f32(synth.segment_kv(1, 0, 0, 0, 1)[0]).view(np.uint32) >> 16, (16, 1)).astype(np.uint16)
    MN, MX = oracle.minmax_summaries(K, 16)
    assert np.array_equal(MN, MX)
    qb = oracle.group_query(synth.queries(1, 0, 0, 0, 4, nsteps=1)[0])
    exact = float(_f32(K[0]).astype(np.float64) @ qb.astype(np.float64))
    assert oracle.minmax_scores(qb, MN, MX)[0] == pytest.approx(exact, rel=1e-5, abs=1e-4)
