"""Pins of the oracle's hierarchical index (O9 windowed k-means, O10 two-stage descent; reading
R27).  Each pin is independent of the oracle's own code path:
degenerate parameters that reduce to the flat top-k, exactly separable point clouds, the
k-means fixed-point / nearest-centroid invariants checked in float64 numpy, and an independent
numpy restatement of the descent given the oracle's O3 block scores."""
import numpy as np
import pytest

import oracle
import synth


def _bf16(x):
    return (np.asarray(x, np.float32).view(np.uint32) >> 16).astype(np.uint16)


def _f32(b):
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32)


@pytest.mark.parametrize("n,P,k,seed", [(4096, 16, 32, 0), (3000, 16, 20, 1), (900, 4, 40, 2), (700, 1, 64, 3)])
def test_ratio_one_reduces_to_flat_topk(n, P, k, seed):
    # one centroid per block: every block is its own centroid, the top-(4k) centroids contain
    # the flat top-k, so the descent returns exactly O5's ids (SPEC.md:126,134 degenerate case)
    K, _ = synth.segment_kv(seed, 0, 0, 0, n)
    S = oracle.block_summaries(K, P)
    cent, cent_of = oracle.index_build(S, 1)
    assert cent.shape[0] == S.shape[0] and np.array_equal(cent_of, np.arange(S.shape[0]))
    assert np.array_equal(cent, S)
    pin = oracle.pinned_blocks(n, P)
    for t in range(3):
        q = synth.queries(seed, 0, 0, 0, 4, t0=t, nsteps=1)[0]
        ids, _, la = oracle.index_select(oracle.group_query(q), S, cent, cent_of, pin, k,
                                         oracle.index_fanout(k, 1, cent.shape[0], pin.sum()))
        ref, sc = oracle.segment_select(q, S, pin, k)
        assert np.array_equal(ids, ref)
        cand = np.zeros(len(pin), bool)
        # candidates = non-pinned blocks of the top 4k centroids; every block scored
        assert np.array_equal(la[~pin.astype(bool)][np.isin(np.arange(len(pin))[~pin.astype(bool)], ids)],
                              sc[ids])


def test_separable_clouds_one_centroid_each():
    # one window of 64 blocks: blocks 0..31 around A, 32..63 around B (far apart), 2 centroids;
    # each cloud is +-e symmetric around its centre, so the fp32 mean is exactly the centre
    d = 128
    A = np.zeros(d, np.float32); A[0] = 64.0
    B = np.zeros(d, np.float32); B[1] = 64.0
    rng = np.random.default_rng(5)
    S = np.empty((64, d), np.float32)
    for c0, centre in ((0, A), (32, B)):
        e = rng.integers(-2, 3, size=(16, d)).astype(np.float32)
        S[c0:c0 + 16] = centre + e
        S[c0 + 16:c0 + 32] = centre - e
    perm = rng.permutation(64)                       # interleave the clouds inside the window
    Sb = _bf16(S[perm])
    cent, cent_of = oracle.index_build(Sb, 32)
    assert cent.shape[0] == 2
    cloud = (perm >= 32).astype(np.int32)             # 0 = A, 1 = B
    # the two centroids partition the blocks exactly by cloud
    assert len(set(zip(cloud, cent_of))) == 2
    for c in range(2):
        members = cloud[cent_of == c]
        centre = A if members[0] == 0 else B
        assert np.array_equal(_f32(cent[c]), centre)


def test_kmeans_invariants_float64():
    K, _ = synth.segment_kv(7, 0, 0, 0, 20000)
    S = oracle.block_summaries(K, 16)                # 1250 blocks: 19 full windows + a short one
    for ratio in (2, 4, 8):
        cent, cent_of = oracle.index_build(S, ratio)
        nb = S.shape[0]
        win = np.arange(nb) // oracle.IDX_WINDOW
        # every centroid has members, all inside one window; centroids numbered window by window
        assert np.array_equal(np.unique(cent_of), np.arange(cent.shape[0]))
        cw = np.array([win[cent_of == c][0] for c in range(cent.shape[0])])
        assert all((win[cent_of == c] == cw[c]).all() for c in range(cent.shape[0]))
        assert (np.diff(cw) >= 0).all()
        nwin = -(-np.bincount(win) // ratio)
        assert cent.shape[0] <= nwin.sum()
        # nearest centroid among the window's (float64, within the fp32/bf16 rounding margin)
        X = _f32(S).astype(np.float64)
        C = _f32(cent).astype(np.float64)
        for b in range(0, nb, 7):
            cs = np.nonzero(cw == win[b])[0]
            dist = ((X[b] - C[cs]) ** 2).sum(1)
            a = ((X[b] - C[cent_of[b]]) ** 2).sum()
            assert a <= dist.min() + 1e-2 * (1 + dist.min()), (ratio, b)


def _descent_numpy(qbar, S, cent, cent_of, pinned, k, m):
    """Independent restatement of the two-stage descent, on the oracle's O3 scores."""
    cs = oracle.block_scores(qbar, cent)
    bs = oracle.block_scores(qbar, S)

    def order(sc):                                   # score desc (NaN lowest), id asc
        key = np.where(np.isnan(sc), -np.inf, sc)
        return np.lexsort((np.arange(len(sc)), -key.astype(np.float64)))
    top = order(cs)[:m]
    cand = np.isin(cent_of, top) & ~pinned.astype(bool)
    if cand.sum() < k:
        cand = ~pinned.astype(bool)
    idx = np.nonzero(cand)[0]
    ids = np.sort(idx[order(bs[idx])[:k]])
    la = np.where(cand, bs, cs[cent_of])
    return ids.astype(np.int32), cs, la.astype(np.float32)


@pytest.mark.parametrize("seed,alpha", [(0, 0.9), (1, 0.0), (2, 0.9)])
def test_descent_matches_independent_restatement(seed, alpha):
    n, P, k, ratio = 65536, 16, 128, 4
    K, _ = synth.segment_kv(seed, 0, 1, 2, n)
    S = oracle.block_summaries(K, P)
    cent, cent_of = oracle.index_build(S, ratio)
    pin = oracle.pinned_blocks(n, P)
    m = oracle.index_fanout(k, ratio, cent.shape[0], pin.sum())
    assert m == 128 + 5
    for t in range(2):
        q = synth.queries(seed, 0, 1, 2, 4, t0=t, nsteps=1, alpha=alpha)[0]
        qb = oracle.group_query(q)
        ids, cs, la = oracle.index_select(qb, S, cent, cent_of, pin, k, m)
        rid, rcs, rla = _descent_numpy(qb, S, cent, cent_of, pin, k, m)
        assert np.array_equal(ids, rid)
        assert np.array_equal(cs.view(np.uint32), rcs.view(np.uint32))
        assert np.array_equal(la.view(np.uint32), rla.view(np.uint32))


def test_fanout_always_leaves_k_candidates():
    # m >= k + pinned and every centroid owns a block: stage 2 never runs short of candidates
    for n, P, ratio, k in [(2048, 16, 8, 100), (5000, 4, 16, 200), (1500, 16, 2, 60)]:
        K, _ = synth.segment_kv(4, 0, 0, 0, n)
        S = oracle.block_summaries(K, P)
        cent, cent_of = oracle.index_build(S, ratio)
        pin = oracle.pinned_blocks(n, P)
        m = oracle.index_fanout(k, ratio, cent.shape[0], pin.sum())
        for t in range(3):
            qb = oracle.group_query(synth.queries(4, 0, 0, 0, 4, t0=t, nsteps=1)[0])
            top = np.lexsort((np.arange(cent.shape[0]), -oracle.block_scores(qb, cent).astype(np.float64)))[:m]
            cand = np.isin(cent_of, top) & ~pin.astype(bool)
            assert cand.sum() >= k


def test_few_candidates_fall_back_to_every_block():
    # k larger than the members of the chosen centroids: every non-pinned block is a candidate
    n, P = 2048, 16
    K, _ = synth.segment_kv(3, 0, 0, 0, n)
    S = oracle.block_summaries(K, P)
    cent, cent_of = oracle.index_build(S, 8)
    pin = oracle.pinned_blocks(n, P)
    q = synth.queries(3, 0, 0, 0, 4, nsteps=1)[0]
    k = 100
    ids, _, _ = oracle.index_select(oracle.group_query(q), S, cent, cent_of, pin, k, 1)
    ref, _ = oracle.segment_select(q, S, pin, k)
    assert np.array_equal(ids, ref)


def test_index_recall_on_clustered_workload_is_high():
    # information, not parity: the windowed index keeps most of the flat top-k
    n, P, k = 131072, 16, 128
    K, _ = synth.segment_kv(0, 0, 0, 0, n)
    S = oracle.block_summaries(K, P)
    cent, cent_of = oracle.index_build(S, 4)
    pin = oracle.pinned_blocks(n, P)
    rec = []
    for t in range(4):
        q = synth.queries(0, 0, 0, 0, 4, t0=t, nsteps=1)[0]
        ids, _, _ = oracle.index_select(oracle.group_query(q), S, cent, cent_of, pin, k,
                                        oracle.index_fanout(k, 4, cent.shape[0], pin.sum()))
        ref, _ = oracle.segment_select(q, S, pin, k)
        rec.append(len(set(ids) & set(ref)) / k)
    assert np.mean(rec) > 0.8, rec
