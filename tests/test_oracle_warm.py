"""Pins of the oracle's importance-guided warm-up (O14): the importances are a
distribution per query (they sum to G x n_obs), agree with torch's softmax (an independent
library routine), a query aligned with one block puts that block first, and the placement keeps
the pinned blocks, fills exactly the free slots with the most important blocks."""
import numpy as np
import torch

import oracle
import synth


def test_importance_is_attention_mass():
    n, P = 3000, 16
    K, _ = synth.segment_kv(2, 0, 0, 0, n)
    q = synth.queries(2, 0, 0, 0, 4, nsteps=16).transpose(1, 0, 2)   # [G][n_obs][d]
    imp = oracle.warm_importance(q, K, P)
    assert imp.shape == ((n + P - 1) // P,)
    assert abs(imp.sum() - 4 * 16) < 1e-9
    Qt = torch.from_numpy(oracle._f64(q).reshape(-1, 128))
    Kt = torch.from_numpy(oracle._f64(K))
    w = torch.softmax(Qt @ Kt.T / 128 ** 0.5, dim=1).sum(0).numpy()
    ref = np.add.reduceat(w, np.arange(0, n, P))
    assert np.allclose(imp, ref, rtol=1e-10, atol=1e-12)


def test_aligned_query_picks_its_block_first():
    n, P = 1024, 16
    rng = np.random.default_rng(3)
    Kf = rng.standard_normal((n, 128)).astype(np.float32) * 0.1
    Kf[37 * 16:38 * 16] += 3.0                                       # block 37 aligned with the query
    K = (Kf.view(np.uint32) >> 16).astype(np.uint16)
    q = (np.full((1, 1, 128), 1.0, np.float32).view(np.uint32) >> 16).astype(np.uint16)
    imp = oracle.warm_importance(q, K, P)
    assert int(np.argmax(imp)) == 37


def test_warm_placement():
    n, P, C = 4096, 16, 69
    K, _ = synth.segment_kv(4, 0, 0, 0, n)
    q = synth.queries(4, 0, 0, 0, 4, nsteps=16).transpose(1, 0, 2)
    imp = oracle.warm_importance(q, K, P)
    pin = oracle.pinned_blocks(n, P)
    c = oracle.SegmentCache(len(pin), C, pin)
    chosen = oracle.warm_start(c, imp)
    assert len(chosen) == C - pin.sum() and (c.slot_block >= 0).all()
    assert all(c.table[b] >= 0 for b in np.nonzero(pin)[0])
    free = np.nonzero(~pin.astype(bool))[0]
    top = free[np.argsort(-imp[free], kind="stable")][:len(chosen)]
    assert set(top.tolist()) == set(chosen.tolist())
    assert np.all(np.diff(c.slot_block[pin.sum():]) > 0)             # ascending block order
