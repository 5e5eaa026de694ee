"""Pins for oracle O1-O5 (summaries, group query, scores, pinned set, top-k).

Each test checks the oracle against something other than itself: the SPEC.md
worked examples (tests/golden), closed forms, exact integer arithmetic, a
library routine (torch bf16 conversion), error bounds, or brute force.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bits(x):
    """float32 values that are exactly bf16-representable -> bf16 bit patterns."""
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32)
    assert np.all((u & 0xFFFF) == 0), "value not bf16-exact"
    return (u >> 16).astype(np.uint16)


def torch_bf16_bits(x):
    t = torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


# ------------------------------------------------------------------ O1
def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.standard_normal(5000).astype(np.float32) * 3,
        rng.standard_normal(500).astype(np.float32) * 1e-39,       # subnormals
        np.array([0.0, -0.0, 1.0, -1.0, 3.4e38, -3.4e38, np.inf, -np.inf], np.float32),
        # exact ties: low 16 bits == 0x8000 with even / odd bf16 lsb
        (np.array([0x3F808000, 0x3F818000, 0xBF808000, 0x7F7F8000], np.uint32)).view(np.float32),
    ])
    assert np.array_equal(oracle.f32_to_bf16(x), torch_bf16_bits(x))


def test_summary_block_size_one_is_the_key():
    # c=1 => representative equals its single key bit-exactly
    K, _ = synth.segment_kv(1, 0, 0, 0, 100)
    assert np.array_equal(oracle.block_summaries(K, 1), K)


@pytest.mark.parametrize("n,P", [(64, 16), (67, 16), (9, 4), (8, 4), (50, 8)])
def test_summary_exact_mean_small_integers(n, P):
    # Integer keys: the fp32 sum is exact, so S = bf16_rne(fp32(sum / cnt)) with
    # one IEEE division; checked against int64 sums, numpy division, torch RNE.
    rng = np.random.default_rng(n * 31 + P)
    Ki = rng.integers(-8, 9, size=(n, 5))
    S = oracle.block_summaries(bits(Ki.astype(np.float32)), P)
    nb = (n + P - 1) // P
    assert S.shape == (nb, 5)                                    # SPEC.md:116-117 chunk count
    for b in range(nb):
        blk = Ki[P * b: min(n, P * b + P)]
        mean32 = np.float32(blk.sum(0)) / np.float32(len(blk))   # IEEE fp32 division
        assert np.array_equal(S[b], torch_bf16_bits(mean32))


def test_summary_chunk_counts_spec():
    g = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))["build_chunks"]
    for ex in g:
        K = bits(np.ones((ex["n"], 2), np.float32))
        S = oracle.block_summaries(K, ex["c"])
        assert S.shape[0] == ex["n_chunks"], ex["cite"]
        assert np.array_equal(S, bits(np.ones((ex["n_chunks"], 2), np.float32)))


# ------------------------------------------------------------------ O2 / O3
def test_dot_scores_spec_examples():
    g = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))["dot_scores"]
    for ex in g:
        q = bits(np.array([ex["query"]], np.float32))                # G = 1
        S = bits(np.array(ex["keys"], np.float32))
        sc = oracle.block_scores(oracle.group_query(q), S)
        assert np.array_equal(sc, np.array(ex["scores"], np.float32)), ex["cite"]


def test_order_sensitive_examples():
    g = json.load(open(os.path.join(GOLD, "order_sensitive.json")))
    for ex in g["group_query"]:
        qb = oracle.group_query(bits(np.array(ex["q"], np.float32)))
        assert np.array_equal(qb, np.array(ex["qbar"], np.float32)), ex["why"]
    for ex in g["scores"]:
        sc = oracle.block_scores(np.array(ex["qbar"], np.float32), bits(np.array(ex["s"], np.float32)))
        assert np.array_equal(sc, np.array(ex["score"], np.float32)), ex["why"]


def test_scores_exact_on_integers():
    rng = np.random.default_rng(3)
    G, d, nb = 4, 128, 300
    q = rng.integers(-16, 17, size=(G, d))
    S = rng.integers(-16, 17, size=(nb, d))
    qb = oracle.group_query(bits(q.astype(np.float32)))
    assert np.array_equal(qb, q.sum(0).astype(np.float32))
    sc = oracle.block_scores(qb, bits(S.astype(np.float32)))
    assert np.array_equal(sc, (S @ q.sum(0)).astype(np.float32))   # |dot| < 2^24: exact


def test_scores_within_fp32_error_bound():
    # |fl(sum) - sum| <= gamma_d * sum |qbar_j s_j|,  gamma_d = d u / (1 - d u), u = 2^-24
    K, _ = synth.segment_kv(5, 0, 0, 0, 16 * 200)
    q = synth.queries(5, 0, 0, 0, 4)[0]
    S = oracle.block_summaries(K, 16)
    qb = oracle.group_query(q)
    sc = oracle.block_scores(qb, S).astype(np.float64)
    Sf = synth.bf16_bits_to_f32(S).astype(np.float64)
    exact = Sf @ qb.astype(np.float64)
    d, u = 128, 2.0 ** -24
    gamma = d * u / (1 - d * u)
    bound = gamma * (np.abs(Sf) @ np.abs(qb.astype(np.float64)))
    assert np.all(np.abs(sc - exact) <= bound)
    # and qbar is the fp32 sum of the bf16 heads (error bound for G=4 adds)
    qf = synth.bf16_bits_to_f32(q).astype(np.float64)
    assert np.all(np.abs(qb - qf.sum(0)) <= 4 * u * np.abs(qf).sum(0) + 1e-30)


# ------------------------------------------------------------------ O4
@pytest.mark.parametrize("n,P,expect", [
    (4096, 16, [0, 252, 253, 254, 255]),
    (4095, 16, [0, 251, 252, 253, 254, 255]),
    (80, 16, [0, 1, 2, 3, 4]),
    (50, 16, [0, 1, 2, 3]),
    (100, 1, [0, 1, 2, 3] + list(range(36, 100))),
    (100, 2, [0, 1] + list(range(18, 50))),
    (130, 4, [0] + list(range(16, 33))),
])
def test_pinned_blocks_enumerated(n, P, expect):
    # sink = first 4 tokens, local = last 64 tokens (block-granular, R9)
    m = oracle.pinned_blocks(n, P, 4, 64)
    assert list(np.nonzero(m)[0]) == expect


def test_pinned_blocks_cover_exactly_sink_and_local_tokens():
    for n in range(1, 300, 7):
        for P in (1, 2, 4, 8, 16):
            m = oracle.pinned_blocks(n, P, 4, 64)
            tok_pinned = set()
            for b in np.nonzero(m)[0]:
                tok_pinned |= set(range(P * b, min(n, P * b + P)))
            need = set(range(min(4, n))) | set(range(max(0, n - 64), n))
            assert need <= tok_pinned
            # minimal: every pinned block contains a sink or local token
            for b in np.nonzero(m)[0]:
                assert set(range(P * b, min(n, P * b + P))) & need


# ------------------------------------------------------------------ O5
def _ref_topk(scores, pinned, k):
    """Brute force: key = (is-not-nan, score, -id) descending, via Python sort."""
    cands = [b for b in range(len(scores)) if not pinned[b]]

    def key(b):
        s = float(scores[b])
        return (0, 0.0, b) if np.isnan(s) else (1, -s, b)

    ordered = sorted(cands, key=lambda b: (-key(b)[0], key(b)[1], key(b)[2]))
    return sorted(ordered[:k])


def test_topk_spec_examples():
    g = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))["exact_topk"]
    for ex in g:
        ids = oracle.topk(np.array(ex["scores"], np.float32), np.zeros(len(ex["scores"]), np.uint8), ex["k"])
        assert list(ids) == ex["ids"], ex["cite"]


def test_topk_brute_force_with_ties_nan_signed_zero():
    rng = np.random.default_rng(7)
    for trial in range(300):
        nb = int(rng.integers(1, 60))
        sc = rng.integers(-3, 4, size=nb).astype(np.float32)       # many ties
        sc[rng.random(nb) < 0.1] = np.nan
        sc[rng.random(nb) < 0.1] = -0.0
        pinned = (rng.random(nb) < 0.2).astype(np.uint8)
        m = int((pinned == 0).sum())
        k = int(rng.integers(0, m + 1))
        ids = oracle.topk(sc, pinned, k)
        assert list(ids) == _ref_topk(sc, pinned, k)
        # order property: every selected ranks at or above every unselected candidate
        sel = set(ids.tolist())
        for a in sel:
            for b in range(nb):
                if pinned[b] or b in sel:
                    continue
                sa, sb = sc[a], sc[b]
                assert not np.isnan(sa) or np.isnan(sb)
                if not np.isnan(sa) and not np.isnan(sb):
                    assert sa > sb or (sa == sb and a < b)


def test_topk_k_too_large_is_error():
    with pytest.raises(oracle.OracleError):
        oracle.topk(np.zeros(5, np.float32), np.array([1, 0, 0, 0, 1], np.uint8), 4)


def test_topk_permutation_equivariance_and_scale_invariance():
    # permuting keys permutes the output; positive query scale
    # (a power of two keeps every product exact) does not change the set.
    rng = np.random.default_rng(11)
    K, _ = synth.segment_kv(2, 0, 0, 0, 16 * 64)
    S = oracle.block_summaries(K, 16)
    q = synth.queries(2, 0, 0, 0, 4)[0]
    qb = oracle.group_query(q)
    pinned = np.zeros(64, np.uint8)
    ids = oracle.topk(oracle.block_scores(qb, S), pinned, 8)
    perm = rng.permutation(64)
    ids_p = oracle.topk(oracle.block_scores(qb, S[perm]), pinned, 8)
    assert sorted(perm[ids_p].tolist()) == ids.tolist()
    ids_s = oracle.topk(oracle.block_scores(qb * np.float32(4.0), S), pinned, 8)
    assert np.array_equal(ids_s, ids)


def test_block_size_one_reduces_to_exact_token_topk():
    # PAPER.md:246-247 "naive" index / SPEC.md:134,159: with P = 1 the block index is
    # the exact top-k over tokens.  Integer inputs keep every dot exact so the
    # brute-force token ranking (int64) is unambiguous.
    rng = np.random.default_rng(13)
    n, G, k = 200, 4, 20
    Ki = rng.integers(-6, 7, size=(n, 128))
    qi = rng.integers(-6, 7, size=(G, 128))
    pinned = oracle.pinned_blocks(n, 1, 4, 64)
    ids, _ = oracle.segment_select(bits(qi.astype(np.float32)), oracle.block_summaries(bits(Ki.astype(np.float32)), 1), pinned, k)
    tok = Ki @ qi.sum(0)
    cands = [i for i in range(n) if not pinned[i]]
    exact = sorted(sorted(cands, key=lambda i: (-tok[i], i))[:k])
    assert ids.tolist() == exact
