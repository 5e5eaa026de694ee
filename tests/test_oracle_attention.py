"""Pins for oracle O8 (attention over the selected blocks, fp64).

k = all candidates reduces the method to dense softmax attention, checked
against torch.nn.functional.scaled_dot_product_attention in fp64 (a library
routine); closed-form special cases and the SPEC softmax examples pin the rest.
"""
import json
import os

import numpy as np
import torch

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bits(x):
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32)
    assert np.all((u & 0xFFFF) == 0)
    return (u >> 16).astype(np.uint16)


def test_all_blocks_equals_dense_sdpa():
    n, P, G = 1000, 16, 4                                   # ragged last block (1000 = 62*16 + 8)
    K, V = synth.segment_kv(3, 1, 2, 1, n)
    q = synth.queries(3, 1, 2, 1, G)[0]
    nb = (n + P - 1) // P
    o, lse = oracle.attention(q, K, V, P, np.arange(nb, dtype=np.int32))
    qt = torch.from_numpy(synth.bf16_bits_to_f32(q).astype(np.float64))[None, :, None, :]   # [1,G,1,d]
    kt = torch.from_numpy(synth.bf16_bits_to_f32(K).astype(np.float64))[None, None].expand(1, G, n, 128)
    vt = torch.from_numpy(synth.bf16_bits_to_f32(V).astype(np.float64))[None, None].expand(1, G, n, 128)
    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt)[0, :, 0].numpy()
    assert np.max(np.abs(o - ref)) <= 1e-6 * max(1.0, np.abs(ref).max())
    z = (qt[0, :, 0] @ kt[0, 0].T) / np.sqrt(128.0)
    assert np.allclose(lse, torch.logsumexp(z, dim=-1).numpy(), rtol=1e-6, atol=1e-6)


def test_full_selection_through_topk_is_dense():
    # the whole select path with k = every candidate + the pinned set = all blocks
    n, P, G = 700, 16, 4
    K, V = synth.segment_kv(4, 0, 0, 0, n)
    q = synth.queries(4, 0, 0, 0, G)[0]
    pinned = oracle.pinned_blocks(n, P, 4, 64)
    nb = len(pinned)
    k = int((pinned == 0).sum())
    c = oracle.SegmentCache(nb, nb, pinned)
    r = oracle.segment_step(c, q, oracle.block_summaries(K, P), K, V, P, k, 1, oracle.LRU, nb)
    o_dense, _ = oracle.attention(q, K, V, P, np.arange(nb, dtype=np.int32))
    assert np.array_equal(r["o"], o_dense)


def test_single_token_returns_its_value():
    n, P = 33, 16                                          # block 2 holds one token
    K, V = synth.segment_kv(6, 0, 0, 0, n)
    q = synth.queries(6, 0, 0, 0, 2)[0]
    o, lse = oracle.attention(q, K, V, P, np.array([2], np.int32))
    assert np.array_equal(o, np.broadcast_to(synth.bf16_bits_to_f32(V[32]), o.shape))


def test_equal_logits_give_mean_value():
    n, P = 48, 16
    K, V = synth.segment_kv(7, 0, 0, 0, n)
    q = np.zeros((3, 128), np.uint16)                      # zero query: every logit is 0
    o, lse = oracle.attention(q, K, V, P, np.array([0, 2], np.int32))
    vf = synth.bf16_bits_to_f32(V).astype(np.float64)
    mean = np.concatenate([vf[0:16], vf[32:48]]).mean(0)
    assert np.allclose(o, mean, rtol=0, atol=1e-7)
    assert np.allclose(lse, np.log(32.0), atol=1e-6)


def test_spec_softmax_examples():
    # SPEC.md:64-66 via d = 1, one query head, logits z = q * k.
    g = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))["softmax_weights"]
    for ex in g:
        z = np.array(ex["logits"], np.float32)
        n = len(z)
        Kd = bits(z.reshape(n, 1))                         # q = 1 -> z_i = k_i / sqrt(1)
        Vd = bits(np.eye(n, dtype=np.float32)[:, :1]) if n == 2 else None
        # value = one-hot of token 0: o = weight of token 0
        Vd = bits((np.arange(n) == 0).astype(np.float32).reshape(n, 1))
        o, _ = oracle.attention(bits(np.ones((1, 1), np.float32)), Kd, Vd, 1,
                                np.arange(n, dtype=np.int32))
        assert abs(float(o[0, 0]) - ex["weights"][0]) <= ex["tol"], ex["cite"]
    # [1,2,3] vs the direct exp/sum formula within 1e-9
    z = np.array([1.0, 2.0, 3.0])
    w = np.exp(z) / np.exp(z).sum()
    for i in range(3):
        Vd = bits((np.arange(3) == i).astype(np.float32).reshape(3, 1))
        o, _ = oracle.attention(bits(np.ones((1, 1), np.float32)), bits(z.astype(np.float32).reshape(3, 1)), Vd, 1,
                                np.arange(3, dtype=np.int32))
        assert abs(float(o[0, 0]) - w[i]) <= 1e-7               # fp32 output rounding


def test_lse_merge_of_disjoint_block_sets():
    # softmax over A u B from the two halves: m = max, l = sum l_s e^{m_s-m},
    # o = sum e^{m_s - m} l_s o_s / l  (the split-K merge)
    n, P, G = 640, 16, 4
    K, V = synth.segment_kv(8, 0, 0, 0, n)
    q = synth.queries(8, 0, 0, 0, G)[0]
    A = np.arange(0, 20, dtype=np.int32)
    B = np.arange(20, 40, dtype=np.int32)
    oa, la = oracle.attention(q, K, V, P, A)
    ob, lb = oracle.attention(q, K, V, P, B)
    o, l = oracle.attention(q, K, V, P, np.concatenate([A, B]))
    la, lb = la.astype(np.float64), lb.astype(np.float64)
    m = np.maximum(la, lb)
    wa, wb = np.exp(la - m), np.exp(lb - m)
    merged = (wa[:, None] * oa + wb[:, None] * ob) / (wa + wb)[:, None]
    assert np.allclose(merged, o, atol=2e-6)
    assert np.allclose(m + np.log(wa + wb), l, atol=2e-6)
