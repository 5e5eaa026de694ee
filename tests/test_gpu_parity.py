"""GPU parity: libkvd (through the C ABI) vs the CPU oracle, element by element.

Bar (north_star): selected ids, block scores, attention lists, block tables,
slot maps and slot metadata bit-exact; attention output <= 2e-3 row-normwise
relative error; every occupied slot byte-identical to its block's K/V.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_harness import Case, row_normwise_err
from paper_2605_18071_b200 import KVDError

pytestmark = pytest.mark.gpu


def test_c1_resident_full_parity():
    # BASELINE configs[0]: 1 request, 1 layer, 8q/2kv, 4k ctx, block 16, top-k 32, resident
    c = Case(L=1, B=1, Hq=8, Hkv=2, n=4096, P=16, k=32)
    assert c.cache.resident
    c.run(steps=6, check_slots_every=3)
    s = c.cache.stats()
    assert s["misses"] == 0 and s["hits"] == s["selected"] == 6 * 2 * 32


def test_summaries_bit_exact():
    c = Case(L=2, B=2, Hq=8, Hkv=2, n=1000, P=16, k=8, ragged=True)
    for (l, r, h), S in c.S.items():
        assert np.array_equal(c.cache.read_summaries(l, r, h, S.shape[0]), S), (l, r, h)


@pytest.mark.parametrize("policy", ["lru", "lfu", "la"])
@pytest.mark.parametrize("alpha", [0.9, 0.0])
def test_c1_evict_slot_maps(policy, alpha):
    # c1-evict: C = 64 + 5 slots (window x2 for k = 32), host-backed, 24 steps
    c = Case(L=1, B=1, Hq=8, Hkv=2, n=4096, P=16, k=32, C=69, policy=policy, alpha=alpha, seed=3)
    assert not c.cache.resident
    c.run(steps=24, check_slots_every=6)
    s = c.cache.stats()
    assert s["misses"] > 0 and s["fetched_bytes"] == s["misses"] * 8192


def test_ragged_multi_layer_multi_request_la():
    c = Case(L=2, B=3, Hq=8, Hkv=2, n=3000, P=16, k=20, C=60, policy="la", ragged=True, seed=5)
    c.run(steps=8, check_slots_every=4)


def test_noncontiguous_request_ids():
    c = Case(L=1, B=3, Hq=8, Hkv=2, n=2048, P=16, k=16, C=40, policy="lru", reqs=[4, 1, 6], R=8, seed=6)
    c.run(steps=5)


@pytest.mark.parametrize("P,n,k,C", [(1, 600, 64, None), (2, 700, 40, 100), (4, 1000, 40, 90), (8, 1500, 30, 70)])
def test_block_sizes(P, n, k, C):
    c = Case(L=1, B=2, Hq=8, Hkv=2, n=n, P=P, k=k, C=C, policy="lru", ragged=True, seed=7)
    c.run(steps=4, check_slots_every=2)


def test_qwen_group_of_seven_lfu():
    # Qwen2.5-7B-1M head grouping: 28q / 4kv (G = 7), shrunk to 14q / 2kv
    c = Case(L=1, B=2, Hq=14, Hkv=2, n=2048, P=16, k=24, C=48, policy="lfu", seed=8)
    c.run(steps=6)


def test_k_all_candidates_is_dense_attention():
    n, P = 1024, 16
    nb = n // P
    c = Case(L=1, B=1, Hq=8, Hkv=2, n=n, P=P, k=nb - 5, seed=9)
    q = c.queries(0, 0)
    g = c.gpu_layer(0, q, 1)
    for h in range(2):
        K, V = c.kv[(0, 0, h)]
        o, lse = oracle.attention(q[0, 4 * h:4 * h + 4], K, V, P, np.arange(nb, dtype=np.int32))
        assert row_normwise_err(g["out"][0, 4 * h:4 * h + 4], o) <= 2e-3
        assert np.allclose(g["lse"][0, 4 * h:4 * h + 4], lse, atol=1e-3)


def test_k_zero_attends_pinned_only():
    c = Case(L=1, B=1, Hq=8, Hkv=2, n=1000, P=16, k=0, C=10, seed=10)
    c.run(steps=2)


def test_abi_errors_and_device_flag():
    c = Case(L=1, B=1, Hq=8, Hkv=2, n=512, P=16, k=8, C=20, seed=11)
    q = torch.zeros((1, 8, 128), dtype=torch.int16, device="cuda")
    ids = torch.zeros((1, 2, 40), dtype=torch.int32, device="cuda")
    with pytest.raises(KVDError) as e:                                  # 32 blocks - 5 pinned = 27 candidates
        c.cache.select_topk(0, q, [0], 28, ids)
    assert e.value.status in ("KVD_EINVAL", "KVD_ERANGE")
    with pytest.raises(KVDError) as e:
        c.cache.select_topk(0, q, [0, 0], 4, ids)                      # repeated request
    assert e.value.status == "KVD_EINVAL"
    with pytest.raises(KVDError) as e:
        c.cache.select_topk(1, q, [0], 4, ids)                         # bad layer
    assert e.value.status == "KVD_EINVAL"
    # capacity: k + pinned > C
    c2 = Case(L=1, B=1, Hq=8, Hkv=2, n=512, P=16, k=16, C=20, seed=11)
    with pytest.raises(KVDError) as e:
        c2.cache.select_topk(0, q, [0], 16, ids)
    assert e.value.status == "KVD_ECAPACITY"
    # a non-ascending id list is flagged on the device, reported by kvd_check
    bad = torch.tensor([[[9, 3, 4, 5, 6, 7, 8, 10], [1, 2, 3, 4, 5, 6, 7, 8]]], dtype=torch.int32, device="cuda")
    attn = torch.empty((1, 2, c.W, 2), dtype=torch.int32, device="cuda")
    c.cache.resolve_and_fetch(0, [0], bad, 8, 1, attn)
    with pytest.raises(KVDError) as e:
        c.cache.check()
    assert e.value.status == "KVD_EDEVICE"
    assert (attn[0, 0].cpu().numpy() == -1).all()
    c.cache.check()                                                     # flag cleared


def test_hit_rate_reported_and_plausible():
    # workload property, not a parity criterion: window x2, alpha 0.9
    c = Case(L=1, B=2, Hq=8, Hkv=2, n=8192, P=16, k=32, C=69, policy="la", seed=12)
    c.run(steps=20, check_state=False)
    hr = c.hit_rate()
    assert 0.3 < hr < 1.0, hr


def test_deterministic_across_runs():
    a = Case(L=1, B=2, Hq=8, Hkv=2, n=2048, P=16, k=16, C=40, policy="la", seed=13)
    b = Case(L=1, B=2, Hq=8, Hkv=2, n=2048, P=16, k=16, C=40, policy="la", seed=13)
    for t in range(5):
        q = a.queries(0, t)
        ga, gb = a.gpu_layer(0, q, t + 1), b.gpu_layer(0, q, t + 1)
        for key in ("ids", "attn"):
            assert np.array_equal(ga[key], gb[key])
        assert np.array_equal(ga["out"], gb["out"])


# ---- top-k cluster geometries (k_select.cu topk_geometry): P = 1 makes blocks == tokens, so
# the segment spans 1, 2, 4 and 8 CTAs of the selection cluster; every id, score and list is
# compared with the oracle's sort-based top-k (O3).
@pytest.mark.parametrize("n", [3000, 9000, 20000, 40000])
def test_topk_cluster_spans(n):
    c = Case(L=1, B=2, Hq=8, Hkv=2, n=n, P=1, k=96, seed=21, ragged=True)
    c.run(steps=2)


def _bf16(x):
    return (np.asarray(x, np.float32).view(np.uint32) >> 16).astype(np.uint16)


@pytest.mark.parametrize("mode,n,P", [("zero", 16384, 16), ("one_dim", 16384, 16), ("zero", 40000, 1),
                                      ("one_dim", 40000, 1)])
def test_topk_ties_lowest_id(mode, n, P):
    """R10 ties: a zero query makes every score +0 (all keys equal: the k lowest candidate ids);
    a query on one dim makes scores = one bf16 summary coordinate (many exact ties inside the
    threshold bin).  P = 1 at n = 40,000: a 4-CTA cluster whose threshold bin overflows the
    compacted list (full-scan digits and emission)."""
    c = Case(L=1, B=2, Hq=8, Hkv=2, n=n, P=P, k=128, C=300 if P == 16 else 2000, policy="la", seed=22)

    def queries(l, t):
        q = np.zeros((c.B, c.Hq, 128), np.float32)
        if mode == "one_dim":
            q[:, :, 0] = 1.0 + t
        return _bf16(q)
    c.queries = queries
    c.run(steps=3)
    if mode == "zero":
        ids = c.ids.cpu().numpy()
        first = -(-4 // P)                                        # sink blocks are pinned
        assert (ids[:, :, :c.k] == np.arange(first, first + c.k)).all()


# ---- the fused select + resolve + fetch call (kvd_select_resolve_fetch) against the oracle:
# same decisions, slot maps, metadata, slot bytes and attention as the two separate calls
@pytest.mark.parametrize("policy", ["lru", "lfu", "la"])
def test_fused_select_resolve_fetch_evict(policy):
    c = Case(L=1, B=2, Hq=8, Hkv=2, n=4096, P=16, k=32, C=69, policy=policy, alpha=0.0, seed=31, fused=True)
    c.run(steps=8, check_slots_every=2)


@pytest.mark.parametrize("n,P,C", [(3000, 16, 60), (20000, 1, None), (40000, 1, 2000)])
def test_fused_ragged_and_cluster_spans(n, P, C):
    c = Case(L=2, B=3, Hq=8, Hkv=2, n=n, P=P, k=40, C=C, policy="la", ragged=True, seed=32, fused=True)
    c.run(steps=3)


def test_fused_k_zero_and_group_of_seven():
    Case(L=1, B=1, Hq=8, Hkv=2, n=1000, P=16, k=0, C=10, seed=33, fused=True).run(steps=2)
    Case(L=1, B=2, Hq=14, Hkv=2, n=2048, P=16, k=24, C=48, policy="lfu", seed=34, fused=True).run(steps=4)


# ---- degenerate and maximum shapes
@pytest.mark.parametrize("n,k", [(1, 0), (40, 0), (68, 0), (69, 0), (100, 1), (129, 2)])
def test_tiny_contexts_all_or_mostly_pinned(n, k):
    """n <= sink + local pins every block (no candidates, k = 0); slightly longer contexts leave
    one or two candidates; partial last blocks everywhere."""
    for fused in (False, True):
        c = Case(L=1, B=2, Hq=8, Hkv=2, n=n, P=16, k=k, C=None, seed=41, ragged=False, fused=fused)
        c.run(steps=2)


@pytest.mark.parametrize("fused", [False, True])
def test_max_batch_many_segments(fused):
    """KVD_MAX_BATCH requests x 8 KV heads = 2048 segments per call: more segments than attention
    workers, so most workers finalise whole segments in place; host-backed with evictions."""
    c = Case(L=1, B=256, Hq=32, Hkv=8, n=600, P=16, k=8, C=20, policy="lru", seed=42, fused=fused)
    c.run(steps=2, check_state=True)


# ---- a cluster whose CTAs disagree on whether their threshold-bin list fits:
# one outlier score stretches the linear first digit so that almost every candidate lands in the
# threshold bin; the 4-CTA cluster's full CTAs overflow the 4096-entry list while its short last
# CTA does not.  Keys are (nearly) distinct, so the LIST / WHOLE modes run, not EQUAL.
@pytest.mark.parametrize("fused", [False, True])
def test_topk_cluster_mixed_list_overflow(monkeypatch, fused):
    n, P = 40000, 1

    def fake_request_kv(seed, layer, req, Hkv, n_, d=128, out_k=None, out_v=None):
        rng = np.random.default_rng(1000 + 10 * req + layer)
        K = np.zeros((Hkv, n_, d), np.float32)
        K[:, :, 0] = rng.standard_normal((Hkv, n_)).astype(np.float32)
        K[:, :, 1] = rng.standard_normal((Hkv, n_)).astype(np.float32)
        K[:, 5000, 0] = 3.0e4                                      # the outlier (CTA 0)
        V = rng.standard_normal((Hkv, n_, d)).astype(np.float32)
        return _bf16(K), _bf16(V)
    monkeypatch.setattr(synth, "request_kv", fake_request_kv)
    c = Case(L=1, B=2, Hq=8, Hkv=2, n=n, P=P, k=96, C=None, policy="la", seed=23, ragged=True, fused=fused)

    def queries(l, t):
        q = np.zeros((c.B, c.Hq, 128), np.float32)
        q[:, :, 0] = 1.0
        q[:, :, 1] = 0.25 * (t + 1)                                # dim 1 makes the keys distinct
        return _bf16(q)
    c.queries = queries
    c.run(steps=2)


# ---- the general top-k path (self-scoring select_kernel): a cluster whose candidates would not
# fit rank 0's candidate area (k x cluster size > 8192) -- P = 1, 40,000 blocks in a cluster of 8,
# k = 2000 -- resident and host-backed, both call paths
@pytest.mark.parametrize("fused,C", [(False, None), (True, None), (True, 3000), (False, 3000)])
def test_general_select_path_large_k(fused, C):
    c = Case(L=1, B=2, Hq=8, Hkv=2, n=40000, P=1, k=2000, C=C, policy="la", seed=24, ragged=True, fused=fused)
    c.run(steps=2)


# ---- the split-K plan is a function of the segment (its k) only: a request attended alone and
# the same request inside a 16-request call give bit-identical outputs
@pytest.mark.parametrize("fused", [False, True])
def test_attention_bitwise_independent_of_batch(fused):
    alone = Case(L=1, B=1, Hq=8, Hkv=2, n=8192, P=16, k=128, C=None, seed=24, reqs=[5], R=16, fused=fused)
    batch = Case(L=1, B=16, Hq=8, Hkv=2, n=8192, P=16, k=128, C=None, seed=24, fused=fused)
    for t in range(2):
        ga = alone.gpu_layer(0, alone.queries(0, t), t + 1)
        gb = batch.gpu_layer(0, batch.queries(0, t), t + 1)
        assert np.array_equal(ga["ids"][0], gb["ids"][5])
        assert np.array_equal(ga["out"][0].view(np.uint32), gb["out"][5].view(np.uint32))
        assert np.array_equal(ga["lse"][0].view(np.uint32), gb["lse"][5].view(np.uint32))


# ---- the hierarchical centroid index (R27; k_index.cu): the k-means build bit-exact against the
# oracle's O9 (centroid bf16 bits, block -> centroid), then select / resolve / attention as usual
@pytest.mark.parametrize("ratio,policy,fused", [(4, "la", False), (4, "la", True), (2, "lru", True),
                                                (8, "lfu", False), (1, "la", True)])
def test_hierarchical_index_parity(ratio, policy, fused):
    c = Case(L=1, B=2, Hq=8, Hkv=2, n=20000, P=16, k=32, C=200, policy=policy, seed=51, ragged=True,
             fused=fused, index_ratio=ratio)
    c.check_index()
    c.run(steps=4, check_slots_every=2)


def test_hierarchical_index_full_context_cluster_stage1():
    # a 1M-token segment (65536 blocks, 16384 centroids): stage 1 on an 8-CTA cluster, k = 128
    c = Case(L=1, B=1, Hq=14, Hkv=2, n=1 << 20, P=16, k=128, C=4096, policy="la", seed=52, fused=True,
             index_ratio=4)
    c.check_index()
    c.run(steps=2)


# ---- 2D layer-head window scaling (R28): heterogeneous per layer-head capacities; slot maps
# bit-exact against oracle caches of those capacities, nothing ever placed beyond a window
@pytest.mark.parametrize("policy,fused", [("la", True), ("lru", False), ("lfu", True)])
def test_window_scaling_heterogeneous_capacities(policy, fused):
    caps = {(0, 0): 40, (0, 1): 90, (1, 0): 160, (1, 1): 45}
    c = Case(L=2, B=2, Hq=8, Hkv=2, n=6000, P=16, k=32, C=160, policy=policy, seed=61, ragged=True,
             fused=fused, caps=caps)
    c.run(steps=10, check_slots_every=3)
    sel, mis = c.cache.segment_stats()
    assert sel.sum() == c.cache.stats()["selected"] and mis.sum() == c.cache.stats()["misses"]
    assert mis[0, 0] > mis[1, 0]                  # the small window misses more


def test_window_scaling_shrink_and_errors():
    c = Case(L=1, B=1, Hq=8, Hkv=2, n=4096, P=16, k=32, C=120, policy="la", seed=62)
    c.run(steps=4)
    c.cache.set_segment_capacity(0, 1, 50)        # shrink: residents of slots >= 50 are dropped
    st = c.cache.read_segment(0, 0, 1)
    assert (st["slot_block"][50:] == -1).all()
    assert all(st["table"][b] < 50 for b in np.nonzero(st["table"] >= 0)[0])
    with pytest.raises(KVDError) as e:
        c.cache.set_segment_capacity(0, 0, 3)     # below the pinned blocks
    assert e.value.status == "KVD_EINVAL"
    c.cache.set_segment_capacity(0, 0, 36)        # 32 + 5 pinned do not fit in 36
    q = torch.zeros((1, 8, 128), dtype=torch.int16, device="cuda")
    ids = torch.zeros((1, 2, 32), dtype=torch.int32, device="cuda")
    with pytest.raises(KVDError) as e:
        c.cache.select_topk(0, q, [0], 32, ids)
    assert e.value.status == "KVD_ECAPACITY"


# ---- Quest min/max summaries (R30), the paper's comparison baseline as a second selection
# workload: summaries bit-exact, selection / resolve / attention as usual
def test_minmax_summaries_bit_exact():
    c = Case(L=1, B=2, Hq=8, Hkv=2, n=1000, P=16, k=8, ragged=True, summary="minmax")
    for (l, r, h), (mn, mx) in c.S.items():
        gmn, gmx = c.cache.read_minmax(l, r, h, mn.shape[0])
        assert np.array_equal(gmn, mn) and np.array_equal(gmx, mx), (l, r, h)


@pytest.mark.parametrize("n,P,C,policy,fused", [(4096, 16, 69, "la", True), (3000, 16, 60, "lru", False),
                                                (40000, 1, 2000, "la", True), (2000, 4, None, "lfu", False)])
def test_minmax_select_parity(n, P, C, policy, fused):
    c = Case(L=1, B=2, Hq=8, Hkv=2, n=n, P=P, k=32, C=C, policy=policy, seed=71, ragged=True, fused=fused,
             summary="minmax")
    c.run(steps=4, check_slots_every=2)


# ---- decode-time append (R16, O13): tokens join the local window, new blocks are admitted,
# summaries follow; selection / slot maps / attention stay bit-exact with the oracle
@pytest.mark.parametrize("C,policy,fused,summary", [(None, "la", True, "mean"), (60, "la", True, "mean"),
                                                   (60, "lru", False, "mean"), (70, "lfu", True, "minmax")])
def test_append_tokens(C, policy, fused, summary):
    c = Case(L=2, B=2, Hq=8, Hkv=2, n=1000, P=16, k=24, C=C, policy=policy, seed=81, ragged=True, fused=fused,
             summary=summary, extra=48)
    c.run(steps=40, append_every=1, check_slots_every=5)
    assert all(v == c.n[r] + 40 for (l, r), v in c.nl.items())


def test_append_errors():
    c = Case(L=1, B=1, Hq=8, Hkv=2, n=500, P=16, k=8, C=40, seed=82, extra=1)
    c.append(1)
    k = torch.zeros((1, 2, 128), dtype=torch.int16, device="cuda")
    with pytest.raises(KVDError) as e:
        c.cache.append_token(0, [0], k, k, 2)                    # context full
    assert e.value.status == "KVD_ERANGE"


# ---- importance-guided warm-up (R29, O14): the initial residency is the oracle's (slot map
# bit-exact right after the prefix load), then every step as usual; warm starts miss less
@pytest.mark.parametrize("policy,fused,caps", [("la", True, None), ("lru", False, {(0, 1): 40})])
def test_warm_start(policy, fused, caps):
    c = Case(L=1, B=2, Hq=8, Hkv=2, n=6000, P=16, k=24, C=69, policy=policy, seed=91, ragged=True, fused=fused,
             warm_obs=16, caps=caps)
    for (l, r, h), oc in c.oc.items():
        st = c.cache.read_segment(l, r, h)
        assert np.array_equal(st["slot_block"][:len(oc.slot_block)], oc.slot_block), (l, r, h, "warm slot map")
        assert np.array_equal(st["table"][:oc.nb], oc.table), (l, r, h, "warm table")
    c.run(steps=6, check_slots_every=3)
    cold = Case(L=1, B=2, Hq=8, Hkv=2, n=6000, P=16, k=24, C=69, policy=policy, seed=91, ragged=True, fused=fused,
                caps=caps)
    cold.run(steps=6, check_state=False)
    assert c.cache.stats()["misses"] < cold.cache.stats()["misses"]
