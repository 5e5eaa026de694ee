"""CPU ORACLE for the KVDrive decode-step hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2605_18071_b200``) never imports it and shares no code with it.

This module is argument marshalling over ``kvd_oracle.c`` (plain C, -O2
-ffp-contract=off, no fast-math) plus ``segment_step``, which composes the
per-segment steps O1..O8 in the paper's order (PAPER.md:241-244, 386:
select via the index -> fetch the missing entries -> attend over resident and
fetched).  Every arithmetic step lives in the C file, each citing its passage.

Parity status: every function is pinned (tests/test_oracle_*.py); no function
here is "parity unpinned".
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libkvd_oracle.so")
_lib = None

LRU, LFU, LA = 0, 1, 2
POLICIES = {"lru": LRU, "lfu": LFU, "la": LA}
RECORD_TOKENS_DIMS = 2  # a block record is K[P][d] followed by V[P][d]


def build(force: bool = False) -> str:
    """Compile the oracle (plain C).  Building the checker is not using it."""
    src = os.path.join(_HERE, "kvd_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-shared", "-fPIC", "-o", _SO, src, "-lm"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        p, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        L.or_f32_to_bf16_rne.argtypes = [ctypes.c_float]
        L.or_f32_to_bf16_rne.restype = ctypes.c_uint16
        L.or_block_summaries.argtypes = [p, i64, i32, i32, p]
        L.or_block_summaries.restype = None
        L.or_group_query.argtypes = [p, i32, i32, p]
        L.or_group_query.restype = None
        L.or_block_scores.argtypes = [p, p, i64, i32, p]
        L.or_block_scores.restype = None
        L.or_pinned_blocks.argtypes = [i64, i32, i32, i32, p]
        L.or_pinned_blocks.restype = i64
        L.or_topk.argtypes = [p, i64, p, i32, p]
        L.or_topk.restype = i32
        L.or_cache_init.argtypes = [i64, i64, p, p, p, p, p, p]
        L.or_cache_init.restype = i32
        L.or_resolve.argtypes = [i64, i64, p, p, p, p, p, p, p, i32, u32, i32, p, i32, p, p, p, p]
        L.or_resolve.restype = i32
        L.or_fetch.argtypes = [p, p, i64, p, i32]
        L.or_fetch.restype = None
        L.or_attention.argtypes = [p, i32, i32, p, p, i64, i32, p, i32, p, p]
        L.or_attention.restype = None
        L.or_index_build.argtypes = [p, i64, i32, i32, p, p]
        L.or_index_build.restype = i64
        L.or_index_select.argtypes = [p, p, p, p, i64, i64, i32, p, i32, i32, p, p, p]
        L.or_index_select.restype = i32
        L.or_minmax_summaries.argtypes = [p, i64, i32, i32, p, p]
        L.or_minmax_summaries.restype = None
        L.or_minmax_scores.argtypes = [p, p, p, i64, i32, p]
        L.or_minmax_scores.restype = None
        L.or_append_block.argtypes = [i64, i64, p, p, p, p, p, p, u32, i32, p]
        L.or_append_block.restype = i32
        L.or_mckp_greedy.argtypes = [p, p, i32, i32, ctypes.c_double, p]
        L.or_mckp_greedy.restype = ctypes.c_double
        L.or_mckp_exact.argtypes = [p, p, i32, i32, ctypes.c_double, p]
        L.or_mckp_exact.restype = ctypes.c_double
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


def _c(a, dt):
    return np.ascontiguousarray(np.asarray(a, dtype=dt))


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what}: status {code}")
        self.code = code


# ---------------------------------------------------------------- O1..O5
def f32_to_bf16(x):
    """bf16 RNE bit patterns of float32 values (elementwise; O1's rounding)."""
    x = np.asarray(x, np.float32)
    f = lib().or_f32_to_bf16_rne
    return np.array([f(float(v)) for v in x.ravel()], np.uint16).reshape(x.shape)


def block_summaries(K, P):
    """O1: K [n][d] bf16 bits -> S [nb][d] bf16 bits."""
    K = _c(K, np.uint16)
    n, d = K.shape
    S = np.empty(((n + P - 1) // P, d), np.uint16)
    lib().or_block_summaries(_p(K), n, d, P, _p(S))
    return S


def group_query(q):
    """O2: q [G][d] bf16 bits -> qbar [d] float32."""
    q = _c(q, np.uint16)
    G, d = q.shape
    out = np.empty(d, np.float32)
    lib().or_group_query(_p(q), G, d, _p(out))
    return out


def block_scores(qbar, S):
    """O3: qbar [d] f32, S [nb][d] bf16 bits -> scores [nb] f32."""
    qbar = _c(qbar, np.float32)
    S = _c(S, np.uint16)
    nb, d = S.shape
    out = np.empty(nb, np.float32)
    lib().or_block_scores(_p(qbar), _p(S), nb, d, _p(out))
    return out


def pinned_blocks(n, P, sink=4, local=64):
    """O4: uint8 mask [nb] of the always-resident blocks."""
    nb = (n + P - 1) // P
    m = np.empty(nb, np.uint8)
    lib().or_pinned_blocks(n, P, sink, local, _p(m))
    return m


def topk(scores, is_pinned, k):
    """O5: k block ids, ascending."""
    scores = _c(scores, np.float32)
    is_pinned = _c(is_pinned, np.uint8)
    ids = np.empty(max(k, 1), np.int32)
    rc = lib().or_topk(_p(scores), len(scores), _p(is_pinned), k, _p(ids))
    if rc:
        raise OracleError(rc, "topk")
    return ids[:k]


# ---------------------------------------------------------------- O6..O7
class SegmentCache:
    """O6 state of one segment's GPU cache (table, slot map, metadata)."""

    def __init__(self, nb, C, is_pinned):
        self.nb, self.C = nb, C
        self.is_pinned = _c(is_pinned, np.uint8)
        self.table = np.empty(nb, np.int32)
        self.slot_block = np.empty(C, np.int32)
        self.last_use = np.empty(C, np.uint32)
        self.phase = np.empty(C, np.uint8)
        self.use_count = np.empty(C, np.uint32)
        rc = lib().or_cache_init(nb, C, _p(self.is_pinned), _p(self.table), _p(self.slot_block),
                                 _p(self.last_use), _p(self.phase), _p(self.use_count))
        if rc:
            raise OracleError(rc, "cache_init")

    def resolve(self, S, step, policy, scores, W):
        """O6: returns (attn [W][2], miss [k][2] (block, slot), n_miss, n_hit)."""
        S = _c(S, np.int32)
        k = len(S)
        attn = np.empty((W, 2), np.int32)
        miss = np.empty((max(k, 1), 2), np.int32)
        nm, nh = ctypes.c_int32(0), ctypes.c_int32(0)
        sc = _c(scores, np.float32) if scores is not None else None
        rc = lib().or_resolve(self.nb, self.C, _p(self.is_pinned), _p(self.table), _p(self.slot_block),
                              _p(self.last_use), _p(self.phase), _p(self.use_count), _p(S), k,
                              step, policy, _p(sc), W, _p(attn), _p(miss),
                              ctypes.byref(nm), ctypes.byref(nh))
        if rc:
            raise OracleError(rc, "resolve")
        return attn, miss[:k], nm.value, nh.value


def append_token(cache, K, V, S, n, P, k_new, v_new, step, policy, scores, sink=4, local=64, summary="mean"):
    """O13 + O1: append one token (k_new, v_new [d] bf16) at position n of a segment.
    Returns the new (K, V, S, pinned): the keys / values grown by one row, the summaries recomputed
    by O1 (O12 for min/max) over the grown keys, the pinned set of n + 1 tokens; the cache admits
    the new block when the token opens one (or_append_block)."""
    K = np.concatenate([K, np.asarray(k_new, np.uint16)[None, :]], axis=0)
    V = np.concatenate([V, np.asarray(v_new, np.uint16)[None, :]], axis=0)
    S = block_summaries(K, P) if summary == "mean" else minmax_summaries(K, P)
    pinned = pinned_blocks(n + 1, P, sink, local)
    nb_new = len(pinned)
    cache.is_pinned = _c(pinned, np.uint8)
    if nb_new > cache.nb:                          # the token opens block nb_new - 1
        cache.table = np.concatenate([cache.table, np.full(nb_new - cache.nb, -1, np.int32)])
        cache.nb = nb_new
        sc = _c(scores, np.float32) if scores is not None else None
        rc = lib().or_append_block(nb_new, cache.C, _p(cache.is_pinned), _p(cache.table), _p(cache.slot_block),
                                   _p(cache.last_use), _p(cache.phase), _p(cache.use_count), step, policy, _p(sc))
        if rc:
            raise OracleError(rc, "append_block")
    return K, V, S, pinned


def warm_importance(q_obs, K, P):
    """O14: importance of every block of a segment from the prompt's final
    observation window -- "for each query within this window, we compute its attention weights
    over all prefix keys and aggregate them across heads" -- in fp64 from the bf16 inputs:
    I_b = sum over the G x n_obs queries q of sum over tokens t of block b of softmax_t(q.K_t / sqrt(d)).
    q_obs [G][n_obs][d], K [n][d] bf16 bits -> I [nb] float64."""
    Q = _f64(q_obs).reshape(-1, q_obs.shape[-1])
    Kf = _f64(K)
    z = Q @ Kf.T / np.sqrt(Kf.shape[1])
    w = np.exp(z - z.max(axis=1, keepdims=True))
    w /= w.sum(axis=1, keepdims=True)
    tok = w.sum(axis=0)
    nb = (Kf.shape[0] + P - 1) // P
    return np.array([tok[P * b:P * b + P].sum() for b in range(nb)])


def warm_start(cache, importance):
    """O14 placement (reading R29): a host-backed segment cache starts with its C - pinned most
    important non-pinned blocks resident (importance desc, block id asc), in the slots after the
    pinned blocks, ascending by block id; last use 0, phase 1, count 1.  A fully resident cache is
    unchanged."""
    nb, C = cache.nb, cache.C
    if C >= nb:
        return np.zeros(0, np.int32)
    pin = cache.is_pinned.astype(bool)
    cand = np.nonzero(~pin)[0]
    room = C - int(pin.sum())
    order = np.lexsort((cand, -importance[cand]))
    chosen = np.sort(cand[order[:room]]).astype(np.int32)
    s = int(pin.sum())
    for b in chosen:
        cache.table[b] = s
        cache.slot_block[s] = b
        cache.last_use[s], cache.phase[s], cache.use_count[s] = 0, 1, 1
        s += 1
    return chosen


def _f64(bits):
    return (np.asarray(bits, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def fetch(host_records, slot_pool, miss, n_miss):
    """O7: slot_pool[slot] := host_records[block] for each miss (in place)."""
    assert host_records.flags.c_contiguous and slot_pool.flags.c_contiguous
    rb = host_records.strides[0]
    miss = _c(miss, np.int32)
    lib().or_fetch(_p(host_records), _p(slot_pool), rb, _p(miss), n_miss)


# ---------------------------------------------------------------- O8
def attention(q, K, V, P, blocks):
    """O8: q [G][d], K/V [n][d] bf16 bits, blocks (ids, -1 ignored) ->
    (o [G][d] f32, lse [G] f32), fp64 inside."""
    q = _c(q, np.uint16)
    K = _c(K, np.uint16)
    V = _c(V, np.uint16)
    blocks = _c(blocks, np.int32)
    G, d = q.shape
    o = np.empty((G, d), np.float32)
    lse = np.empty(G, np.float32)
    lib().or_attention(_p(q), G, d, _p(K), _p(V), K.shape[0], P, _p(blocks), len(blocks), _p(o), _p(lse))
    return o, lse


# ---------------------------------------------------------------- O9..O10 hierarchical index
IDX_WINDOW = 64        # blocks per k-means window (OR_IDX_WIN)
IDX_FANOUT = 4         # stage 1 keeps ceil(IDX_FANOUT * k / ratio) centroids (reading R27)


def index_build(S, ratio):
    """O9: block summaries S [nb][d] bf16 -> (centroids [nc][d] bf16, cent_of [nb] int32)."""
    S = _c(S, np.uint16)
    nb, d = S.shape
    cent = np.empty((max(nb, 1), d), np.uint16)
    cent_of = np.empty(max(nb, 1), np.int32)
    nc = lib().or_index_build(_p(S), nb, d, ratio, _p(cent), _p(cent_of))
    return cent[:nc].copy(), cent_of[:nb].copy()


def index_fanout(k, ratio, nc, pinned):
    """Stage-1 centroid count m for top-k (reading R27): ceil(IDX_FANOUT * k / ratio), at least
    k + pinned (every centroid has a member, so the m best centroids then hold >= k non-pinned
    members and stage 2 always has k candidates), at most nc."""
    return min(nc, max(-(-IDX_FANOUT * k // ratio), k + int(pinned)))


def index_select(qbar, S, cent, cent_of, is_pinned, k, m):
    """O10: (ids [k] ascending, centroid scores [nc], lookahead scores [nb])."""
    qbar = _c(qbar, np.float32)
    S = _c(S, np.uint16)
    cent = _c(cent, np.uint16)
    cent_of = _c(cent_of, np.int32)
    is_pinned = _c(is_pinned, np.uint8)
    nb, d = S.shape
    nc = cent.shape[0]
    ids = np.empty(max(k, 1), np.int32)
    cs = np.empty(max(nc, 1), np.float32)
    la = np.empty(max(nb, 1), np.float32)
    rc = lib().or_index_select(_p(qbar), _p(S), _p(cent), _p(cent_of), nb, nc, d, _p(is_pinned), k, m,
                               _p(ids), _p(cs), _p(la))
    if rc:
        raise OracleError(rc, "index_select")
    return ids[:k], cs[:nc], la[:nb]


# ---------------------------------------------------------------- O12 Quest min/max summaries
def minmax_summaries(K, P):
    """O12: K [n][d] bf16 -> (MN, MX) [nb][d] bf16: channel-wise min / max of each block."""
    K = _c(K, np.uint16)
    n, d = K.shape
    nb = (n + P - 1) // P
    MN = np.empty((nb, d), np.uint16)
    MX = np.empty((nb, d), np.uint16)
    lib().or_minmax_summaries(_p(K), n, d, P, _p(MN), _p(MX))
    return MN, MX


def minmax_scores(qbar, MN, MX):
    """O12: Quest upper-bound scores [nb] f32."""
    qbar = _c(qbar, np.float32)
    MN = _c(MN, np.uint16)
    MX = _c(MX, np.uint16)
    nb, d = MN.shape
    out = np.empty(nb, np.float32)
    lib().or_minmax_scores(_p(qbar), _p(MN), _p(MX), nb, d, _p(out))
    return out


# ---------------------------------------------------------------- O11 2D window scaling (MCKP)
def mckp(benefit, cost, budget, exact=False):
    """O11: (total benefit, choice [pairs]) for benefit / cost [pairs][sizes];
    greedy by benefit-to-cost ratio, or exhaustive (exact=True, tiny instances)."""
    b = _c(benefit, np.float64)
    c = _c(cost, np.float64)
    pairs, sizes = b.shape
    choice = np.empty(pairs, np.int32)
    f = lib().or_mckp_exact if exact else lib().or_mckp_greedy
    tot = f(_p(b), _p(c), pairs, sizes, float(budget), _p(choice))
    if tot < 0:
        raise OracleError(-1, "mckp (infeasible or too large)")
    return tot, choice


# ---------------------------------------------------------------- composition
def segment_select(q_group, S, is_pinned, k):
    """O2 -> O3 -> O5 for one segment: returns (ids, scores)."""
    scores = block_scores(group_query(q_group), S)
    return topk(scores, is_pinned, k), scores


def segment_step(cache, q_group, S, K, V, P, k, step, policy, W, index=None):
    """One decode step of one segment, in the paper's order (PAPER.md:241-244,
    386): select (O2,O3,O5; or the hierarchical index O9-O10 when index =
    (centroids, cent_of, ratio)) -> resolve (O6) -> attend (O8).  Returns a dict."""
    if isinstance(S, tuple):                      # Quest min/max summaries (O12)
        scores = minmax_scores(group_query(q_group), S[0], S[1])
        ids = topk(scores, cache.is_pinned, k)
    elif index is None:
        ids, scores = segment_select(q_group, S, cache.is_pinned, k)
    else:
        cent, cent_of, ratio = index
        ids, _, scores = index_select(group_query(q_group), S, cent, cent_of, cache.is_pinned, k,
                                      index_fanout(k, ratio, cent.shape[0], cache.is_pinned.sum()))
    attn, miss, nm, nh = cache.resolve(ids, step, policy, scores, W)
    o, lse = attention(q_group, K, V, P, attn[:, 0])
    return dict(ids=ids, scores=scores, attn=attn, miss=miss, n_miss=nm, n_hit=nh, o=o, lse=lse)
