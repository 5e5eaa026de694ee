"""Test harness: drive libkvd (through its C ABI) and the CPU oracle on the same
seeded synthetic inputs, step by step, and compare.

The oracle side never sees anything the CUDA path produced: both sides start
from the synth generator's bytes; the oracle runs its own O1..O8.
"""
import numpy as np
import torch

import oracle
import synth
from paper_2605_18071_b200 import KVCache
from paper_2605_18071_b200.kvd import record_to_kv

ATTN_TOL = 2e-3      # north_star: <= 2e-3 max relative error (row-normwise, DESIGN.md §3 R18)
LSE_TOL = 1e-3


def row_normwise_err(o, ref):
    """max over rows of ||o - ref||_inf / ||ref||_inf (rows = (request, q-head))."""
    o = np.asarray(o, np.float64).reshape(-1, 128)
    ref = np.asarray(ref, np.float64).reshape(-1, 128)
    den = np.maximum(np.abs(ref).max(axis=1), 1e-30)
    return float((np.abs(o - ref).max(axis=1) / den).max())


class Case:
    def __init__(self, *, L=1, B=1, Hq=8, Hkv=2, n=4096, P=16, k=32, C=None, policy="lru", seed=0,
                 alpha=0.9, ragged=False, sink=4, local=64, alias=0, reqs=None, R=None, device=0,
                 fused=False, index_ratio=0, caps=None, summary="mean", extra=0, warm_obs=0):
        self.fused = fused            # kvd_select_resolve_fetch instead of select_topk + resolve_and_fetch
        self.index_ratio = index_ratio  # hierarchical centroid index (R27); 0 = flat
        self.L, self.B, self.Hq, self.Hkv, self.P, self.k = L, B, Hq, Hkv, P, k
        self.G = Hq // Hkv
        self.policy, self.pol = policy, oracle.POLICIES[policy]
        self.seed, self.alpha, self.sink, self.local = seed, alpha, sink, local
        self.reqs = list(range(B)) if reqs is None else list(reqs)
        R = R if R is not None else max(self.reqs) + 1
        self.n = {r: (n - 17 * r if ragged else n) for r in self.reqs}
        self.extra = extra                        # decode-time appends this case may make
        nb_max = (n + extra + P - 1) // P
        self.C = nb_max if C is None else C
        self.alias = alias
        self.cache = KVCache(num_layers=L, num_q_heads=Hq, num_kv_heads=Hkv, block_tokens=P, max_requests=R,
                             max_context=n + extra, slots_per_segment=self.C, max_select=k, sink_tokens=sink,
                             local_tokens=local, policy=policy, host_layer_alias=alias, device=device,
                             index_ratio=index_ratio, summary_kind=summary)
        self.summary = summary
        self.W = self.cache.attn_width(k)
        self.caps = dict(caps or {})              # 2D window scaling: (layer, head) -> slots (R28)
        for (l, h), cap in self.caps.items():
            self.cache.set_segment_capacity(l, h, cap)
        self.dev = torch.device("cuda", device)
        self.kv = {}
        self.oc = {}
        self.S = {}
        self.index = {}
        for l in range(L):
            for r in self.reqs:
                src_l = l % alias if alias else l
                K, V = synth.request_kv(seed, src_l, r, Hkv, self.n[r])
                qobs = None
                if warm_obs:
                    # the prompt's observation window: the query stream's first n_obs steps (the
                    # decode queries continue that stream, AR(1) temporal locality)
                    qobs = np.ascontiguousarray(np.concatenate(
                        [synth.queries(seed, l, r, h, self.G, nsteps=warm_obs, alpha=alpha).transpose(1, 0, 2)
                         for h in range(Hkv)], axis=0))                           # [Hq][n_obs][128]
                self.cache.load_prefix(l, r, K, V, self.n[r], q_obs=qobs)
                for h in range(Hkv):
                    self.kv[(l, r, h)] = (K[h], V[h])
                    self.S[(l, r, h)] = (oracle.block_summaries(K[h], P) if summary == "mean"
                                         else oracle.minmax_summaries(K[h], P))
                    if index_ratio:
                        cent, cent_of = oracle.index_build(self.S[(l, r, h)], index_ratio)
                        self.index[(l, r, h)] = (cent, cent_of, index_ratio)
                    pinned = oracle.pinned_blocks(self.n[r], P, sink, local)
                    self.oc[(l, r, h)] = oracle.SegmentCache(len(pinned), self.caps.get((l, h), self.C), pinned)
                    if warm_obs:
                        imp = oracle.warm_importance(qobs[h * self.G:(h + 1) * self.G], K[h], P)
                        oracle.warm_start(self.oc[(l, r, h)], imp)
        self.nl = {(l, r): self.n[r] for l in range(L) for r in self.reqs}   # tokens per (layer, request)
        self.last_scores = {}
        self.ids = torch.empty((B, Hkv, max(k, 1)), dtype=torch.int32, device=self.dev)
        self.sel_scores = torch.empty((B, Hkv, max(k, 1)), dtype=torch.float32, device=self.dev)
        self.attn = torch.empty((B, Hkv, self.W, 2), dtype=torch.int32, device=self.dev)
        self.out = torch.empty((B, Hq, 128), dtype=torch.float32, device=self.dev)
        self.lse = torch.empty((B, Hq), dtype=torch.float32, device=self.dev)

    def queries(self, l, t):
        return synth.batch_queries(self.seed, l, self.reqs, self.Hkv, self.G, t0=t, nsteps=1, alpha=self.alpha)[0]

    def gpu_layer(self, l, q_np, step):
        q = torch.from_numpy(q_np.view(np.int16)).to(self.dev)
        c = self.cache
        if self.fused:
            c.select_resolve_fetch(l, q, self.reqs, self.k, step, self.ids, self.attn, self.sel_scores)
        else:
            c.select_topk(l, q, self.reqs, self.k, self.ids, self.sel_scores)
            c.resolve_and_fetch(l, self.reqs, self.ids, self.k, step, self.attn)
        c.sparse_decode(l, q, self.reqs, self.attn, self.W, self.out, self.lse)
        torch.cuda.synchronize()
        c.check()
        return dict(ids=self.ids.cpu().numpy()[:, :, :self.k].copy(),
                    sel_scores=self.sel_scores.cpu().numpy()[:, :, :self.k].copy(),
                    attn=self.attn.cpu().numpy().copy(), out=self.out.cpu().numpy().copy(),
                    lse=self.lse.cpu().numpy().copy())

    def oracle_layer(self, l, q_np, step):
        res = {}
        for bi, r in enumerate(self.reqs):
            for h in range(self.Hkv):
                K, V = self.kv[(l, r, h)]
                qg = q_np[bi, h * self.G:(h + 1) * self.G]
                res[(bi, h)] = oracle.segment_step(self.oc[(l, r, h)], qg, self.S[(l, r, h)], K, V, self.P,
                                                   self.k, step, self.pol, self.W,
                                                   index=self.index.get((l, r, h)))
                self.last_scores[(l, r, h)] = res[(bi, h)]["scores"]
        return res

    def append(self, step):
        """Decode-time append of the next synthetic token of every request in every layer, on the
        GPU (kvd_append_token) and in the oracle (O13, with the layer's last select scores)."""
        import torch as _t
        for l in range(self.L):
            src_l = l % self.alias if self.alias else l
            knew = np.empty((self.B, self.Hkv, 128), np.uint16)
            vnew = np.empty_like(knew)
            for bi, r in enumerate(self.reqs):
                n = self.nl[(l, r)]
                Kf, Vf = synth.request_kv(self.seed, src_l, r, self.Hkv, n + 1)
                knew[bi], vnew[bi] = Kf[:, n], Vf[:, n]
            self.cache.append_token(l, self.reqs, _t.from_numpy(knew.view(np.int16)).to(self.dev),
                                    _t.from_numpy(vnew.view(np.int16)).to(self.dev), step)
            for bi, r in enumerate(self.reqs):
                n = self.nl[(l, r)]
                for h in range(self.Hkv):
                    K, V = self.kv[(l, r, h)]
                    nb = (n + self.P - 1) // self.P
                    sc = self.last_scores.get((l, r, h), np.zeros(nb, np.float32))
                    K, V, S, _ = oracle.append_token(self.oc[(l, r, h)], K, V, self.S[(l, r, h)], n, self.P,
                                                     knew[bi, h], vnew[bi, h], step, self.pol, sc, self.sink,
                                                     self.local, self.summary)
                    self.kv[(l, r, h)] = (K, V)
                    self.S[(l, r, h)] = S
                self.nl[(l, r)] = n + 1

    def compare_layer(self, l, g, o, check_state=True, check_slots=False):
        """Assert parity for one layer's outputs; returns the max attention error."""
        worst = 0.0
        for bi, r in enumerate(self.reqs):
            for h in range(self.Hkv):
                ref = o[(bi, h)]
                nb = len(ref["scores"])
                assert np.array_equal(g["ids"][bi, h], ref["ids"]), (l, r, h, "ids")
                if not self.index_ratio or self.policy == "la":   # index mode keeps lookahead scores only
                    sc = self.cache.read_scores(l, r, h, nb)
                    assert np.array_equal(sc.view(np.uint32), ref["scores"].view(np.uint32)) or \
                        np.array_equal(sc, ref["scores"]), (l, r, h, "scores")
                    assert np.array_equal(g["sel_scores"][bi, h], ref["scores"][ref["ids"]]), (l, r, h, "sel scores")
                assert np.array_equal(g["attn"][bi, h], ref["attn"]), (l, r, h, "attention list")
                if check_state:
                    st = self.cache.read_segment(l, r, h)
                    oc = self.oc[(l, r, h)]
                    assert np.array_equal(st["table"][:nb], oc.table), (l, r, h, "table")
                    Cs = len(oc.slot_block)                  # the segment's window (2D scaling)
                    assert np.array_equal(st["slot_block"][:Cs], oc.slot_block), (l, r, h, "slot map")
                    assert (st["slot_block"][Cs:] == -1).all(), (l, r, h, "slots beyond the window")
                    pin = oc.is_pinned
                    occ = (oc.slot_block >= 0)
                    occ &= ~pin[np.maximum(oc.slot_block, 0)].astype(bool)
                    assert np.array_equal(st["last_use"][:Cs][occ], oc.last_use[occ]), (l, r, h, "last_use")
                    assert np.array_equal(st["phase"][:Cs][occ], oc.phase[occ]), (l, r, h, "phase")
                    assert np.array_equal(st["use_count"][:Cs][occ], oc.use_count[occ]), (l, r, h, "use_count")
                if check_slots:
                    self.check_slot_bytes(l, r, h)
                G = self.G
                e = row_normwise_err(g["out"][bi, h * G:(h + 1) * G], ref["o"])
                worst = max(worst, e)
                assert e <= ATTN_TOL, (l, r, h, "attention err", e)
                assert np.max(np.abs(g["lse"][bi, h * G:(h + 1) * G] - ref["lse"])) <= LSE_TOL, (l, r, h, "lse")
        return worst

    def check_index(self):
        """O9 parity: every segment's centroids (bf16 bits) and block -> centroid map bit-exact."""
        for (l, r, h), (cent, cent_of, _) in self.index.items():
            gc, gof = self.cache.read_index(l, r, h, len(cent_of))
            assert gc.shape == cent.shape, (l, r, h, gc.shape, cent.shape)
            assert np.array_equal(gc, cent), (l, r, h, "centroids")
            assert np.array_equal(gof, cent_of), (l, r, h, "cent_of")

    def check_slot_bytes(self, l, r, h):
        """O7 invariant: every occupied slot holds exactly its block's K/V (from the generator)."""
        K, V = self.kv[(l, r, h)]
        st = self.cache.read_segment(l, r, h)
        n, P = self.nl[(l, r)], self.P
        for s, b in enumerate(st["slot_block"]):
            if b < 0:
                continue
            kk, vv = record_to_kv(self.cache.read_slot(l, r, h, s), P)
            cnt = min(P, n - P * b)
            assert np.array_equal(kk[:cnt], K[P * b:P * b + cnt]), (l, r, h, s, b, "slot K bytes")
            assert np.array_equal(vv[:cnt], V[P * b:P * b + cnt]), (l, r, h, s, b, "slot V bytes")
            assert not kk[cnt:].any() and not vv[cnt:].any()

    def run(self, steps, t0=0, check_state=True, check_slots_every=0, append_every=0):
        worst = 0.0
        for t in range(t0, t0 + steps):
            if append_every and t % append_every == 0:
                self.append(t + 1)
            for l in range(self.L):
                q = self.queries(l, t)
                g = self.gpu_layer(l, q, t + 1)
                o = self.oracle_layer(l, q, t + 1)
                cs = bool(check_slots_every) and (t % check_slots_every == 0)
                worst = max(worst, self.compare_layer(l, g, o, check_state, cs))
        return worst

    def hit_rate(self):
        s = self.cache.stats()
        return s["hits"] / max(1, s["selected"])
