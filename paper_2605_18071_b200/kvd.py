"""ctypes binding of libkvd.so — same names as include/kvd.h, marshalling only.

Tensors are passed as raw pointers: torch tensors (device or pinned host) via
``data_ptr()``, numpy arrays via their buffer address.  Streams are raw
``cudaStream_t`` handles (``torch.cuda.Stream.cuda_stream``).  Every non-OK
status raises KVDError carrying kvd_last_error().
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkvd.so")

POLICY = {"lru": 0, "lfu": 1, "la": 2, "lookahead": 2}
SUMMARY_KIND = {"mean": 0, "minmax": 1}
STATUS = {0: "KVD_OK", 1: "KVD_EINVAL", 2: "KVD_ERANGE", 3: "KVD_ECAPACITY", 4: "KVD_ENOMEM",
          5: "KVD_ECUDA", 6: "KVD_EDEVICE", 7: "KVD_ESTATE"}
KVD_MAX_BATCH = 256


class KVDError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class Config(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("block_tokens", ctypes.c_int32), ("max_requests", ctypes.c_int32),
                ("max_context", ctypes.c_int64), ("slots_per_segment", ctypes.c_int64),
                ("max_select", ctypes.c_int32), ("sink_tokens", ctypes.c_int32),
                ("local_tokens", ctypes.c_int32), ("policy", ctypes.c_int32),
                ("host_layer_alias", ctypes.c_int32), ("device", ctypes.c_int32), ("index_ratio", ctypes.c_int32),
                ("summary_kind", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("selected", ctypes.c_uint64), ("hits", ctypes.c_uint64), ("misses", ctypes.c_uint64),
                ("pinned", ctypes.c_uint64), ("fetched_bytes", ctypes.c_uint64)]

    def asdict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


class Info(ctypes.Structure):
    _fields_ = [("nb_max", ctypes.c_int64), ("nb_pad", ctypes.c_int64), ("slots_per_segment", ctypes.c_int64),
                ("max_pinned", ctypes.c_int32), ("record_bytes", ctypes.c_int32), ("resident", ctypes.c_int32),
                ("host_layers", ctypes.c_int32)]


_lib = None
EXPORTS = ["kvd_required_bytes", "kvd_create_cache", "kvd_destroy_cache", "kvd_get_info", "kvd_attn_width",
           "kvd_load_prefix", "kvd_select_topk", "kvd_resolve_and_fetch", "kvd_sparse_decode",
           "kvd_read_segment", "kvd_read_slot", "kvd_read_host_record", "kvd_read_summaries",
           "kvd_read_scores", "kvd_get_stats", "kvd_reset_stats", "kvd_check", "kvd_last_error",
           "kvd_version", "kvd_set_device_step", "kvd_launch_count",
           "kvd_select_resolve_fetch", "kvd_select_resolve_fetch_heads", "kvd_sparse_decode_heads",
           "kvd_enable_kernel_timer", "kvd_read_kernel_timer",
           "kvd_probe_zero_copy", "kvd_read_index", "kvd_set_segment_capacity", "kvd_get_segment_stats",
           "kvd_plan_window_scaling", "kvd_read_minmax", "kvd_append_token", "kvd_load_prefix_obs",
           "kvd_read_warm_importance"]


def lib():
    """Load libkvd.so (fails loudly if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        p, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        sig = {
            "kvd_required_bytes": ([p, p, p], i32),
            "kvd_create_cache": ([p, p], i32),
            "kvd_destroy_cache": ([p], None),
            "kvd_get_info": ([p, p], i32),
            "kvd_set_device_step": ([p, p], i32),
            "kvd_attn_width": ([p, i32], i32),
            "kvd_load_prefix": ([p, i32, i32, p, p, i64, p], i32),
            "kvd_select_topk": ([p, i32, p, p, i32, i32, p, p, p], i32),
            "kvd_resolve_and_fetch": ([p, i32, p, i32, p, i32, u32, p, p], i32),
            "kvd_sparse_decode": ([p, i32, p, p, i32, p, i32, p, p, p], i32),
            "kvd_read_segment": ([p, i32, i32, i32, p, p, p, p, p], i32),
            "kvd_read_slot": ([p, i32, i32, i32, i64, p], i32),
            "kvd_read_host_record": ([p, i32, i32, i32, i64, p], i32),
            "kvd_read_summaries": ([p, i32, i32, i32, p], i32),
            "kvd_read_scores": ([p, i32, i32, i32, p], i32),
            "kvd_get_stats": ([p, p], i32),
            "kvd_reset_stats": ([p], i32),
            "kvd_check": ([p], i32),
            "kvd_last_error": ([], ctypes.c_char_p),
            "kvd_version": ([], ctypes.c_char_p),
            "kvd_launch_count": ([], ctypes.c_uint64),
            "kvd_select_resolve_fetch": ([p, i32, p, p, i32, i32, u32, p, p, p, p], i32),
            "kvd_select_resolve_fetch_heads": ([p, i32, p, p, i32, i32, i32, i32, u32, p, p, p, p], i32),
            "kvd_sparse_decode_heads": ([p, i32, p, p, i32, i32, i32, p, i32, p, p, p], i32),
            "kvd_enable_kernel_timer": ([p, i32], i32),
            "kvd_read_kernel_timer": ([p, p, p], i32),
            "kvd_probe_zero_copy": ([p, p, ctypes.c_size_t, i32, p], i32),
            "kvd_read_index": ([p, i32, i32, i32, p, p, p], i32),
            "kvd_set_segment_capacity": ([p, i32, i32, i64], i32),
            "kvd_get_segment_stats": ([p, p, p], i32),
            "kvd_plan_window_scaling": ([p, p, i32, i32, ctypes.c_double, p], i32),
            "kvd_read_minmax": ([p, i32, i32, i32, p, p], i32),
            "kvd_append_token": ([p, i32, p, i32, p, p, u32, p], i32),
            "kvd_load_prefix_obs": ([p, i32, i32, p, p, i64, p, i32, p], i32),
            "kvd_read_warm_importance": ([p, i32, i64, p], i32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(code):
    if code != 0:
        raise KVDError(code, lib().kvd_last_error().decode())


def ptr(x):
    """Raw address of a C-contiguous torch tensor or numpy array, an int, or None (a strided
    view raises: the C ABI takes dense arrays)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array is not C-contiguous (np.ascontiguousarray it)")
        return x.ctypes.data
    if not x.is_contiguous():
        raise ValueError("tensor is not contiguous")
    return x.data_ptr()


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _reqs(req_ids):
    a = np.ascontiguousarray(np.asarray(req_ids, dtype=np.int32))
    return a, len(a)


class KVCache:
    """One libkvd cache (all layers, requests and KV heads of one GPU)."""

    def __init__(self, *, num_layers, num_q_heads, num_kv_heads, block_tokens, max_requests, max_context,
                 slots_per_segment, max_select, sink_tokens=4, local_tokens=64, policy="lru",
                 host_layer_alias=0, device=0, head_dim=128, index_ratio=0, summary_kind=0):
        self.cfg = Config(num_layers, num_q_heads, num_kv_heads, head_dim, block_tokens, max_requests,
                          max_context, slots_per_segment, max_select, sink_tokens, local_tokens,
                          POLICY[policy] if isinstance(policy, str) else int(policy), host_layer_alias, device,
                          index_ratio, SUMMARY_KIND[summary_kind] if isinstance(summary_kind, str) else summary_kind)
        self.index_ratio = index_ratio
        h = ctypes.c_void_p()
        _check(lib().kvd_create_cache(ctypes.byref(self.cfg), ctypes.byref(h)))
        self.h = h
        info = Info()
        _check(lib().kvd_get_info(self.h, ctypes.byref(info)))
        self.info = info
        self.nb_max, self.nb_pad, self.C = info.nb_max, info.nb_pad, info.slots_per_segment
        self.max_pinned, self.record_bytes = info.max_pinned, info.record_bytes
        self.resident = bool(info.resident)
        self.G = num_q_heads // num_kv_heads

    @staticmethod
    def required_bytes(**kw):
        cfg = Config(kw["num_layers"], kw["num_q_heads"], kw["num_kv_heads"], kw.get("head_dim", 128),
                     kw["block_tokens"], kw["max_requests"], kw["max_context"], kw["slots_per_segment"],
                     kw["max_select"], kw.get("sink_tokens", 4), kw.get("local_tokens", 64),
                     POLICY[kw.get("policy", "lru")], kw.get("host_layer_alias", 0), kw.get("device", 0),
                     kw.get("index_ratio", 0), kw.get("summary_kind", 0))
        d, hb = ctypes.c_size_t(), ctypes.c_size_t()
        _check(lib().kvd_required_bytes(ctypes.byref(cfg), ctypes.byref(d), ctypes.byref(hb)))
        return d.value, hb.value

    def close(self):
        if getattr(self, "h", None):
            lib().kvd_destroy_cache(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def attn_width(self, k_blocks):
        return lib().kvd_attn_width(self.h, k_blocks)

    def set_device_step(self, dev_step):
        """Resolve reads the step index from this device uint32 (graph replay); None = host arg."""
        _check(lib().kvd_set_device_step(self.h, ptr(dev_step)))

    # ------------------------------------------------------------ setup
    def load_prefix(self, layer, req, k, v, n_tokens, stream=None, q_obs=None):
        """kvd_load_prefix; with q_obs [Hq][n_obs][128] the importance-guided warm-up
        (kvd_load_prefix_obs)."""
        if q_obs is None:
            _check(lib().kvd_load_prefix(self.h, layer, req, ptr(k), ptr(v), n_tokens, _stream(stream)))
        else:
            _check(lib().kvd_load_prefix_obs(self.h, layer, req, ptr(k), ptr(v), n_tokens, ptr(q_obs),
                                             int(q_obs.shape[1]), _stream(stream)))

    # ------------------------------------------------------------ step
    def select_topk(self, layer, q, req_ids, k_blocks, out_ids, out_scores=None, stream=None):
        r, B = _reqs(req_ids)
        _check(lib().kvd_select_topk(self.h, layer, ptr(q), r.ctypes.data, B, k_blocks, ptr(out_ids),
                                     ptr(out_scores), _stream(stream)))

    def resolve_and_fetch(self, layer, req_ids, ids, k_blocks, step, out_attn, stream=None):
        r, B = _reqs(req_ids)
        _check(lib().kvd_resolve_and_fetch(self.h, layer, r.ctypes.data, B, ptr(ids), k_blocks, step,
                                           ptr(out_attn), _stream(stream)))

    def select_resolve_fetch(self, layer, q, req_ids, k_blocks, step, out_ids, out_attn, out_scores=None,
                             stream=None, heads=None):
        """select_topk + resolve_and_fetch in one fused launch sequence (identical results).
        heads=(h0, nh): only KV heads [h0, h0+nh) (kvd_select_resolve_fetch_heads)."""
        r, B = _reqs(req_ids)
        if heads is None:
            _check(lib().kvd_select_resolve_fetch(self.h, layer, ptr(q), r.ctypes.data, B, k_blocks, step,
                                                  ptr(out_ids), ptr(out_scores), ptr(out_attn), _stream(stream)))
        else:
            _check(lib().kvd_select_resolve_fetch_heads(self.h, layer, ptr(q), r.ctypes.data, B, heads[0], heads[1],
                                                        k_blocks, step, ptr(out_ids), ptr(out_scores), ptr(out_attn),
                                                        _stream(stream)))

    def append_token(self, layer, req_ids, k, v, step, stream=None):
        """Decode-time append of one token per request (kvd_append_token); k, v [B][Hkv][128]."""
        r, B = _reqs(req_ids)
        _check(lib().kvd_append_token(self.h, layer, r.ctypes.data, B, ptr(k), ptr(v), step, _stream(stream)))

    def sparse_decode(self, layer, q, req_ids, attn, W, out, out_lse=None, stream=None, heads=None):
        """heads=(h0, nh): only KV heads [h0, h0+nh) (kvd_sparse_decode_heads)."""
        r, B = _reqs(req_ids)
        if heads is None:
            _check(lib().kvd_sparse_decode(self.h, layer, ptr(q), r.ctypes.data, B, ptr(attn), W, ptr(out),
                                           ptr(out_lse), _stream(stream)))
        else:
            _check(lib().kvd_sparse_decode_heads(self.h, layer, ptr(q), r.ctypes.data, B, heads[0], heads[1],
                                                 ptr(attn), W, ptr(out), ptr(out_lse), _stream(stream)))

    # ------------------------------------------------------------ introspection
    def read_segment(self, layer, req, head):
        t = np.empty(self.nb_pad, np.int32)
        sb = np.empty(self.C, np.int32)
        lu = np.empty(self.C, np.uint32)
        ph = np.empty(self.C, np.uint8)
        uc = np.empty(self.C, np.uint32)
        _check(lib().kvd_read_segment(self.h, layer, req, head, ptr(t), ptr(sb), ptr(lu), ptr(ph), ptr(uc)))
        return dict(table=t, slot_block=sb, last_use=lu, phase=ph, use_count=uc)

    def read_slot(self, layer, req, head, slot):
        out = np.empty(self.record_bytes, np.uint8)
        _check(lib().kvd_read_slot(self.h, layer, req, head, slot, ptr(out)))
        return out

    def read_host_record(self, layer, req, head, block):
        out = np.empty(self.record_bytes, np.uint8)
        _check(lib().kvd_read_host_record(self.h, layer, req, head, block, ptr(out)))
        return out

    def read_summaries(self, layer, req, head, nb):
        out = np.empty((nb, 128), np.uint16)
        _check(lib().kvd_read_summaries(self.h, layer, req, head, ptr(out)))
        return out

    def read_warm_importance(self, head, nb):
        """Block importances of the last warm-up (kvd_read_warm_importance)."""
        out = np.empty(nb, np.float32)
        _check(lib().kvd_read_warm_importance(self.h, head, nb, ptr(out)))
        return out

    def read_minmax(self, layer, req, head, nb):
        """Quest min/max summaries (summary_kind 1): (mn, mx) [nb][128] uint16."""
        mn = np.empty((nb, 128), np.uint16)
        mx = np.empty((nb, 128), np.uint16)
        _check(lib().kvd_read_minmax(self.h, layer, req, head, ptr(mn), ptr(mx)))
        return mn, mx

    def read_index(self, layer, req, head, nb):
        """(centroids [nc][128] uint16, cent_of [nb] int32) of a segment's hierarchical index."""
        nc = ctypes.c_int64()
        _check(lib().kvd_read_index(self.h, layer, req, head, ctypes.byref(nc), None, None))
        cent = np.empty((max(nc.value, 1), 128), np.uint16)
        cof = np.empty(max(nb, 1), np.int32)
        _check(lib().kvd_read_index(self.h, layer, req, head, ctypes.byref(nc), ptr(cent), ptr(cof)))
        return cent[:nc.value], cof[:nb]

    def read_scores(self, layer, req, head, nb):
        out = np.empty(nb, np.float32)
        _check(lib().kvd_read_scores(self.h, layer, req, head, ptr(out)))
        return out

    def stats(self):
        s = Stats()
        _check(lib().kvd_get_stats(self.h, ctypes.byref(s)))
        return s.asdict()

    def reset_stats(self):
        _check(lib().kvd_reset_stats(self.h))

    def check(self):
        _check(lib().kvd_check(self.h))

    def set_segment_capacity(self, layer, head, slots):
        """2D window scaling: slots the layer-head pair may use (kvd_set_segment_capacity)."""
        _check(lib().kvd_set_segment_capacity(self.h, layer, head, slots))

    def segment_stats(self):
        """(selected [L][Hkv], misses [L][Hkv]) since reset_stats."""
        L, H = self.cfg.num_layers, self.cfg.num_kv_heads
        sel = np.zeros((L, H), np.uint64)
        mis = np.zeros((L, H), np.uint64)
        _check(lib().kvd_get_segment_stats(self.h, ptr(sel), ptr(mis)))
        return sel, mis

    KERNEL_KINDS = ("select", "resolve", "gather", "attn", "score")

    def enable_kernel_timer(self, enable=True):
        """Device-side launch timing of every step kernel (kvd.h); zeroes the accumulators."""
        _check(lib().kvd_enable_kernel_timer(self.h, 1 if enable else 0))

    def read_kernel_timer(self):
        """{kind: (summed launch ns, launches)} since the last enable."""
        ns = np.zeros(len(self.KERNEL_KINDS), np.uint64)
        n = np.zeros(len(self.KERNEL_KINDS), np.uint64)
        _check(lib().kvd_read_kernel_timer(self.h, ptr(ns), ptr(n)))
        return {k: (int(ns[i]), int(n[i])) for i, k in enumerate(self.KERNEL_KINDS)}


def plan_window_scaling(benefit, cost, budget):
    """Greedy MCKP planner of 2D window scaling (kvd_plan_window_scaling): choice [pairs]."""
    b = np.ascontiguousarray(np.asarray(benefit, np.float64))
    c = np.ascontiguousarray(np.asarray(cost, np.float64))
    pairs, sizes = b.shape
    choice = np.empty(pairs, np.int32)
    _check(lib().kvd_plan_window_scaling(ptr(b), ptr(c), pairs, sizes, float(budget), ptr(choice)))
    return choice


def probe_zero_copy(host, dev, nbytes, ctas, stream=None):
    """Zero-copy host-link probe (kvd_probe_zero_copy): pinned host -> device, gather pattern."""
    _check(lib().kvd_probe_zero_copy(ptr(host), ptr(dev), nbytes, ctas, _stream(stream)))


def record_to_kv(rec, P, d=128):
    """Decode a library block record (K||V, swizzled rows) into K, V [P][d] uint16.

    Layout: row t of K at byte t*256; its 16-byte chunk c at
    position c ^ (t & 7); V follows K.  Used only by tests."""
    rec = np.asarray(rec, np.uint8).reshape(2, P, 16, 16)
    out = np.empty_like(rec)
    for t in range(P):
        for c in range(16):
            out[:, t, c] = rec[:, t, c ^ (t & 7)]
    kv = out.reshape(2, P, d * 2).view(np.uint16)
    return kv[0], kv[1]
