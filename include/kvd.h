/*
 * kvd.h — C ABI of libkvd.so, the B200 (sm_100a) decode-step hot path of
 * KVDrive (arxiv 2605.18071).
 *
 * The calls follow the paper's statement of one decode step (PAPER.md:241-244,
 * 386): "identifying critical KV entries via the index (1); fetching the
 * selected entries from DRAM ... into GPU HBM (2); and executing attention ...
 * over the union of the newly fetched and resident KV entries (3)":
 *
 *   (1) kvd_select_topk        score the decode query against the per-block
 *                              mean-key summaries and keep the
 *                              top-k blocks
 *   (2) kvd_resolve_and_fetch  look the chosen blocks up in the GPU cache's
 *                              block table (hit/miss), evict by
 *                              LRU / LFU / lookahead and gather
 *                              the missed blocks from pinned host DRAM
 *                              (sparse block fetch)
 *   (3) kvd_sparse_decode      split-K sparse decode attention over the
 *                              selected + pinned blocks with a log-sum-exp merge
 *
 * A "segment" is one (request, layer, KV head).  Block = P consecutive tokens
 * (P = block_tokens).  Always-resident ("pinned") blocks are those overlapping
 * the first sink_tokens and the last local_tokens tokens of the request
 * (4 sink + 64 local).  Readings of the paper that fix the exact
 * arithmetic (fp32 sequential-FMA scores, bf16 summaries, tie rules, victim
 * keys) are listed in DESIGN.md §3.
 *
 * Conventions
 *  - Every pointer is a plain host or device pointer; sizes are element counts
 *    unless named *_bytes.  bf16 tensors are passed as uint16_t bit patterns.
 *  - Step calls (select / resolve_and_fetch / sparse_decode) are asynchronous
 *    on `stream`, never synchronise, never allocate, use fixed grids, and are
 *    therefore CUDA-graph capturable.
 *  - Arguments are validated synchronously before anything is launched; on a
 *    non-OK status nothing was launched.  KVD_EINVAL: null pointer, bad shape,
 *    unknown request; KVD_ERANGE: k larger than the candidate count of some
 *    request; KVD_ECAPACITY: k + pinned > slots per segment.
 *  - Faults only visible on the device (e.g. an id list that is not ascending,
 *    out of range or names a pinned block) set a sticky device flag; the kernel
 *    skips that segment and kvd_check reports KVD_EDEVICE.
 *  - No exception crosses the ABI.  kvd_last_error() returns a thread-local
 *    message for the last non-OK status of the calling thread.
 *  - A cache is not safe for concurrent mutation: drive it from one host
 *    thread; step calls on different streams must touch disjoint requests.
 *  - Given identical inputs and call sequence (including `step`), every
 *    integer output (ids, slot maps, attention lists, miss lists) is
 *    bit-identical, independent of how many segments share the GPU.
 */
#ifndef KVD_H_
#define KVD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kvd_cache kvd_cache;      /* opaque; owns all cache state */
typedef struct CUstream_st* kvd_stream;  /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    KVD_OK = 0,
    KVD_EINVAL = 1,     /* bad argument / shape / null pointer */
    KVD_ERANGE = 2,     /* k_blocks > candidates (nb_r - pinned_r) for some request */
    KVD_ECAPACITY = 3,  /* k_blocks + pinned_r > slots_per_segment */
    KVD_ENOMEM = 4,     /* device or pinned-host allocation failed */
    KVD_ECUDA = 5,      /* CUDA API / launch failure (message has cudaGetErrorString) */
    KVD_EDEVICE = 6,    /* a kernel flagged bad device-side input (see kvd_check) */
    KVD_ESTATE = 7      /* call out of order (e.g. request not loaded) */
} kvd_status;

typedef enum {
    KVD_POLICY_LRU = 0,        /* evict min (last_use, phase, block) */
    KVD_POLICY_LFU = 1,        /* evict min (use_count, last_use, phase, block) */
    KVD_POLICY_LOOKAHEAD = 2   /* evict lowest current-step score, larger block first */
} kvd_policy;

#define KVD_MAX_BATCH 256      /* max requests per step call */
#define KVD_HEAD_DIM 128       /* the only supported head_dim */
#define KVD_MAX_GROUP 8        /* max num_q_heads / num_kv_heads */

typedef struct {
    int32_t num_layers;          /* L */
    int32_t num_q_heads;         /* Hq */
    int32_t num_kv_heads;        /* Hkv; Hq % Hkv == 0 and Hq / Hkv <= KVD_MAX_GROUP */
    int32_t head_dim;            /* must be KVD_HEAD_DIM */
    int32_t block_tokens;        /* P in {1, 2, 4, 8, 16} */
    int32_t max_requests;        /* request slots 0 .. max_requests-1 */
    int64_t max_context;         /* tokens per request (upper bound) */
    int64_t slots_per_segment;   /* C, including the pinned blocks.  C >= ceil(max_context/P)
                                    => fully resident: no host store, block b lives in slot b.
                                    A host-backed cache ranks its victims on chip: it needs
                                    8*C + 20*max_select + ceil(max_context/P)/8 <= 227 KiB
                                    (C <= ~27,000 at max_select 128), else KVD_EINVAL.
                                    Blocks per request <= 262,144 (top-k cluster capacity). */
    int32_t max_select;          /* largest k_blocks any step call will use (sizes scratch) */
    int32_t sink_tokens;         /* 4 */
    int32_t local_tokens;        /* 64 */
    int32_t policy;              /* kvd_policy */
    int32_t host_layer_alias;    /* A: host store holds A layers; layer l uses host layer l % A.
                                    0 or >= num_layers => one host layer per layer.  Benchmark
                                    affordance for hosts with less RAM than the KV: the caller must
                                    load identical prefixes for layers l and l' when l == l' mod A. */
    int32_t device;              /* CUDA device ordinal */
    int32_t index_ratio;         /* 0: flat index -- every block summary is scored (default).
                                    r in 1..64: hierarchical centroid index (
                                    DESIGN.md R27): kvd_load_prefix clusters each segment's block
                                    summaries by k-means inside windows of 64 blocks into
                                    ceil(len / r) centroids per window; the select calls score the
                                    centroids, keep the m = min(nc, max(ceil(4k/r), k + pinned)) best
                                    and score only their member blocks (exact top-k among those).
                                    Needs min(blocks, 64 m) <= 16384 (KVD_EINVAL otherwise). */
    int32_t summary_kind;        /* 0: mean key per block (default).  1: Quest's
                                    channel-wise minimum and maximum of the block's keys
                                    (R30): score = sum over j of
                                    max(qbar_j * min_j, qbar_j * max_j), fp32 in j order -- the
                                    paper's comparison baseline as a second selection workload
                                    (twice the summary bytes).  Not with index_ratio > 0. */
} kvd_config;

typedef struct {
    uint64_t selected;           /* selected (non-pinned) blocks resolved */
    uint64_t hits;               /* of those, found resident ("served from the GPU cache") */
    uint64_t misses;             /* of those, fetched from the host store */
    uint64_t pinned;             /* pinned blocks attended (always resident; not in hit rate) */
    uint64_t fetched_bytes;      /* host -> HBM bytes copied by the gather */
} kvd_stats;

typedef struct {
    int64_t nb_max;              /* ceil(max_context / P) */
    int64_t nb_pad;              /* nb_max rounded up to 128 (summary / table row length) */
    int64_t slots_per_segment;   /* C */
    int32_t max_pinned;          /* upper bound on pinned blocks per segment */
    int32_t record_bytes;        /* 2 * P * 128 * 2 */
    int32_t resident;            /* 1 if C >= nb_max (no host store) */
    int32_t host_layers;         /* A */
} kvd_cache_info;

/* Bytes the cache will allocate for `cfg`: device HBM and pinned host. */
kvd_status kvd_required_bytes(const kvd_config* cfg, size_t* dev_bytes, size_t* host_pinned_bytes);

/* Create a cache on cfg->device (makes it current).  *out receives the handle.
 * Allocates the slot pool [L][R][Hkv][C] of block records (K[P][128] || V[P][128]
 * bf16, 16-byte chunks XOR-swizzled per row), the dim-major summaries
 * [L][R][Hkv][128][nb_pad] bf16, scores, block tables, slot metadata and, unless
 * fully resident, the mapped pinned host store [A][R][Hkv][nb] records. */
kvd_status kvd_create_cache(const kvd_config* cfg, kvd_cache** out);
void       kvd_destroy_cache(kvd_cache* c);   /* synchronises the device; NULL is a no-op */

/* Ingest request `req`'s prefix for `layer` (setup; not part of a decode step).
 * k, v: bf16 [Hkv][n_tokens][128] token-major, host or device memory, copied
 * (caller may free them once `stream` has synchronised).  Writes the host
 * store (host-backed caches), builds the block summaries (a0: mean key per
 * block, fp32 sum in token order, IEEE divide, bf16 RNE) and
 * resets the segment caches: fully resident => block b in slot b; otherwise
 * cold with the pinned blocks in slots 0..p-1.  May synchronise `stream`.
 * n_tokens in [1, max_context]. */
kvd_status kvd_load_prefix(kvd_cache* c, int32_t layer, int32_t req,
                           const uint16_t* k, const uint16_t* v, int64_t n_tokens,
                           kvd_stream stream);

/* Importance-guided warm-up (R29): kvd_load_prefix, then for a
 * host-backed cache the C - pinned non-pinned blocks with the highest attention mass from the
 * prompt's final observation window start resident (instead of a cold cache): importance of block
 * b = sum over the G x n_obs observation queries of its tokens' softmax weights over the whole
 * prefix (fp32); ties -> lower block; placed after the pinned blocks, ascending by block, as
 * admitted at step 0 (last use 0, phase 1, count 1).  q_obs: bf16 [Hq][n_obs][128] (host or
 * device), n_obs <= 16 and G x n_obs <= 128.  A fully resident cache ignores it. */
kvd_status kvd_load_prefix_obs(kvd_cache* c, int32_t layer, int32_t req, const uint16_t* k, const uint16_t* v,
                               int64_t n_tokens, const uint16_t* q_obs, int32_t n_obs, kvd_stream stream);

/* (1) Select.  q: device bf16 [B][Hq][128].  req_ids: host int32 [B] (distinct,
 * loaded).  For each request b and KV head h: qbar = fp32 sum of the group's
 * G query heads (g ascending); score_j = sequential fp32 FMA chain over the 128
 * dims of qbar x summary_j; keep the k_blocks non-pinned blocks with the highest
 * score (ties -> lower block id; NaN lowest; -0 == +0).
 * out_ids: device int32 [B][Hkv][k_blocks], ascending per segment.
 * out_scores: device fp32 [B][Hkv][k_blocks] (scores of out_ids) or NULL.
 * Every block's score is also kept inside the cache for the lookahead policy. */
kvd_status kvd_select_topk(kvd_cache* c, int32_t layer, const uint16_t* q,
                           const int32_t* req_ids, int32_t B, int32_t k_blocks,
                           int32_t* out_ids, float* out_scores, kvd_stream stream);

/* (2) Resolve + fetch.  ids: device int32 [B][Hkv][k_blocks] from select (same
 * layer, same requests; for the lookahead policy select must have run for
 * this layer and these requests first).  Per segment: hits = ids resident;
 * misses M (ascending) go to free slots (ascending) then to victims (residents
 * neither selected nor pinned, by the policy key); victims' table entries are
 * cleared; metadata updated with `step` (hits: last=step, phase 0, count+1;
 * admitted: last=step, phase 1, count 1).  Then each missed block's 8 KiB
 * record is copied from the pinned host store into its slot by SM zero-copy
 * reads over the host link.
 * out_attn: device int32 [B][Hkv][W][2] of (block, slot) for selected u pinned,
 * ascending by block, (-1,-1) padded; W = k_blocks + max pinned, see
 * kvd_attn_width.  stats: accumulated inside the cache (kvd_get_stats). */
kvd_status kvd_resolve_and_fetch(kvd_cache* c, int32_t layer, const int32_t* req_ids,
                                 int32_t B, const int32_t* ids, int32_t k_blocks,
                                 uint32_t step, int32_t* out_attn, kvd_stream stream);

/* (1)+(2) fused -- "identifying critical KV entries via the index" then "fetching
 * the selected entries from DRAM".  Exactly kvd_select_topk
 * followed by kvd_resolve_and_fetch: same arguments (q, req_ids, B, k_blocks as for
 * select; step as for resolve), same results, same cache state, bit for bit.  The
 * top-k, the resolve and the miss fetch of a segment run in one kernel (one
 * thread-block cluster per segment; rank 0 resolves and copies the misses), so the
 * step has no kernel boundary between selection and fetch.  out_ids (device int32
 * [B][Hkv][k_blocks]) and out_scores (or NULL) are written as by select; out_attn
 * as by resolve.  Caller owns every buffer; asynchronous on `stream`.  Errors as for
 * the two calls (validated synchronously; nothing launched on error). */
kvd_status kvd_select_resolve_fetch(kvd_cache* c, int32_t layer, const uint16_t* q,
                                    const int32_t* req_ids, int32_t B, int32_t k_blocks,
                                    uint32_t step, int32_t* out_ids, float* out_scores,
                                    int32_t* out_attn, kvd_stream stream);

/* The fused call for the KV heads [h0, h0 + nh) only (0 <= h0, 1 <= nh, h0 + nh <= Hkv; KVD_EINVAL
 * otherwise).  Arrays keep their full layouts (q [B][Hq][128], out_ids [B][Hkv][k_blocks], out_attn
 * [B][Hkv][W][2]); only the range's segments are read and written, with results bit for bit those of
 * kvd_select_resolve_fetch for those segments.  Segments are independent, so disjoint head ranges
 * may be issued on different streams (micro-batch chains of fewer heads than a request has). */
kvd_status kvd_select_resolve_fetch_heads(kvd_cache* c, int32_t layer, const uint16_t* q,
                                          const int32_t* req_ids, int32_t B, int32_t h0, int32_t nh,
                                          int32_t k_blocks, uint32_t step, int32_t* out_ids, float* out_scores,
                                          int32_t* out_attn, kvd_stream stream);

/* Decode-time append ("each step appending new key and value vectors"; DESIGN.md
 * R16): one new token for each listed request of `layer`, at position n_r (the layer's token
 * count), k / v: device bf16 [B][Hkv][128].  The token joins the always-resident local window;
 * when it opens a new block, that block is admitted at `step` (fully resident: slot = block;
 * otherwise the lowest free slot of the layer-head's window, else the resident block with the
 * smallest policy key among those not pinned after the append is evicted).  The token's K / V rows
 * are written to the slot record (and the host store), the block's summary is recomputed over its
 * tokens as kvd_load_prefix computes it, and the layer's token count grows by one.  Asynchronous on
 * `stream`; the host-side token counts advance at the call (do not replay it from a CUDA graph).
 * KVD_ERANGE when a context is full; KVD_ESTATE with the hierarchical index or host-layer aliasing. */
kvd_status kvd_append_token(kvd_cache* c, int32_t layer, const int32_t* req_ids, int32_t B, const uint16_t* k,
                            const uint16_t* v, uint32_t step, kvd_stream stream);

/* CUDA-graph support for (2): when dev_step != NULL, every later resolve reads
 * the decode-step index from *dev_step (device uint32) when the kernel runs and
 * ignores its host `step` argument, so one captured step can be replayed for
 * step t, t+1, ... by advancing *dev_step on the stream.  NULL restores the
 * host argument.  dev_step must stay valid while the cache uses it. */
kvd_status kvd_set_device_step(kvd_cache* c, const uint32_t* dev_step);

kvd_status kvd_get_info(const kvd_cache* c, kvd_cache_info* out);

/* Width W of the attention list for k_blocks (k_blocks + max pinned blocks). */
int32_t kvd_attn_width(const kvd_cache* c, int32_t k_blocks);

/* (3) Attend.  q: device bf16 [B][Hq][128]; attn: device int32 [B][Hkv][W][2]
 * from resolve, W == kvd_attn_width(c, k) for the k used there.  For every query head: softmax(q K^T / sqrt(128)) V over the
 * tokens of the listed blocks (partial last block masked), split-K over the
 * list with a log-sum-exp merge.  out: device fp32 [B][Hq][128];
 * out_lse: device fp32 [B][Hq] (natural log) or NULL.  q is read before the kernel waits on its
 * stream predecessor (programmatic dependent launch): pass the q of this step's select call, not a
 * buffer written by the kernel launched immediately before this call. */
kvd_status kvd_sparse_decode(kvd_cache* c, int32_t layer, const uint16_t* q,
                             const int32_t* req_ids, int32_t B, const int32_t* attn,
                             int32_t W, float* out, float* out_lse, kvd_stream stream);

/* kvd_sparse_decode for the KV heads [h0, h0 + nh) only (their query heads h*G .. h*G+G-1);
 * arrays keep their full layouts (attn [B][Hkv][W][2], out [B][Hq][128], out_lse [B][Hq]).  Outputs
 * are bit for bit those of kvd_sparse_decode for those heads (the split plan depends on k only). */
kvd_status kvd_sparse_decode_heads(kvd_cache* c, int32_t layer, const uint16_t* q,
                                   const int32_t* req_ids, int32_t B, int32_t h0, int32_t nh,
                                   const int32_t* attn, int32_t W, float* out, float* out_lse,
                                   kvd_stream stream);

/* Introspection (synchronous; tests / bench only).  Copy one segment's state
 * to host buffers: table [nb_pad] int32, slot_block/last_use/use_count [C],
 * phase [C] u8; any pointer may be NULL. */
kvd_status kvd_read_segment(kvd_cache* c, int32_t layer, int32_t req, int32_t head,
                            int32_t* table, int32_t* slot_block, uint32_t* last_use,
                            uint8_t* phase, uint32_t* use_count);
/* Copy one slot's record (2*P*128 bf16, library layout) or one host-store record. */
kvd_status kvd_read_slot(kvd_cache* c, int32_t layer, int32_t req, int32_t head,
                         int64_t slot, void* out_record);
kvd_status kvd_read_host_record(kvd_cache* c, int32_t layer, int32_t req, int32_t head,
                                int64_t block, void* out_record);
/* Copy a segment's summaries as [nb][128] bf16 (block-major, unpadded). */
kvd_status kvd_read_summaries(kvd_cache* c, int32_t layer, int32_t req, int32_t head,
                              uint16_t* out);
/* Block importances [nb] of `head` computed by the last kvd_load_prefix_obs (setup scratch). */
kvd_status kvd_read_warm_importance(kvd_cache* c, int32_t head, int64_t nb, float* out);
/* Quest min/max summaries of a segment (summary_kind 1): mn, mx [nb][128] bf16, block-major. */
kvd_status kvd_read_minmax(kvd_cache* c, int32_t layer, int32_t req, int32_t head, uint16_t* mn, uint16_t* mx);
/* Hierarchical index of one segment (index_ratio > 0): *nc receives the centroid count;
 * centroids [nc][128] bf16 (block-major copy) and cent_of [nb] (block -> centroid) may be NULL. */
kvd_status kvd_read_index(kvd_cache* c, int32_t layer, int32_t req, int32_t head, int64_t* nc,
                          uint16_t* centroids, int32_t* cent_of);
/* Copy a segment's current block scores [nb] fp32 (last select of that layer; with the
 * hierarchical index: the lookahead scores -- exact for the candidates, else the centroid's). */
kvd_status kvd_read_scores(kvd_cache* c, int32_t layer, int32_t req, int32_t head, float* out);

kvd_status kvd_get_stats(kvd_cache* c, kvd_stats* out);   /* synchronises the device */

/* 2D layer-head window scaling (R28).
 * kvd_set_segment_capacity: layer-head pair (layer, head) of every request may use only slots
 * 0 .. slots-1 of its segment (its "window"); pinned <= slots <= slots_per_segment.  Shrinking
 * drops the residents of the cut slots (their blocks are fetched again when selected).  Host-backed
 * caches only (KVD_ESTATE otherwise).  Synchronises the device.  A step call needs k + pinned <=
 * the smallest capacity of its layer (KVD_ECAPACITY).
 * kvd_get_segment_stats: per layer-head counters since kvd_reset_stats, [L][Hkv] each: selected
 * (non-pinned) blocks resolved and misses -- the profile of Benefit(w) (transfer reduction).
 * kvd_plan_window_scaling: the offline planner: greedy multiple-choice knapsack over `pairs`
 * layer-head pairs x `sizes` candidate windows (benefit / cost [pairs][sizes], sizes in increasing
 * cost); choice[pairs] receives the chosen size index.  Host only (no GPU); KVD_EINVAL if the
 * smallest sizes exceed the budget. */
kvd_status kvd_set_segment_capacity(kvd_cache* c, int32_t layer, int32_t head, int64_t slots);
kvd_status kvd_get_segment_stats(kvd_cache* c, uint64_t* selected, uint64_t* misses);
kvd_status kvd_plan_window_scaling(const double* benefit, const double* cost, int32_t pairs, int32_t sizes,
                                   double budget, int32_t* choice);

/* Kernel timer (measurement; bench.py).  While enabled, every step kernel records its own
 * launch duration on the device: from the earliest start of any of its CTAs / warps after
 * griddepcontrol.wait to the end of the last one (%globaltimer), accumulated per kind:
 * [0] select (score + top-k, fused: + resolve + fetch), [1] resolve (kvd_resolve_and_fetch),
 * [2] gather (kvd_resolve_and_fetch, host-backed), [3] attention (split-K + merge).  This
 * times the kernels of a CUDA-graph / multi-stream step exactly as it runs, with no event node
 * between kernels (which would break their programmatic overlap).  Costs two device-scope
 * atomics per CTA (per warp for attention).  kvd_enable_kernel_timer synchronises and zeroes
 * the accumulators (allocating on first use); enable = 0 stops recording.  Step calls capture
 * the on/off state when they are issued (or captured into a graph).
 * kvd_read_kernel_timer synchronises and copies ns[5] (summed launch durations) and
 * launches[5] (counts), by kernel kind: select, resolve, gather, attention, score. */
kvd_status kvd_enable_kernel_timer(kvd_cache* c, int32_t enable);
/* Host-link probe (measurement; the gather's denominator): copy `bytes` (a
 * multiple of 16) from pinned host memory `host` to device memory `dev` with the miss gather's
 * own access pattern (16-byte zero-copy loads, 8 in flight per thread) on `ctas` CTAs of 256
 * threads.  Asynchronous on `stream`; KVD_EINVAL if `host` is not pinned host memory. */
kvd_status kvd_probe_zero_copy(const void* host, void* dev, size_t bytes, int32_t ctas, kvd_stream stream);
kvd_status kvd_read_kernel_timer(kvd_cache* c, uint64_t* ns, uint64_t* launches);
kvd_status kvd_reset_stats(kvd_cache* c);                 /* synchronises the device */

/* Synchronise the device and report KVD_EDEVICE if any kernel flagged bad input
 * since the last check (the flag is cleared), else KVD_OK / KVD_ECUDA. */
kvd_status kvd_check(kvd_cache* c);
const char* kvd_last_error(void);

/* Library build identity, e.g. "kvd 0.2 sm_100a". */
const char* kvd_version(void);

/* Number of step kernels (select, resolve, gather, attention, merge) this process
 * has launched through libkvd so far (thread-safe counter; a launch recorded into
 * a CUDA graph counts once, when it is captured).  The difference across one
 * step call sequence is that step's launch count.  Never fails. */
uint64_t kvd_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* KVD_H_ */
