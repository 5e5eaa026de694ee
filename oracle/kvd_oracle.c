/*
 * kvd_oracle.c — CPU ORACLE for the KVDrive decode-step hot path.
 *
 *   *** TEST INFRASTRUCTURE ONLY. ***
 *   Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 *   --impl reference legs may load this library.  The product path
 *   (paper_2605_18071_b200/, libkvd.so) never links, imports or calls it,
 *   and this file shares no code, header, table or constant with it.
 *
 * A plain, slow, obviously-correct restatement of what one decode step
 * computes for one segment = one (request, layer, KV head), written from
 * the paper (/root/reference/PAPER.md, cited as PAPER.md:<line>) and the
 * binding readings of SURVEY.md §8.4.1 (listed again in DESIGN.md §3).
 * No blocking, no fusion, no reordering beyond what the definitions say.
 *
 *   O1  or_block_summaries  mean key per block ("the mean key of each page
 *                           is used as its representative")
 *   O2  or_group_query      GQA query of a KV head (paper silent; reading R3)
 *   O3  or_block_scores     query x summary dot product ("multiplying the
 *                           query vector with ...")
 *   O4  or_pinned_blocks    sink 4 + local 64 tokens always resident
 *
 *   O5  or_topk             top-k blocks ("retrieving only the Top-K
 *                           important chunks")
 *   O6  or_resolve          hit/miss against the GPU cache + eviction
 *                           (LRU/LFU baselines PAPER.md:223,254,840-859;
 *                           lookahead "entries with the lowest current-step
 *                           attention scores are discarded")
 *   O7  or_fetch            copy missed blocks host -> cache slot
 *                           (sparse block-level fetch)
 *   O8  or_attention        softmax attention over the selected tokens, in
 *                           fp64 ("computing attention
 *                           over the union of fetched and resident entries")
 *
 * Precision: the paper states none (its only dtype is "FP16" in future work,
 * PAPER.md:1056).  Readings R2/R5 fix O1/O3 to fp32 with a stated order so
 * that selected ids are reproducible bit for bit; O8 is fp64.
 *
 * Pins (tests/test_oracle_*.py) — every function here is pinned:
 *   O1: P=1 => summary == key bit-exactly; dyadic keys => exact mean vs int64;
 *       bf16 RNE vs torch.Tensor.bfloat16 (library routine).
 *   O2/O3: SPEC worked examples; integer inputs vs int64 dot; fp64 error bound.
 *   O4: hand-enumerated pinned sets.
 *   O5: brute-force total-order check, sort-all, permutation equivariance,
 *       P=1 => exact token top-k.
 *   O6: independent Python LRU (OrderedDict two-phase) / LFU / LA simulators.
 *   O7: memcmp invariant.
 *   O8: k = all => dense softmax (torch SDPA fp64); closed-form special cases.
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (no OpenMP).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ bf16 */
/* bf16 is the top 16 bits of an IEEE binary32. */
static float bf16_to_f32(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* Round-to-nearest-even binary32 -> bf16 (reading R2).  NaN -> quiet NaN. */
uint16_t or_f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu) != 0)
        return (uint16_t)((u >> 16) | 0x0040u);          /* quiet NaN */
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;                                   /* ties to even */
    return (uint16_t)(u >> 16);
}

/* -------------------------------------------------------------- O1 summary */
/* For block b with cnt_b = min(P, n - P*b) valid tokens and every dim j:
 *   acc = +0f; for t = 0..cnt_b-1: acc = acc + f32(K[P*b+t][j])
 *   S[b][j] = bf16_rne(acc / (float)cnt_b)
 * K is token-major [n][d] bf16; S is block-major [nb][d] bf16. */
void or_block_summaries(const uint16_t* K, int64_t n, int32_t d, int32_t P,
                        uint16_t* S) {
    int64_t nb = (n + P - 1) / P;
    for (int64_t b = 0; b < nb; ++b) {
        int64_t cnt = n - (int64_t)P * b;
        if (cnt > P) cnt = P;
        for (int32_t j = 0; j < d; ++j) {
            float acc = 0.0f;
            for (int64_t t = 0; t < cnt; ++t)
                acc = acc + bf16_to_f32(K[((int64_t)P * b + t) * d + j]);
            S[b * d + j] = or_f32_to_bf16_rne(acc / (float)cnt);
        }
    }
}

/* ---------------------------------------------------------- O2 group query */
/* qbar[j] = ((+0 + q[0][j]) + q[1][j]) + ... + q[G-1][j]   (fp32, g ascending)
 * q holds the G query heads of one KV head, [G][d] bf16. */
void or_group_query(const uint16_t* q, int32_t G, int32_t d, float* qbar) {
    for (int32_t j = 0; j < d; ++j) {
        float acc = 0.0f;
        for (int32_t g = 0; g < G; ++g) acc = acc + bf16_to_f32(q[(int64_t)g * d + j]);
        qbar[j] = acc;
    }
}

/* -------------------------------------------------------------- O3 scores */
/* score_b = fma chain over j = 0..d-1 from +0:  acc = fmaf(qbar[j], S[b][j], acc).
 * No 1/sqrt(d): ranking is invariant to a positive scale (reading R4). */
void or_block_scores(const float* qbar, const uint16_t* S, int64_t nb, int32_t d,
                     float* scores) {
    for (int64_t b = 0; b < nb; ++b) {
        float acc = 0.0f;
        for (int32_t j = 0; j < d; ++j) acc = fmaf(qbar[j], bf16_to_f32(S[b * d + j]), acc);
        scores[b] = acc;
    }
}

/* ------------------------------------------------------------- O4 pinned */
/* Sink: every block overlapping the first `sink` tokens, i.e. blocks
 * 0 .. ceil(sink/P)-1.  Local: every block overlapping the last
 * `local` tokens, i.e. blocks floor(max(0, n-local)/P) .. nb-1 when local > 0
 * (reading R9: block-granular pinning of PAPER.md:685's 4 sink + 64 local).
 * Writes is_pinned[nb] (0/1), returns the pinned count. */
int64_t or_pinned_blocks(int64_t n, int32_t P, int32_t sink, int32_t local,
                         uint8_t* is_pinned) {
    int64_t nb = (n + P - 1) / P;
    int64_t count = 0;
    for (int64_t b = 0; b < nb; ++b) is_pinned[b] = 0;
    for (int64_t b = 0; b < nb && (int64_t)P * b < sink; ++b) is_pinned[b] = 1;
    if (local > 0) {
        int64_t first_tok = n - local;
        if (first_tok < 0) first_tok = 0;
        for (int64_t b = first_tok / P; b < nb; ++b) is_pinned[b] = 1;
    }
    for (int64_t b = 0; b < nb; ++b) count += is_pinned[b];
    return count;
}

/* --------------------------------------------------------------- O5 top-k */
/* Total order (reading R10): score descending, NaN below everything, -0 == +0
 * (IEEE equality), then block id ascending.  Candidates are the non-pinned
 * blocks.  Output: the first k in that order, emitted ascending by id. */
typedef struct { float s; int64_t id; } or_cand;

static int or_score_better(float a, float b) {        /* a ranks strictly above b */
    if (isnan(a)) return 0;
    if (isnan(b)) return 1;
    return a > b;
}
static int or_cand_cmp(const void* x, const void* y) {
    const or_cand* a = (const or_cand*)x;
    const or_cand* b = (const or_cand*)y;
    if (or_score_better(a->s, b->s)) return -1;
    if (or_score_better(b->s, a->s)) return 1;
    return (a->id < b->id) ? -1 : (a->id > b->id);
}
static int or_i32_cmp(const void* x, const void* y) {
    int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    return (a > b) - (a < b);
}

/* returns 0, or 2 (ERANGE) when k exceeds the candidate count */
int32_t or_topk(const float* scores, int64_t nb, const uint8_t* is_pinned, int32_t k,
                int32_t* ids) {
    or_cand* c = (or_cand*)malloc(sizeof(or_cand) * (size_t)(nb > 0 ? nb : 1));
    int64_t m = 0;
    for (int64_t b = 0; b < nb; ++b)
        if (!is_pinned[b]) { c[m].s = scores[b]; c[m].id = b; ++m; }
    if (k < 0 || k > m) { free(c); return 2; }
    qsort(c, (size_t)m, sizeof(or_cand), or_cand_cmp);
    for (int32_t i = 0; i < k; ++i) ids[i] = (int32_t)c[i].id;
    qsort(ids, (size_t)k, sizeof(int32_t), or_i32_cmp);
    free(c);
    return 0;
}

/* ------------------------------------------------------------- O6 resolve */
/* One segment's GPU cache: C slots, a block table, per-slot metadata.
 *   table[b]      slot holding block b, or -1
 *   slot_block[s] block held by slot s, or -1 (free)
 *   last_use[s], phase[s], use_count[s]  policy metadata of slot s's block
 * Initial state (reading R14): fully resident if C >= nb (block b in slot b);
 * otherwise cold: only the pinned blocks, in slots 0..p-1, ascending id. */
enum { OR_LRU = 0, OR_LFU = 1, OR_LA = 2 };

int32_t or_cache_init(int64_t nb, int64_t C, const uint8_t* is_pinned,
                      int32_t* table, int32_t* slot_block, uint32_t* last_use,
                      uint8_t* phase, uint32_t* use_count) {
    for (int64_t b = 0; b < nb; ++b) table[b] = -1;
    for (int64_t s = 0; s < C; ++s) { slot_block[s] = -1; last_use[s] = 0; phase[s] = 0; use_count[s] = 0; }
    if (C >= nb) {
        for (int64_t b = 0; b < nb; ++b) { table[b] = (int32_t)b; slot_block[b] = (int32_t)b; }
        return 0;
    }
    int64_t s = 0;
    for (int64_t b = 0; b < nb; ++b) {
        if (!is_pinned[b]) continue;
        if (s >= C) return 3;                                  /* ECAPACITY */
        table[b] = (int32_t)s; slot_block[s] = (int32_t)b; ++s;
    }
    return 0;
}

typedef struct {
    int64_t slot;
    int64_t block;
    uint32_t last, count;
    uint8_t phase;
    float score;
    int policy;
} or_victim;

/* Policy keys, smallest evicted first (reading R12 / SURVEY §8.4 O6):
 *   LRU: (last_use, phase, block)          LFU: (use_count, last_use, phase, block)
 *   LA : (this step's score ascending with NaN lowest and -0 == +0, block descending) */
static int or_victim_cmp(const void* x, const void* y) {
    const or_victim* a = (const or_victim*)x;
    const or_victim* b = (const or_victim*)y;
    if (a->policy == OR_LA) {
        if (or_score_better(b->score, a->score)) return -1;   /* a lower -> evict first */
        if (or_score_better(a->score, b->score)) return 1;
        return (a->block > b->block) ? -1 : (a->block < b->block);
    }
    if (a->policy == OR_LFU && a->count != b->count) return (a->count < b->count) ? -1 : 1;
    if (a->last != b->last) return (a->last < b->last) ? -1 : 1;
    if (a->phase != b->phase) return (a->phase < b->phase) ? -1 : 1;
    return (a->block < b->block) ? -1 : (a->block > b->block);
}

/* Resolve step `step` for the selected set S (k ids, ascending, non-pinned):
 *  (1) hits = {b in S : table[b] >= 0};  M = S \ hits, ascending
 *  (2) F = free slots, ascending
 *  (3) V = the first max(0, |M|-|F|) resident blocks not in S and not pinned,
 *      by the policy key
 *  (4) M[i] -> (F ++ V)[i]; each victim's table entry -> -1
 *  (5) hits: last=step, phase=0, count+=1; admitted: last=step, phase=1, count=1
 * Outputs:
 *  attn[W][2]  (block, slot) for S u pinned, ascending by block, (-1,-1) padded
 *  miss[k][2]  (block, slot) for M in order, (-1,-1) padded;  *n_miss
 *  *n_hit      |hits| (selected, non-pinned)
 * Returns 0, 3 (ECAPACITY: |M| > |F| + |evictable|), or 1 (EINVAL: S pinned/out of range). */
int32_t or_resolve(int64_t nb, int64_t C, const uint8_t* is_pinned,
                   int32_t* table, int32_t* slot_block, uint32_t* last_use,
                   uint8_t* phase, uint32_t* use_count,
                   const int32_t* S, int32_t k, uint32_t step, int32_t policy,
                   const float* scores, int32_t W,
                   int32_t* attn, int32_t* miss, int32_t* n_miss, int32_t* n_hit) {
    uint8_t* in_S = (uint8_t*)calloc((size_t)(nb > 0 ? nb : 1), 1);
    for (int32_t i = 0; i < k; ++i) {
        if (S[i] < 0 || S[i] >= nb || is_pinned[S[i]]) { free(in_S); return 1; }
        in_S[S[i]] = 1;
    }
    /* (1) */
    int32_t* M = (int32_t*)malloc(sizeof(int32_t) * (size_t)(k > 0 ? k : 1));
    int32_t nm = 0, nh = 0;
    for (int32_t i = 0; i < k; ++i) {
        if (table[S[i]] >= 0) ++nh; else M[nm++] = S[i];
    }
    /* (2) */
    int64_t* dest = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nm > 0 ? nm : 1));
    int32_t nd = 0;
    for (int64_t s = 0; s < C && nd < nm; ++s)
        if (slot_block[s] < 0) dest[nd++] = s;
    /* (3) */
    if (nd < nm) {
        or_victim* v = (or_victim*)malloc(sizeof(or_victim) * (size_t)C);
        int64_t nv = 0;
        for (int64_t s = 0; s < C; ++s) {
            int32_t b = slot_block[s];
            if (b < 0 || in_S[b] || is_pinned[b]) continue;
            v[nv].slot = s; v[nv].block = b; v[nv].last = last_use[s];
            v[nv].count = use_count[s]; v[nv].phase = phase[s];
            v[nv].score = scores ? scores[b] : 0.0f; v[nv].policy = policy;
            ++nv;
        }
        if (nv < nm - nd) { free(v); free(dest); free(M); free(in_S); return 3; }
        qsort(v, (size_t)nv, sizeof(or_victim), or_victim_cmp);
        for (int64_t i = 0; nd < nm; ++i) {
            table[v[i].block] = -1;
            dest[nd++] = v[i].slot;
        }
        free(v);
    }
    /* (4)+(5) */
    for (int32_t i = 0; i < k; ++i) {
        int32_t b = S[i];
        if (table[b] >= 0) {                       /* hit (tables of victims already cleared;
                                                      victims are never in S) */
            int32_t s = table[b];
            last_use[s] = step; phase[s] = 0; use_count[s] += 1;
        }
    }
    for (int32_t i = 0; i < nm; ++i) {
        int64_t s = dest[i];
        table[M[i]] = (int32_t)s; slot_block[s] = M[i];
        last_use[s] = step; phase[s] = 1; use_count[s] = 1;
        miss[2 * i] = M[i]; miss[2 * i + 1] = (int32_t)s;
    }
    for (int32_t i = nm; i < k; ++i) { miss[2 * i] = -1; miss[2 * i + 1] = -1; }
    /* attention list: S u pinned, ascending by block */
    int32_t w = 0;
    for (int64_t b = 0; b < nb; ++b) {
        if (!(in_S[b] || is_pinned[b])) continue;
        if (w >= W) { free(dest); free(M); free(in_S); return 3; }
        attn[2 * w] = (int32_t)b; attn[2 * w + 1] = table[b];
        ++w;
    }
    for (; w < W; ++w) { attn[2 * w] = -1; attn[2 * w + 1] = -1; }
    *n_miss = nm; *n_hit = nh;
    free(dest); free(M); free(in_S);
    return 0;
}

/* --------------------------------------------------------------- O7 fetch */
/* For each (block, slot) in miss: slot_pool[slot] := host_records[block]
 * (record_bytes each; byte copy). */
void or_fetch(const uint8_t* host_records, uint8_t* slot_pool, int64_t record_bytes,
              const int32_t* miss, int32_t n_miss) {
    for (int32_t i = 0; i < n_miss; ++i)
        memcpy(slot_pool + (int64_t)miss[2 * i + 1] * record_bytes,
               host_records + (int64_t)miss[2 * i] * record_bytes, (size_t)record_bytes);
}

/* ----------------------------------------------------------- O8 attention */
/* For each query head g (of the G heads sharing this KV head): over the token
 * set T = U_{b in blocks} {P*b + t : t < cnt_b}, in fp64 from the bf16 inputs:
 *   z_i = (q_g . K_i) / sqrt(d);  m = max z;  p_i = exp(z_i - m);  l = sum p_i
 *   o_g = sum p_i V_i / l  (stored fp32);  lse_g = m + ln l  (stored fp32)
 * K, V token-major [n][d] bf16; q [G][d] bf16; blocks: nblk block ids (-1 skipped). */
void or_attention(const uint16_t* q, int32_t G, int32_t d, const uint16_t* K,
                  const uint16_t* V, int64_t n, int32_t P, const int32_t* blocks,
                  int32_t nblk, float* o, float* lse) {
    int64_t ntok = 0;
    for (int32_t i = 0; i < nblk; ++i) if (blocks[i] >= 0) ntok += P;
    int64_t* tok = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ntok > 0 ? ntok : 1));
    double* z = (double*)malloc(sizeof(double) * (size_t)(ntok > 0 ? ntok : 1));
    double* acc = (double*)malloc(sizeof(double) * (size_t)d);
    int64_t nt = 0;
    for (int32_t i = 0; i < nblk; ++i) {
        int64_t b = blocks[i];
        if (b < 0) continue;
        for (int64_t t = 0; t < P; ++t)
            if ((int64_t)P * b + t < n) tok[nt++] = (int64_t)P * b + t;
    }
    const double scale = 1.0 / sqrt((double)d);
    for (int32_t g = 0; g < G; ++g) {
        double m = -INFINITY;
        for (int64_t i = 0; i < nt; ++i) {
            double s = 0.0;
            for (int32_t j = 0; j < d; ++j)
                s += (double)bf16_to_f32(q[(int64_t)g * d + j]) *
                     (double)bf16_to_f32(K[tok[i] * d + j]);
            z[i] = s * scale;
            if (z[i] > m) m = z[i];
        }
        double l = 0.0;
        for (int32_t j = 0; j < d; ++j) acc[j] = 0.0;
        for (int64_t i = 0; i < nt; ++i) {
            double p = exp(z[i] - m);
            l += p;
            for (int32_t j = 0; j < d; ++j) acc[j] += p * (double)bf16_to_f32(V[tok[i] * d + j]);
        }
        for (int32_t j = 0; j < d; ++j) o[(int64_t)g * d + j] = (float)(acc[j] / l);
        if (lse) lse[g] = (float)(m + log(l));
    }
    free(tok); free(z); free(acc);
}

/* ================================================= O9-O10 hierarchical index
 * "the KV cache is partitioned into chunks, and the mean key of each page is used
 * as its representative, forming higher-level centroids for similarity grouping.
 * Unlike global K-means-based ANNS approaches, this hierarchical structure
 * preserves local semantic continuity among contiguous tokens";
 * "a larger number of centroids improves selection granularity but increases
 * selection cost, as each query must compare against more index representatives"
 * (PAPER.md:549).  Reading R27: blocks (the chunks, with their O1
 * summaries) are clustered inside windows of OR_IDX_WIN consecutive blocks (local
 * grouping) by Lloyd k-means into ceil(len / ratio) centroids per window:
 *   init     centroid i of a window of len blocks = summary of block
 *            start + floor(i * len / nw)  (fp32 of its bf16 values)
 *   assign   block b -> argmin_c dist(b, c), dist = fma chain over j = 0..127 of
 *            (s_b[j] - c[j])^2 from +0 (fp32), ties -> lowest c
 *   update   c[j] = (sum over members in block order from +0) / count (fp32, IEEE);
 *            a centroid without members keeps its value
 *   OR_IDX_ITERS (assign, update) rounds, then a final assign.  Centroids left
 *   without members are dropped; the others are numbered window by window in
 *   ascending order and stored as bf16 (RNE) vectors.
 * Outputs: centroids [nc][d] bf16, cent_of[nb] (block -> centroid), returns nc. */
#define OR_IDX_WIN 64
#define OR_IDX_ITERS 4

static float or_dist(const float* a, const float* c, int32_t d) {
    float acc = 0.0f;
    for (int32_t j = 0; j < d; ++j) {
        float diff = a[j] - c[j];
        acc = fmaf(diff, diff, acc);
    }
    return acc;
}

int64_t or_index_build(const uint16_t* S, int64_t nb, int32_t d, int32_t ratio,
                       uint16_t* centroids, int32_t* cent_of) {
    int64_t nc = 0;
    float* x = (float*)malloc(sizeof(float) * OR_IDX_WIN * (size_t)d);
    float* c = (float*)malloc(sizeof(float) * OR_IDX_WIN * (size_t)d);
    int32_t* as = (int32_t*)malloc(sizeof(int32_t) * OR_IDX_WIN);
    int32_t* cnt = (int32_t*)malloc(sizeof(int32_t) * OR_IDX_WIN);
    int32_t* newid = (int32_t*)malloc(sizeof(int32_t) * OR_IDX_WIN);
    for (int64_t w0 = 0; w0 < nb; w0 += OR_IDX_WIN) {
        int32_t len = (int32_t)(nb - w0 < OR_IDX_WIN ? nb - w0 : OR_IDX_WIN);
        int32_t nw = (len + ratio - 1) / ratio;
        for (int32_t b = 0; b < len; ++b)
            for (int32_t j = 0; j < d; ++j) x[b * d + j] = bf16_to_f32(S[(w0 + b) * d + j]);
        for (int32_t i = 0; i < nw; ++i) {
            int32_t b = (int32_t)(((int64_t)i * len) / nw);
            for (int32_t j = 0; j < d; ++j) c[i * d + j] = x[b * d + j];
        }
        for (int32_t it = 0; it <= OR_IDX_ITERS; ++it) {
            /* assign */
            for (int32_t b = 0; b < len; ++b) {
                int32_t best = 0;
                float bd = or_dist(x + b * d, c, d);
                for (int32_t i = 1; i < nw; ++i) {
                    float di = or_dist(x + b * d, c + i * d, d);
                    if (di < bd) { bd = di; best = i; }
                }
                as[b] = best;
            }
            if (it == OR_IDX_ITERS) break;          /* final assignment only */
            /* update */
            for (int32_t i = 0; i < nw; ++i) {
                int32_t n = 0;
                for (int32_t b = 0; b < len; ++b) n += as[b] == i;
                if (n == 0) continue;
                for (int32_t j = 0; j < d; ++j) {
                    float acc = 0.0f;
                    for (int32_t b = 0; b < len; ++b)
                        if (as[b] == i) acc = acc + x[b * d + j];
                    c[i * d + j] = acc / (float)n;
                }
            }
        }
        for (int32_t i = 0; i < nw; ++i) cnt[i] = 0;
        for (int32_t b = 0; b < len; ++b) cnt[as[b]]++;
        for (int32_t i = 0; i < nw; ++i) {
            if (cnt[i] == 0) { newid[i] = -1; continue; }
            newid[i] = (int32_t)nc;
            for (int32_t j = 0; j < d; ++j) centroids[nc * d + j] = or_f32_to_bf16_rne(c[i * d + j]);
            ++nc;
        }
        for (int32_t b = 0; b < len; ++b) cent_of[w0 + b] = newid[as[b]];
    }
    free(x); free(c); free(as); free(cnt); free(newid);
    return nc;
}

/* O10 two-stage descent ("identifying critical KV entries via the index";
 * reading R27): stage 1 scores every centroid like a block (O3: fma chain of qbar x
 * centroid) and keeps the m best (score desc, centroid index asc; NaN lowest,
 * -0 == +0); stage 2 takes the non-pinned member blocks of those centroids as
 * candidates -- every non-pinned block if they are fewer than k -- scores them
 * exactly (O3) and returns the k best candidates (O5 order), ascending by id.
 * cscores[nc] receives the centroid scores, la[nb] the lookahead eviction score of
 * every block: its exact score if it was a candidate, else its centroid's score.
 * Returns 0, or 2 (ERANGE) when k exceeds the non-pinned blocks. */
int32_t or_index_select(const float* qbar, const uint16_t* S, const uint16_t* centroids,
                        const int32_t* cent_of, int64_t nb, int64_t nc, int32_t d,
                        const uint8_t* is_pinned, int32_t k, int32_t m,
                        int32_t* ids, float* cscores, float* la) {
    or_block_scores(qbar, centroids, nc, d, cscores);
    uint8_t* zero = (uint8_t*)calloc((size_t)(nc > 0 ? nc : 1), 1);
    if (m > nc) m = (int32_t)nc;
    int32_t* top = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int32_t rc = or_topk(cscores, nc, zero, m, top);            /* O5 order over centroids */
    free(zero);
    if (rc) { free(top); return rc; }
    uint8_t* chosen = (uint8_t*)calloc((size_t)(nc > 0 ? nc : 1), 1);
    for (int32_t i = 0; i < m; ++i) chosen[top[i]] = 1;
    free(top);
    /* candidates: non-pinned members of the chosen centroids; all non-pinned if < k */
    uint8_t* excl = (uint8_t*)malloc((size_t)(nb > 0 ? nb : 1));   /* 1 = not a candidate */
    int64_t ncand = 0, nfree = 0;
    for (int64_t b = 0; b < nb; ++b) {
        nfree += !is_pinned[b];
        excl[b] = (uint8_t)(is_pinned[b] || !chosen[cent_of[b]]);
        ncand += !excl[b];
    }
    free(chosen);
    if (ncand < k)
        for (int64_t b = 0; b < nb; ++b) excl[b] = is_pinned[b];
    float* bs = (float*)malloc(sizeof(float) * (size_t)(nb > 0 ? nb : 1));
    or_block_scores(qbar, S, nb, d, bs);                         /* exact scores (O3) */
    for (int64_t b = 0; b < nb; ++b) la[b] = excl[b] ? cscores[cent_of[b]] : bs[b];
    if (k > nfree) { free(bs); free(excl); return 2; }
    rc = or_topk(bs, nb, excl, k, ids);                          /* O5 over the candidates */
    free(bs); free(excl);
    return rc;
}

/* ============================================ O11 2D layer-head window scaling
 * "For each layer l and head h, profiling yields: Benefit_{l,h}(w): transfer reduction
 * achieved with window size w, Cost_{l,h}(w): additional GPU memory consumed by that window
 * size.  Given a total GPU cache budget M, the objective is max sum Benefit s.t. sum Cost <= M
 * ... a variant of the multiple-choice knapsack problem ... for small models, exhaustive search
 * is feasible; for larger ones, we employ a greedy algorithm that starts from the smallest
 * windows and iteratively enlarges the window with the highest benefit-to-cost ratio until the
 * GPU cache budget is met".  benefit/cost: [pairs][sizes], sizes in
 * increasing cost order.  choice[pairs] receives the chosen size index.
 *
 * or_mckp_greedy: all pairs at size 0; repeatedly apply the single upgrade (pair p -> size s > its
 * current size) with the highest (benefit gain) / (cost gain) among those that fit the budget
 * (ties: lower pair, then lower size); stop when none fits.  Returns the total benefit, or
 * -1 if the smallest sizes already exceed the budget. */
double or_mckp_greedy(const double* benefit, const double* cost, int32_t pairs, int32_t sizes,
                      double budget, int32_t* choice) {
    double used = 0.0, total = 0.0;
    for (int32_t p = 0; p < pairs; ++p) { choice[p] = 0; used += cost[p * sizes]; total += benefit[p * sizes]; }
    if (used > budget) return -1.0;
    for (;;) {
        int32_t bp = -1, bs = -1;
        double br = 0.0;
        for (int32_t p = 0; p < pairs; ++p) {
            int32_t cur = choice[p];
            for (int32_t s = cur + 1; s < sizes; ++s) {
                double dc = cost[p * sizes + s] - cost[p * sizes + cur];
                double db = benefit[p * sizes + s] - benefit[p * sizes + cur];
                if (used + dc > budget) continue;
                double r = dc > 0 ? db / dc : (db > 0 ? INFINITY : 0.0);
                if (db <= 0.0 && dc >= 0.0) continue;            /* no gain */
                if (bp < 0 || r > br) { bp = p; bs = s; br = r; }
            }
        }
        if (bp < 0) break;
        used += cost[bp * sizes + bs] - cost[bp * sizes + choice[bp]];
        total += benefit[bp * sizes + bs] - benefit[bp * sizes + choice[bp]];
        choice[bp] = bs;
    }
    return total;
}

/* or_mckp_exact: the optimum by enumeration of every allocation (sizes^pairs <= 1e7), ties ->
 * the lexicographically smallest allocation.  Returns the best total benefit or -1. */
double or_mckp_exact(const double* benefit, const double* cost, int32_t pairs, int32_t sizes,
                     double budget, int32_t* choice) {
    double combos = 1.0;
    for (int32_t p = 0; p < pairs; ++p) combos *= sizes;
    if (combos > 1e7 || pairs < 1) return -1.0;
    int32_t* cur = (int32_t*)calloc((size_t)pairs, sizeof(int32_t));
    double best = -1.0;
    for (;;) {
        double c = 0.0, b = 0.0;
        for (int32_t p = 0; p < pairs; ++p) { c += cost[p * sizes + cur[p]]; b += benefit[p * sizes + cur[p]]; }
        if (c <= budget && b > best) {
            best = b;
            for (int32_t p = 0; p < pairs; ++p) choice[p] = cur[p];
        }
        int32_t p = pairs - 1;                    /* next allocation, lexicographic */
        while (p >= 0 && ++cur[p] == sizes) cur[p--] = 0;
        if (p < 0) break;
    }
    free(cur);
    return best;
}

/* ====================================== O12 Quest min/max block summaries (baseline)
 * "Quest partitions key entries into chunks and estimates their importance by multiplying the
 * query vector with the channel-wise minimum and maximum of the keys".
 * Reading R30: per block and dim, mn[b][j] = min and mx[b][j] = max of the valid tokens' bf16
 * keys (exact: a min / max of bf16 values is a bf16 value); the block's score bounds the dot
 * product of the query with any of its keys:
 *   acc = +0f; for j in 0..d-1: acc = acc + fmaxf(qbar[j] * mn[b][j], qbar[j] * mx[b][j])
 * (fp32, products rounded, sequential in j).  Selection is then O4-O5 on these scores. */
void or_minmax_summaries(const uint16_t* K, int64_t n, int32_t d, int32_t P, uint16_t* MN, uint16_t* MX) {
    int64_t nb = (n + P - 1) / P;
    for (int64_t b = 0; b < nb; ++b) {
        int64_t cnt = n - (int64_t)P * b;
        if (cnt > P) cnt = P;
        for (int32_t j = 0; j < d; ++j) {
            uint16_t lo = K[((int64_t)P * b) * d + j], hi = lo;
            for (int64_t t = 1; t < cnt; ++t) {
                uint16_t x = K[((int64_t)P * b + t) * d + j];
                if (bf16_to_f32(x) < bf16_to_f32(lo)) lo = x;
                if (bf16_to_f32(x) > bf16_to_f32(hi)) hi = x;
            }
            MN[b * d + j] = lo;
            MX[b * d + j] = hi;
        }
    }
}

void or_minmax_scores(const float* qbar, const uint16_t* MN, const uint16_t* MX, int64_t nb, int32_t d,
                      float* scores) {
    for (int64_t b = 0; b < nb; ++b) {
        float acc = 0.0f;
        for (int32_t j = 0; j < d; ++j) {
            float a = qbar[j] * bf16_to_f32(MN[b * d + j]);
            float c = qbar[j] * bf16_to_f32(MX[b * d + j]);
            acc = acc + fmaxf(a, c);
        }
        scores[b] = acc;
    }
}

/* ============================================ O13 decode-time append (block admission)
 * "each step appending new key and value vectors to the cache".  Reading R16
 * (round 2): the appended token goes to the always-resident local window; when it opens a new
 * block b (= the old block count), that block is admitted like a miss at `step`: a resident cache
 * (C >= blocks) keeps block b in slot b; otherwise the free slot with the lowest index, else the
 * resident block with the smallest O6 policy key among those not pinned after the append (victim:
 * table entry cleared).  Admitted: last = step, phase = 1, count = 1.  table / is_pinned have the
 * new block count nb_new = b + 1 entries.  Returns 0, or 3 (ECAPACITY) when nothing is evictable. */
int32_t or_append_block(int64_t nb_new, int64_t C, const uint8_t* is_pinned, int32_t* table, int32_t* slot_block,
                        uint32_t* last_use, uint8_t* phase, uint32_t* use_count, uint32_t step, int32_t policy,
                        const float* scores) {
    int64_t b = nb_new - 1, dest = -1;
    if (C >= nb_new) {
        dest = b;
    } else {
        for (int64_t s = 0; s < C && dest < 0; ++s)
            if (slot_block[s] < 0) dest = s;
        if (dest < 0) {
            or_victim best;
            int have = 0;
            for (int64_t s = 0; s < C; ++s) {
                int32_t blk = slot_block[s];
                if (blk < 0 || blk >= b || is_pinned[blk]) continue;
                or_victim v = {s, blk, last_use[s], use_count[s], phase[s], scores ? scores[blk] : 0.0f, policy};
                if (!have || or_victim_cmp(&v, &best) < 0) { best = v; have = 1; }
            }
            if (!have) return 3;
            table[best.block] = -1;
            dest = best.slot;
        }
    }
    table[b] = (int32_t)dest;
    slot_block[dest] = (int32_t)b;
    last_use[dest] = step; phase[dest] = 1; use_count[dest] = 1;
    return 0;
}
