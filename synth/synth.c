/*
 * synth.c — seeded synthetic input generator (inputs only).
 *
 * Shared by the CUDA path's tests/bench and by the oracle's tests: it holds
 * NONE of the method's arithmetic (no summaries, scores, selection, cache or
 * attention).  It only turns (seed, layer, request, kv-head, index) counters
 * into bf16 keys, values and decode queries with the structure of the paper's
 * workloads (DESIGN.md §4 "input recipe"):
 *
 *  keys    k_i = mu_{tau(i)} + 0.5 eps_i.  T = 32 topic centres per segment,
 *          mu ~ N(0, I_d) (per-dim unit variance).  Tokens come in topic runs
 *          of geometric length (mean 48 tokens ~ 3 blocks), modelling "local
 *          semantic continuity among contiguous tokens".
 *  values  v_i ~ N(0, I_d).
 *  queries per decode step t: sticky topic tau_t (kept w.p. 0.9), base
 *          direction u_t = normalise(alpha u_{t-1} + (1-alpha)(mu_tau/|mu_tau|
 *          + 0.3 eps)); head g: q = sqrt(d) normalise(u_t + 0.3 eps_g).
 *          alpha = 0.9 "locality-high" (temporal locality),
 *          alpha = 0 "locality-none".
 *  All values are rounded to bf16 (RNE) — the inputs are bf16 tensors.
 *
 * Counter-based (SplitMix64 finaliser over a keyed counter) so any segment can
 * be regenerated independently and in parallel, bit-identically.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t sm_mix(uint64_t x) {
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27; x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}
/* key for one (seed, layer, req, head, stream) tuple */
static inline uint64_t seg_key(uint64_t seed, int64_t l, int64_t r, int64_t h, uint64_t stream) {
    uint64_t k = sm_mix(seed + 0x9E3779B97F4A7C15ull);
    k = sm_mix(k ^ ((uint64_t)l * 0xD1B54A32D192ED03ull));
    k = sm_mix(k ^ ((uint64_t)r * 0xABC98388FB8FAC03ull));
    k = sm_mix(k ^ ((uint64_t)h * 0x8CB92BA72F3D8DD7ull));
    k = sm_mix(k ^ (stream * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull));
    return k;
}
static inline uint64_t ctr_u64(uint64_t key, uint64_t ctr) {
    return sm_mix(key ^ sm_mix(ctr + 0x9E3779B97F4A7C15ull));
}
static inline double ctr_unif(uint64_t key, uint64_t ctr) {       /* (0,1) */
    return ((double)(ctr_u64(key, ctr) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
/* Approximately N(0,1): Irwin-Hall sum of four 16-bit uniforms from one hash,
 * centred and scaled to unit variance (tails bounded at +-3.46).  Integer and
 * exact float arithmetic only: identical on every host. */
static inline float ctr_normal(uint64_t key, uint64_t ctr) {
    uint64_t x = ctr_u64(key, ctr);
    uint32_t s = (uint32_t)(x & 0xFFFF) + (uint32_t)((x >> 16) & 0xFFFF) +
                 (uint32_t)((x >> 32) & 0xFFFF) + (uint32_t)(x >> 48);      /* 0 .. 4*65535 */
    return ((float)s - 131070.0f) * (1.7320508f / 65536.0f);
}
static inline uint16_t to_bf16(float f) {
    uint32_t u; memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

enum { ST_MU = 1, ST_RUN = 2, ST_KEYNOISE = 3, ST_VAL = 4, ST_QTOPIC = 5, ST_QBASE = 6, ST_QHEAD = 7 };
#define SYN_TOPICS 32
#define SYN_RUN_MEAN 48.0

/* topic of every token of a segment (sequential run scan, cheap) */
static void token_topics(uint64_t seed, int64_t l, int64_t r, int64_t h, int64_t n, uint8_t* topic) {
    uint64_t kr = seg_key(seed, l, r, h, ST_RUN);
    uint8_t cur = (uint8_t)(ctr_u64(kr, 0) % SYN_TOPICS);
    for (int64_t i = 0; i < n; ++i) {
        if (i > 0 && ctr_unif(kr, 2 * (uint64_t)i + 1) < 1.0 / SYN_RUN_MEAN)
            cur = (uint8_t)(ctr_u64(kr, 2 * (uint64_t)i + 2) % SYN_TOPICS);
        topic[i] = cur;
    }
}

static void topic_centres(uint64_t seed, int64_t l, int64_t r, int64_t h, int32_t d, float* mu) {
    uint64_t km = seg_key(seed, l, r, h, ST_MU);
    for (int64_t i = 0; i < (int64_t)SYN_TOPICS * d; ++i) mu[i] = (float)ctr_normal(km, (uint64_t)i);
}

/* Exported pieces for the device generator (synth_gpu.cu): topic of every
 * token [n] and topic centres [SYN_TOPICS][d] of one segment, plus the two
 * stream keys.  The device side turns these into exactly the bytes
 * synth_segment_kv writes. */
void synth_segment_plan(uint64_t seed, int64_t l, int64_t r, int64_t h, int64_t n, int32_t d,
                        uint8_t* topic, float* mu, uint64_t* keys2) {
    topic_centres(seed, l, r, h, d, mu);
    token_topics(seed, l, r, h, n, topic);
    keys2[0] = seg_key(seed, l, r, h, ST_KEYNOISE);
    keys2[1] = seg_key(seed, l, r, h, ST_VAL);
}

/* Keys and values of one segment, token-major [n][d] bf16 (caller-owned). */
void synth_segment_kv(uint64_t seed, int64_t l, int64_t r, int64_t h, int64_t n, int32_t d,
                      uint16_t* K, uint16_t* V) {
    float* mu = (float*)malloc(sizeof(float) * SYN_TOPICS * (size_t)d);
    uint8_t* topic = (uint8_t*)malloc((size_t)(n > 0 ? n : 1));
    topic_centres(seed, l, r, h, d, mu);
    token_topics(seed, l, r, h, n, topic);
    uint64_t kk = seg_key(seed, l, r, h, ST_KEYNOISE), kv = seg_key(seed, l, r, h, ST_VAL);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const float* m = mu + (int64_t)topic[i] * d;
        for (int32_t j = 0; j < d; ++j) {
            uint64_t c = (uint64_t)i * (uint64_t)d + (uint64_t)j;
            if (K) K[i * d + j] = to_bf16(m[j] + 0.5f * (float)ctr_normal(kk, c));
            if (V) V[i * d + j] = to_bf16((float)ctr_normal(kv, c));
        }
    }
    free(mu); free(topic);
}

/* All Hkv heads of one (layer, request): K, V are [Hkv][n][d] bf16. */
void synth_request_kv(uint64_t seed, int64_t l, int64_t r, int32_t Hkv, int64_t n, int32_t d,
                      uint16_t* K, uint16_t* V) {
    for (int32_t h = 0; h < Hkv; ++h)
        synth_segment_kv(seed, l, r, h, n, d, K ? K + (int64_t)h * n * d : 0,
                         V ? V + (int64_t)h * n * d : 0);
}

static void normalise(double* x, int32_t d) {
    double s = 0.0;
    for (int32_t j = 0; j < d; ++j) s += x[j] * x[j];
    s = sqrt(s);
    if (s > 0) for (int32_t j = 0; j < d; ++j) x[j] /= s;
}

/* Decode queries of one segment's G query heads for steps t0 .. t0+nsteps-1:
 * out [nsteps][G][d] bf16.  The AR(1) state is replayed from t = 0.  The topic
 * centres are those of the keys of layer lk; the random streams (topic walk,
 * base and head noise) are those of layer ls (ls == lk: synth_queries). */
static void queries_impl(uint64_t seed, int64_t lk, int64_t ls, int64_t r, int64_t h, int32_t G, int32_t d,
                         int64_t t0, int64_t nsteps, double alpha, uint16_t* out) {
    const int64_t l = ls;
    float* mu = (float*)malloc(sizeof(float) * SYN_TOPICS * (size_t)d);
    double* u = (double*)malloc(sizeof(double) * (size_t)d);
    double* x = (double*)malloc(sizeof(double) * (size_t)d);
    double* e = (double*)malloc(sizeof(double) * (size_t)d);
    topic_centres(seed, lk, r, h, d, mu);
    uint64_t kt = seg_key(seed, l, r, h, ST_QTOPIC), kb = seg_key(seed, l, r, h, ST_QBASE),
             kh = seg_key(seed, l, r, h, ST_QHEAD);
    int32_t tau = (int32_t)(ctr_u64(kt, 0) % SYN_TOPICS);
    for (int32_t j = 0; j < d; ++j) u[j] = 0.0;
    for (int64_t t = 0; t < t0 + nsteps; ++t) {
        if (t > 0 && ctr_unif(kt, 2 * (uint64_t)t + 1) >= 0.9)
            tau = (int32_t)(ctr_u64(kt, 2 * (uint64_t)t + 2) % SYN_TOPICS);
        for (int32_t j = 0; j < d; ++j) e[j] = mu[(int64_t)tau * d + j];
        normalise(e, d);
        for (int32_t j = 0; j < d; ++j)
            e[j] += 0.3 / sqrt((double)d) * ctr_normal(kb, (uint64_t)t * (uint64_t)d + (uint64_t)j);
        double a = (t == 0) ? 0.0 : alpha;
        for (int32_t j = 0; j < d; ++j) u[j] = a * u[j] + (1.0 - a) * e[j];
        normalise(u, d);
        if (t < t0) continue;
        for (int32_t g = 0; g < G; ++g) {
            for (int32_t j = 0; j < d; ++j)
                x[j] = u[j] + 0.3 / sqrt((double)d) *
                       ctr_normal(kh, ((uint64_t)t * (uint64_t)G + (uint64_t)g) * (uint64_t)d + (uint64_t)j);
            normalise(x, d);
            uint16_t* o = out + ((t - t0) * G + g) * (int64_t)d;
            for (int32_t j = 0; j < d; ++j) o[j] = to_bf16((float)(sqrt((double)d) * x[j]));
        }
    }
    free(mu); free(u); free(x); free(e);
}

void synth_queries(uint64_t seed, int64_t l, int64_t r, int64_t h, int32_t G, int32_t d,
                   int64_t t0, int64_t nsteps, double alpha, uint16_t* out) {
    queries_impl(seed, l, l, r, h, G, d, t0, nsteps, alpha, out);
}

/* Queries of a whole batch for one layer and a range of steps:
 * out [nsteps][B][Hq][d] with Hq = Hkv*G; request ids req[B].  Key topics of
 * layer lk, random streams of layer ls (synth_batch_queries: ls == lk). */
void synth_batch_queries_x(uint64_t seed, int64_t lk, int64_t ls, const int32_t* req, int32_t B, int32_t Hkv,
                           int32_t G, int32_t d, int64_t t0, int64_t nsteps, double alpha, uint16_t* out) {
    int64_t Hq = (int64_t)Hkv * G;
    #pragma omp parallel for schedule(dynamic) collapse(2)
    for (int32_t b = 0; b < B; ++b)
        for (int32_t h = 0; h < Hkv; ++h) {
            uint16_t* tmp = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(nsteps * G * d));
            queries_impl(seed, lk, ls, req[b], h, G, d, t0, nsteps, alpha, tmp);
            for (int64_t t = 0; t < nsteps; ++t)
                memcpy(out + ((t * B + b) * Hq + (int64_t)h * G) * d, tmp + t * G * d,
                       sizeof(uint16_t) * (size_t)G * (size_t)d);
            free(tmp);
        }
}

void synth_batch_queries(uint64_t seed, int64_t l, const int32_t* req, int32_t B, int32_t Hkv,
                         int32_t G, int32_t d, int64_t t0, int64_t nsteps, double alpha,
                         uint16_t* out) {
    synth_batch_queries_x(seed, l, l, req, B, Hkv, G, d, t0, nsteps, alpha, out);
}
