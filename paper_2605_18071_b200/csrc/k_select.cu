// k_select.cu — rows (a1) summary scoring and (a2) top-k block selection.
//
// (a1) "identifying critical KV entries via the index": every
// block's score is the dot product of the KV head's group query with the
// block's mean-key summary, computed as one fp32 FMA chain
// over the 128 dims in order (DESIGN.md §3 R3, R5) so that ids are bit-exact.
// HBM-bound: 256 B of summary per block.  The summaries are dim-major, so a
// thread owning V consecutive blocks reads one V*2-byte vector per dim row and
// a warp reads 64*V contiguous bytes per row (coalesced).  No shared-memory
// staging: each thread keeps 16-32 rows of its blocks in flight (two ping-pong
// register batches) and runs V independent chains.  V in {2, 4, 8} is picked so the
// grid has >= 2 CTAs per SM.  Rows for the first batch are requested before
// griddepcontrol.wait (summaries are immutable during a step), overlapping
// the previous kernel's tail.
//
// (a2) "retrieving only the Top-K important chunks", fused:
// the last scoring CTA of a segment to finish (arrival counter per segment)
// selects that segment's top-k while other CTAs keep streaming summaries.
// Thread t owns the contiguous blocks [t*KPT*reps, (t+1)*KPT*reps) (keys in
// registers when reps == 1).  A 3-pass radix select (11 + 11 + 10 bits,
// warp-aggregated shared histograms) finds the k-th largest monotone key T
// among the candidates; keys > T are taken and the kk lowest-id keys == T
// (R10).  Two block scans give tie ranks and output positions, so ids come out
// ascending with no sort.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace kvd {

constexpr int kScoreThreads = 256;
constexpr int64_t kDirectTopkMax = 16384;     // segments up to this many blocks: direct top-k

template <int V>
struct VecOf;
template <>
struct VecOf<2> {
    using T = uint32_t;
    static __device__ __forceinline__ uint32_t word(const T& x, int) { return x; }
};
template <>
struct VecOf<4> {
    using T = uint2;
    static __device__ __forceinline__ uint32_t word(const T& x, int i) { return i ? x.y : x.x; }
};
template <>
struct VecOf<8> {
    using T = uint4;
    static __device__ __forceinline__ uint32_t word(const T& x, int i) {
        return i == 0 ? x.x : i == 1 ? x.y : i == 2 ? x.z : x.w;
    }
};

template <int V>
__device__ __forceinline__ void score_tile(const StepParams& p, int bi, int h, int64_t nb, int64_t seg,
                                           const uint16_t* __restrict__ q, const uint16_t* __restrict__ summ,
                                           float* __restrict__ scores, float* qbar, float (&acc)[V]) {
    using Vec = typename VecOf<V>::T;
    const int64_t b0 = (int64_t)blockIdx.x * kScoreThreads * V + (int64_t)threadIdx.x * V;
    const bool ld = b0 < nb;                      // V-groups never straddle nb_pad (V | 128)
    const Vec* base = reinterpret_cast<const Vec*>(summ + seg * kHeadDim * p.nb_pad + (ld ? b0 : 0));
    const int64_t rstride = p.nb_pad / V;         // Vec elements per dim row
    // two register batches of R rows (ping-pong): while one batch is consumed the
    // other is in flight, so 2R rows of this thread's blocks are always requested
    constexpr int R = V == 8 ? 8 : 16;
    Vec bufA[R], bufB[R];
#pragma unroll
    for (int u = 0; u < R; ++u)
        if (ld) bufA[u] = __ldcs(base + u * rstride);
#pragma unroll
    for (int u = 0; u < R; ++u)
        if (ld) bufB[u] = __ldcs(base + (R + u) * rstride);
    griddep_wait();                               // summaries are immutable; q may come from an earlier kernel
    if (threadIdx.x < kHeadDim) {
        // group query: qbar[j] = ((+0 + q_0[j]) + q_1[j]) + ... (fp32, g ascending; R3)
        const uint16_t* qh = q + ((int64_t)bi * p.Hq + (int64_t)h * p.G) * kHeadDim;
        float a = 0.0f;
        for (int g = 0; g < p.G; ++g) a = __fadd_rn(a, bf16_bits(qh[g * kHeadDim + threadIdx.x]));
        qbar[threadIdx.x] = a;
    }
    __syncthreads();
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.0f;
    auto consume = [&](const Vec (&buf)[R], int j0) {
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const float qj = qbar[j0 + u];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const uint32_t w = VecOf<V>::word(buf[u], v >> 1);
                acc[v] = __fmaf_rn(qj, (v & 1) ? bf16_hi(w) : bf16_lo(w), acc[v]);   // sequential in j (R5)
            }
        }
    };
#pragma unroll 1
    for (int j0 = 0; j0 < kHeadDim; j0 += 2 * R) {
        consume(bufA, j0);
        if (ld && j0 + 2 * R < kHeadDim) {
#pragma unroll
            for (int u = 0; u < R; ++u) bufA[u] = __ldcs(base + (j0 + 2 * R + u) * rstride);
        }
        consume(bufB, j0 + R);
        if (ld && j0 + 3 * R < kHeadDim) {
#pragma unroll
            for (int u = 0; u < R; ++u) bufB[u] = __ldcs(base + (j0 + 3 * R + u) * rstride);
        }
    }
    griddep_launch();
    if (!ld) return;
    float* out = scores + seg * p.nb_pad + b0;
    if (b0 + V <= nb) {
#pragma unroll
        for (int v = 0; v < V; v += 2) *reinterpret_cast<float2*>(out + v) = make_float2(acc[v], acc[v + 1]);
    } else {
#pragma unroll
        for (int v = 0; v < V; ++v)
            if (b0 + v < nb) out[v] = acc[v];
    }
}

struct TopkSmem {
    int hist[2048];
    int scan[33];
    uint32_t wmin[32], wmax[32];
    uint32_t digit;
    int above;
};

// CTA-wide top-k (blockDim.x threads, all call it).  Thread t owns `reps` chunks of KPT
// consecutive positions; positions ascend with (t, chunk, i), so emission order is
// ascending position.  load(c, key[KPT], &cm) fills chunk c's monotone keys and
// candidate mask; emit(pos, c, i) writes output slot pos for element (c, i) of this
// thread.  Selects the k largest keys among candidates, ties to the lowest position
// (R10); k must not exceed the candidate count.  3-pass radix select (11 + 11 + 10
// bits) with warp-aggregated shared histograms, then two block scans.
template <int KPT, class Load, class Emit>
__device__ void cta_topk(int k, int reps, Load load, Emit emit, TopkSmem& sm,
                         unsigned long long* ph = nullptr) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    auto phs = [&](int i) {
        if (ph && tid == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            ph[i] = t;
        }
    };
    uint32_t key[KPT];
    uint32_t cm = 0;
    if (reps == 1) load(0, key, cm);
    phs(0);
    // ---- key range of the candidates: the digits start at the highest bit where the
    // candidate keys differ (bits above it are common), so the first histogram is not
    // concentrated in one bin and plain shared atomics suffice
    uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
#pragma unroll 1
    for (int c = 0; c < reps; ++c) {
        if (reps > 1) load(c, key, cm);
#pragma unroll
        for (int i = 0; i < KPT; ++i)
            if ((cm >> i) & 1u) {
                kmin = min(kmin, key[i]);
                kmax = max(kmax, key[i]);
            }
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if ((tid & 31) == 0) {
        sm.wmin[tid >> 5] = kmin;
        sm.wmax[tid >> 5] = kmax;
    }
    __syncthreads();
    kmin = 0xFFFFFFFFu;
    kmax = 0u;
    for (int w = 0; w < (nthr >> 5); ++w) {
        kmin = min(kmin, sm.wmin[w]);
        kmax = max(kmax, sm.wmax[w]);
    }
    const uint32_t diff = kmin ^ kmax;
    int lo = diff ? 32 - __clz(diff) : 0;         // bits [0, lo) still to resolve
    uint32_t mask = lo == 32 ? 0u : ~((1u << lo) - 1u);
    uint32_t prefix = kmin & mask;
    int kk = k;
    phs(0);
#pragma unroll 1
    for (int pass = 0; lo > 0; ++pass) {
        const int width = min(11, lo);
        const int shift = lo - width;
        const int nbins = 1 << width;
        for (int i = tid; i < nbins; i += nthr) sm.hist[i] = 0;
        __syncthreads();
#pragma unroll 1
        for (int c = 0; c < reps; ++c) {
            if (reps > 1) load(c, key, cm);
#pragma unroll
            for (int i = 0; i < KPT; ++i)
                if (((cm >> i) & 1u) && (key[i] & mask) == prefix)
                    atomicAdd(&sm.hist[(key[i] >> shift) & (uint32_t)(nbins - 1)], 1);
        }
        __syncthreads();
        // bins in descending order; thread t owns bins [nbins - (t+1) bpt, nbins - t bpt)
        const int bpt = (nbins + nthr - 1) / nthr;
        int cnt = 0;
        for (int i = 0; i < bpt; ++i) {
            const int d = nbins - 1 - (tid * bpt + i);
            if (d >= 0) cnt += sm.hist[d];
        }
        int tot;
        int above = block_exclusive_scan(cnt, sm.scan, &tot);
        if (above < kk && kk <= above + cnt) {
            for (int i = 0; i < bpt; ++i) {
                const int d = nbins - 1 - (tid * bpt + i);
                const int ci = d >= 0 ? sm.hist[d] : 0;
                if (above + ci >= kk) {
                    sm.digit = (uint32_t)d;
                    sm.above = above;
                    break;
                }
                above += ci;
            }
        }
        __syncthreads();
        prefix |= sm.digit << shift;
        mask |= (uint32_t)(nbins - 1) << shift;
        kk -= sm.above;
        lo = shift;
        __syncthreads();
        phs(1 + min(pass, 2));
    }
    const uint32_t T = prefix;                    // take keys > T, and the kk lowest-position keys == T
    int ngt = 0, neq = 0;
#pragma unroll 1
    for (int c = 0; c < reps; ++c) {
        if (reps > 1) load(c, key, cm);
#pragma unroll
        for (int i = 0; i < KPT; ++i) {
            const bool cand = (cm >> i) & 1u;
            ngt += (cand && key[i] > T) ? 1 : 0;
            neq += (cand && key[i] == T) ? 1 : 0;
        }
    }
    int tot;
    const int tie0 = block_exclusive_scan(neq, sm.scan, &tot);
    const int ntake = min(max(kk - tie0, 0), neq);
    int pos = block_exclusive_scan(ngt + ntake, sm.scan, &tot);
    phs(4);
    int tie = tie0;
#pragma unroll 1
    for (int c = 0; c < reps; ++c) {
        if (reps > 1) load(c, key, cm);
#pragma unroll
        for (int i = 0; i < KPT; ++i) {
            if (!((cm >> i) & 1u)) continue;
            bool take = key[i] > T;
            if (key[i] == T) take = tie++ < kk;
            if (take) emit(pos++, c, i);
        }
    }
}

// Two-level top-k (a2).  Every scoring CTA first keeps its tile's local top-k
// candidates (the k largest (key, -id) pairs of its V*256 blocks, or all of them):
// the segment's top-k is a subset of the union of the tiles' local top-k, so the
// final selection only ranks ntiles*k candidates.  Candidates are stored per tile
// in ascending id order, so the concatenation over tiles is ascending too.  The
// last CTA of the segment to finish (arrival counter) runs the final selection.
struct SelBufs {
    unsigned long long* trace;   // KVD_SEL_TRACE: per-CTA globaltimer stamps [ctas][4] (experiments only)
    uint32_t* cand_key;     // [R][Hkv][max_tiles][kmax]
    int32_t* cand_id;       // [R][Hkv][max_tiles][kmax]
    int32_t* cand_cnt;      // [R][Hkv][max_tiles]
    uint32_t* ctr;          // [R][Hkv]
    int32_t max_tiles, kmax;
};

// grid (tiles per segment, Hkv, B); CTA = kScoreThreads threads scoring kScoreThreads*V blocks.
// TWO = two-level selection (tile-local candidates first; used when nb > 16384) or the
// direct selection over all of the segment's scores by the last CTA.
template <int V, int KPT, bool TWO>
__global__ void __launch_bounds__(kScoreThreads, 2) select_kernel(StepParams p, const uint16_t* __restrict__ q,
                                                                  const uint16_t* __restrict__ summ,
                                                                  float* __restrict__ scores,
                                                                  const int32_t* __restrict__ ntok, SelBufs sb,
                                                                  int reps, int32_t* __restrict__ out_ids,
                                                                  float* __restrict__ out_scores) {
    __shared__ float qbar[kHeadDim];
    __shared__ TopkSmem sm;
    __shared__ int s_last, s_off[kMaxSelTiles + 1];
    const int bi = blockIdx.z, h = blockIdx.y, tile = blockIdx.x;
    const int r = p.req[bi];
    const int n = ntok[r];                        // written only by kvd_load_prefix (setup)
    const int64_t nb = (n + p.P - 1) / p.P;
    const int64_t bpc = (int64_t)kScoreThreads * V;
    if ((int64_t)tile * bpc >= nb) return;        // whole CTA past this request's end (does not arrive)
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    float acc[V];
    const int64_t cta_lin = ((int64_t)bi * p.Hkv + h) * gridDim.x + tile;
    auto stamp = [&](int i) {
        if (sb.trace && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            sb.trace[cta_lin * 4 + i] = t;
        }
    };
    stamp(0);
    score_tile<V>(p, bi, h, nb, seg, q, summ, scores, qbar, acc);
    stamp(1);
    if (p.k == 0) return;
    const SegGeom g = seg_geom(n, p.P, p.sink_tokens, p.local_tokens);
    const int64_t rs = (int64_t)r * p.Hkv + h;
    const int64_t b0 = (int64_t)tile * bpc + (int64_t)threadIdx.x * V;

    if (TWO) {
    // ---- tile-local candidates
    uint32_t lkey[V];
    uint32_t lcm = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const int64_t b = b0 + v;
        lkey[v] = score_key32(acc[v]);
        lcm |= (uint32_t)(b < g.nb && b >= g.sink_end && b < g.local_begin) << v;
    }
    int tot;
    const int cpos = block_exclusive_scan(__popc(lcm), sm.scan, &tot);   // candidates of the tile
    const int kl = min(p.k, tot);
    uint32_t* ck = sb.cand_key + (rs * sb.max_tiles + tile) * sb.kmax;
    int32_t* ci = sb.cand_id + (rs * sb.max_tiles + tile) * sb.kmax;
    if (tot <= p.k) {                             // every candidate of the tile survives
        int pos = cpos;
#pragma unroll
        for (int v = 0; v < V; ++v)
            if ((lcm >> v) & 1u) {
                ck[pos] = lkey[v];
                ci[pos] = (int32_t)(b0 + v);
                ++pos;
            }
    } else {
        cta_topk<V>(
            kl, 1,
            [&](int, uint32_t (&key)[V], uint32_t& cm) {
#pragma unroll
                for (int v = 0; v < V; ++v) key[v] = lkey[v];
                cm = lcm;
            },
            [&](int pos, int, int v) {
                ck[pos] = lkey[v];
                ci[pos] = (int32_t)(b0 + v);
            },
            sm);
    }
    if (threadIdx.x == 0) sb.cand_cnt[rs * sb.max_tiles + tile] = kl;
    }

    // ---- the last CTA of the segment to finish runs the final selection
    const uint32_t ntiles = (uint32_t)((nb + bpc - 1) / bpc);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&sb.ctr[rs], 1u) == ntiles - 1;
        if (s_last) {
            sb.ctr[rs] = 0u;
            __threadfence();
        }
    }
    __syncthreads();
    if (!s_last) return;
    stamp(2);
    int32_t* ids_out = out_ids + ((int64_t)bi * p.Hkv + h) * p.k;
    float* sc_out = out_scores ? out_scores + ((int64_t)bi * p.Hkv + h) * p.k : nullptr;
    const float* sc = scores + seg * p.nb_pad;
    if (!TWO) {
        // direct: thread t owns blocks [t*KPT*reps, (t+1)*KPT*reps), scores re-read from L2
        cta_topk<KPT>(
            p.k, reps,
            [&](int c, uint32_t (&key)[KPT], uint32_t& cm) {
                const int64_t bb = ((int64_t)threadIdx.x * reps + c) * KPT;
                cm = 0;
                if (bb >= g.nb) return;
#pragma unroll
                for (int i = 0; i < KPT; i += 4) {
                    const float4 x = __ldcg(reinterpret_cast<const float4*>(sc + bb + i));
                    key[i] = score_key32(x.x); key[i + 1] = score_key32(x.y);
                    key[i + 2] = score_key32(x.z); key[i + 3] = score_key32(x.w);
                }
#pragma unroll
                for (int i = 0; i < KPT; ++i) {
                    const int64_t b = bb + i;
                    cm |= (uint32_t)(b < g.nb && b >= g.sink_end && b < g.local_begin) << i;
                }
            },
            [&](int pos, int c, int i) {
                const int64_t b = ((int64_t)threadIdx.x * reps + c) * KPT + i;
                ids_out[pos] = (int32_t)b;
                if (sc_out) sc_out[pos] = __ldcg(&sc[b]);
            },
            sm, sb.trace ? sb.trace + (1 << 18) + cta_lin * 8 : nullptr);
        stamp(3);
        return;
    }
    // candidate offsets per tile (ntiles <= max_tiles <= 128 per pass of this loop)
    int total = 0;
    for (int t0 = 0; t0 < (int)ntiles; t0 += kScoreThreads) {
        const int t = t0 + (int)threadIdx.x;
        const int c = t < (int)ntiles ? __ldcg(&sb.cand_cnt[rs * sb.max_tiles + t]) : 0;
        int tt;
        const int off = block_exclusive_scan(c, sm.scan, &tt);
        if (t < (int)ntiles) s_off[t] = total + off;
        total += tt;
    }
    if (threadIdx.x == 0) s_off[ntiles] = total;
    __syncthreads();
    const int nt_ = (int)ntiles;
    // candidate j (concatenated, ascending id) -> (tile, index): tiles hold kl_t <= kmax entries
    auto cand_at = [&](int j, uint32_t& key, int32_t& id) {
        int lo = 0, hi = nt_;                     // largest t with s_off[t] <= j
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_off[mid] <= j) lo = mid; else hi = mid;
        }
        const int64_t base = (rs * sb.max_tiles + lo) * sb.kmax + (j - s_off[lo]);
        key = __ldcg(&sb.cand_key[base]);
        id = __ldcg(&sb.cand_id[base]);
    };
    const int per = (total + kScoreThreads * reps - 1) / (kScoreThreads * reps);   // <= KPT
    cta_topk<KPT>(
        p.k, reps,
        [&](int c, uint32_t (&key)[KPT], uint32_t& cm) {
            const int j0 = ((int)threadIdx.x * reps + c) * per;
            cm = 0;
#pragma unroll
            for (int i = 0; i < KPT; ++i) {
                key[i] = 0u;
                if (i < per && j0 + i < total) {
                    int32_t id;
                    cand_at(j0 + i, key[i], id);
                    cm |= 1u << i;
                }
            }
        },
        [&](int pos, int c, int i) {
            const int j = ((int)threadIdx.x * reps + c) * per + i;
            uint32_t key;
            int32_t id;
            cand_at(j, key, id);
            ids_out[pos] = id;
            if (sc_out) sc_out[pos] = __ldcg(&sc[id]);
        },
        sm);
}

template <int V, int KPT, bool TWO>
static cudaError_t launch_sel(kvd_cache* c, const StepParams& p, const uint16_t* q, int reps, int32_t* out_ids,
                              float* out_scores, cudaStream_t s) {
    const unsigned tiles = (unsigned)((c->nb_pad + kScoreThreads * V - 1) / (kScoreThreads * V));
    static int trace = -1;
    static unsigned long long* tbuf = nullptr;
    if (trace < 0) {
        trace = getenv("KVD_SEL_TRACE") ? 1 : 0;
        if (trace) cudaMalloc(&tbuf, sizeof(unsigned long long) * ((1 << 18) + 8 * (1 << 16)));
    }
    const int64_t nctas = (int64_t)tiles * p.Hkv * p.B;
    if (trace) cudaMemsetAsync(tbuf, 0, sizeof(unsigned long long) * ((1 << 18) + 8 * (1 << 16)), s);
    SelBufs sb{trace && nctas <= (1 << 16) ? tbuf : nullptr, c->cand_key, c->cand_id, c->cand_cnt, c->sel_ctr, c->max_sel_tiles, c->kmax > 0 ? c->kmax : 1};
    cudaError_t e = launch_pdl(select_kernel<V, KPT, TWO>, dim3(tiles, p.Hkv, p.B), dim3(kScoreThreads), 0, s, p, q,
                               (const uint16_t*)c->summ, c->scores, (const int32_t*)c->ntok_dev, sb, reps, out_ids,
                               out_scores);
    if (trace && sb.trace) {   // experiments only: synchronous dump of per-CTA phase times
        cudaStreamSynchronize(s);
        std::vector<unsigned long long> h((size_t)nctas * 4);
        cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull;
        for (int64_t i = 0; i < nctas; ++i) if (h[i * 4] && h[i * 4] < t0) t0 = h[i * 4];
        const char* names[4] = {"entry", "scored", "topk_begin", "topk_end"};
        for (int j = 0; j < 4; ++j) {
            std::vector<double> v;
            for (int64_t i = 0; i < nctas; ++i) if (h[i * 4 + j]) v.push_back((h[i * 4 + j] - t0) * 1e-3);
            if (v.empty()) continue;
            std::sort(v.begin(), v.end());
            fprintf(stderr, "sel trace V=%d %-10s n=%5zu min %7.2f p50 %7.2f p90 %7.2f max %7.2f us\n", V, names[j],
                    v.size(), v[0], v[v.size() / 2], v[v.size() * 9 / 10], v.back());
        }
        // top-k phases relative to topk_begin of the same CTA
        std::vector<unsigned long long> h2((size_t)nctas * 8);
        cudaMemcpy(h2.data(), tbuf + (1 << 18), h2.size() * 8, cudaMemcpyDeviceToHost);
        const char* pn[5] = {"loaded", "pass0", "pass1", "pass2", "scans"};
        for (int j = 0; j < 5; ++j) {
            std::vector<double> v;
            for (int64_t i = 0; i < nctas; ++i)
                if (h2[i * 8 + j] && h[i * 4 + 2]) v.push_back(((double)h2[i * 8 + j] - (double)h[i * 4 + 2]) * 1e-3);
            if (v.empty()) continue;
            std::sort(v.begin(), v.end());
            fprintf(stderr, "sel topk phase %-7s n=%5zu p50 %7.2f max %7.2f us (from topk_begin)\n", pn[j], v.size(),
                    v[v.size() / 2], v.back());
        }
    }
    return e;
}

template <int V>
static cudaError_t launch_sel_v(kvd_cache* c, const StepParams& p, const uint16_t* q, int32_t* out_ids,
                                float* out_scores, cudaStream_t s) {
    if (c->nb_pad <= kDirectTopkMax) {
        // direct selection over the segment's nb scores: KPT per thread, keys re-read per chunk
        const int64_t per = (c->nb_pad + kScoreThreads - 1) / kScoreThreads;
        if (per <= 4) return launch_sel<V, 4, false>(c, p, q, 1, out_ids, out_scores, s);
        if (per <= 8) return launch_sel<V, 8, false>(c, p, q, 1, out_ids, out_scores, s);
        if (per <= 16) return launch_sel<V, 16, false>(c, p, q, 1, out_ids, out_scores, s);
        return launch_sel<V, 32, false>(c, p, q, (int)((per + 31) / 32), out_ids, out_scores, s);
    }
    // two-level: final selection over at most tiles * k candidates
    const int64_t tiles = (c->nb_pad + kScoreThreads * V - 1) / (kScoreThreads * V);
    const int64_t cand = std::min<int64_t>(tiles * std::max(p.k, 1), c->nb_pad);
    const int64_t per = (cand + kScoreThreads - 1) / kScoreThreads;
    if (per <= 8) return launch_sel<V, 8, true>(c, p, q, 1, out_ids, out_scores, s);
    if (per <= 16) return launch_sel<V, 16, true>(c, p, q, 1, out_ids, out_scores, s);
    return launch_sel<V, 16, true>(c, p, q, (int)((per + 15) / 16), out_ids, out_scores, s);
}

cudaError_t launch_select(kvd_cache* c, const StepParams& p, const uint16_t* q, int32_t* out_ids, float* out_scores,
                          cudaStream_t s) {
    // V: largest of 8, 4, 2 blocks per thread that still gives >= 2 CTAs per SM; the
    // two-level path always takes V = 8 (fewest tiles -> fewest candidates)
    const int64_t segs = (int64_t)p.B * p.Hkv;
    auto ctas = [&](int V) { return segs * ((c->nb_pad + kScoreThreads * V - 1) / (kScoreThreads * V)); };
    cudaError_t e;
    if (c->nb_pad > kDirectTopkMax || ctas(8) >= 2 * 148) e = launch_sel_v<8>(c, p, q, out_ids, out_scores, s);
    else if (ctas(4) >= 2 * 148) e = launch_sel_v<4>(c, p, q, out_ids, out_scores, s);
    else e = launch_sel_v<2>(c, p, q, out_ids, out_scores, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace kvd
