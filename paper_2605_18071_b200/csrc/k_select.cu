// k_select.cu — rows (a1) summary scoring and (a2) top-k block selection.
//
// (a1) "identifying critical KV entries via the index": every
// block's score is the dot product of the KV head's group query with the
// block's mean-key summary, computed as one fp32 FMA chain
// over the 128 dims in order (DESIGN.md §3 R3, R5) so that ids are bit-exact.
// HBM-bound: 256 B of summary per block.  The summaries are dim-major, so a
// thread owning V consecutive blocks reads one V*2-byte vector per dim row and
// a warp reads 64*V contiguous bytes per row (coalesced).  No shared-memory
// staging: each thread keeps 8 rows of its blocks in flight (double-buffered
// registers) and runs V independent chains.  V in {2, 4, 8} is picked so the
// grid has >= 2 CTAs per SM.  Rows for the first batch are requested before
// griddepcontrol.wait (summaries are immutable during a step), overlapping
// the previous kernel's tail.
//
// (a2) "retrieving only the Top-K important chunks": one
// 1024-thread CTA per segment.  Thread t owns the contiguous blocks
// [t*KPT, (t+1)*KPT) (keys in registers when nb <= 16384).  A 3-pass radix
// select (11 + 11 + 10 bits, warp-aggregated shared histograms) finds the
// k-th largest monotone key T among the candidates; keys > T are taken and the
// kk lowest-id keys == T (R10).  Two block scans give tie ranks and output
// positions, so ids come out ascending with no sort.
#include "common.cuh"
#include "internal.h"

namespace kvd {

constexpr int kScoreThreads = 256;
constexpr int kScoreRows = 8;                 // dim rows in flight per thread

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
__global__ void __launch_bounds__(kScoreThreads) score_kernel(StepParams p, const uint16_t* __restrict__ q,
                                                              const uint16_t* __restrict__ summ,
                                                              float* __restrict__ scores,
                                                              const int32_t* __restrict__ ntok) {
    using Vec = typename VecOf<V>::T;
    __shared__ float qbar[kHeadDim];
    const int bi = blockIdx.z, h = blockIdx.y;
    const int r = p.req[bi];
    const int64_t cta0 = (int64_t)blockIdx.x * kScoreThreads * V;
    const int n = ntok[r];                        // written only by kvd_load_prefix (setup)
    const int64_t nb = (n + p.P - 1) / p.P;
    if (cta0 >= nb) return;                       // whole CTA past this request's end
    const int64_t b0 = cta0 + (int64_t)threadIdx.x * V;
    const bool ld = b0 < nb;                      // V-groups never straddle nb_pad (V | 128)
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    const Vec* base = reinterpret_cast<const Vec*>(summ + seg * kHeadDim * p.nb_pad + (ld ? b0 : 0));
    const int64_t rstride = p.nb_pad / V;         // Vec elements per dim row

    Vec buf[kScoreRows], cur[kScoreRows];
#pragma unroll
    for (int u = 0; u < kScoreRows; ++u)
        if (ld) buf[u] = __ldcs(base + u * rstride);
    griddep_wait();
    if (threadIdx.x < kHeadDim) {
        // group query: qbar[j] = ((+0 + q_0[j]) + q_1[j]) + ... (fp32, g ascending; R3)
        const uint16_t* qh = q + ((int64_t)bi * p.Hq + (int64_t)h * p.G) * kHeadDim;
        float a = 0.0f;
        for (int g = 0; g < p.G; ++g) a = __fadd_rn(a, bf16_bits(qh[g * kHeadDim + threadIdx.x]));
        qbar[threadIdx.x] = a;
    }
    __syncthreads();
    float acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.0f;
#pragma unroll 1
    for (int j0 = 0; j0 < kHeadDim; j0 += kScoreRows) {
#pragma unroll
        for (int u = 0; u < kScoreRows; ++u) cur[u] = buf[u];
        if (ld && j0 + kScoreRows < kHeadDim) {
#pragma unroll
            for (int u = 0; u < kScoreRows; ++u) buf[u] = __ldcs(base + (j0 + kScoreRows + u) * rstride);
        }
#pragma unroll
        for (int u = 0; u < kScoreRows; ++u) {
            const float qj = qbar[j0 + u];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const uint32_t w = VecOf<V>::word(cur[u], v >> 1);
                acc[v] = __fmaf_rn(qj, (v & 1) ? bf16_hi(w) : bf16_lo(w), acc[v]);   // sequential in j (R5)
            }
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

constexpr int kTopkThreads = 1024;

// KPT keys per thread per chunk; `reps` chunks per thread (reps > 1 re-reads
// the scores from L2 in every pass instead of keeping them in registers).
template <int KPT>
__global__ void __launch_bounds__(kTopkThreads, 1) topk_kernel(StepParams p, const float* __restrict__ scores,
                                                            const int32_t* __restrict__ ntok, int reps,
                                                            int32_t* __restrict__ out_ids,
                                                            float* __restrict__ out_scores) {
    __shared__ int hist[2048];
    __shared__ int scan_scratch[33];
    __shared__ uint32_t s_digit;
    __shared__ int s_above;
    const int bi = blockIdx.y, h = blockIdx.x;
    const int r = p.req[bi];
    const int tid = threadIdx.x;
    if (p.k == 0) return;
    const SegGeom g = seg_geom(ntok[r], p.P, p.sink_tokens, p.local_tokens);
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    const float* sc = scores + seg * p.nb_pad;
    griddep_wait();

    uint32_t key[KPT];
    uint32_t cm = 0;                         // candidate mask of the chunk in registers
    auto load = [&](int c) {
        const int64_t b0 = ((int64_t)tid * reps + c) * KPT;
        cm = 0;
        if (b0 >= g.nb) return;
        float f[KPT];
        if constexpr (KPT % 4 == 0) {
#pragma unroll
            for (int i = 0; i < KPT; i += 4) {
                const float4 x = __ldcg(reinterpret_cast<const float4*>(sc + b0 + i));
                f[i] = x.x; f[i + 1] = x.y; f[i + 2] = x.z; f[i + 3] = x.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < KPT; ++i) f[i] = __ldcg(sc + b0 + i);
        }
#pragma unroll
        for (int i = 0; i < KPT; ++i) {
            const int64_t b = b0 + i;
            const bool cand = b < g.nb && b >= g.sink_end && b < g.local_begin;
            key[i] = score_key32(f[i]);
            cm |= (uint32_t)cand << i;
        }
    };
    if (reps == 1) load(0);

    // ---- radix select over candidates: T = k-th largest key (3 passes)
    uint32_t prefix = 0, mask = 0;
    int kk = p.k;
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
        const int shift = pass == 0 ? 21 : pass == 1 ? 10 : 0;
        const int nbins = pass == 2 ? 1024 : 2048;
        for (int i = tid; i < nbins; i += kTopkThreads) hist[i] = 0;
        __syncthreads();
#pragma unroll 1
        for (int c = 0; c < reps; ++c) {
            if (reps > 1) load(c);
#pragma unroll
            for (int i = 0; i < KPT; ++i) {
                const bool act = ((cm >> i) & 1u) && (key[i] & mask) == prefix;
                warp_hist_add(hist, (key[i] >> shift) & (uint32_t)(nbins - 1), act);
            }
        }
        __syncthreads();
        // bins in descending order: thread t owns bins nbins-1-2t and nbins-2-2t (pass 2: one bin)
        int c0 = 0, c1 = 0;
        const int d0 = nbins == 2048 ? 2047 - 2 * tid : 1023 - tid;
        c0 = hist[d0];
        if (nbins == 2048) c1 = hist[d0 - 1];
        int tot;
        const int above = block_exclusive_scan(c0 + c1, scan_scratch, &tot);
        if (above < kk && kk <= above + c0 + c1) {
            if (above + c0 >= kk) {
                s_digit = (uint32_t)d0;
                s_above = above;
            } else {
                s_digit = (uint32_t)(d0 - 1);
                s_above = above + c0;
            }
        }
        __syncthreads();
        prefix |= s_digit << shift;
        mask |= (uint32_t)(nbins - 1) << shift;
        kk -= s_above;
        __syncthreads();
    }
    griddep_launch();
    const uint32_t T = prefix;               // take keys > T, and the kk lowest-id keys == T

    // ---- tie ranks and output positions (thread-contiguous ownership => ascending ids)
    int ngt = 0, neq = 0;
#pragma unroll 1
    for (int c = 0; c < reps; ++c) {
        if (reps > 1) load(c);
#pragma unroll
        for (int i = 0; i < KPT; ++i) {
            const bool cand = (cm >> i) & 1u;
            ngt += (cand && key[i] > T) ? 1 : 0;
            neq += (cand && key[i] == T) ? 1 : 0;
        }
    }
    int tot;
    const int tie0 = block_exclusive_scan(neq, scan_scratch, &tot);
    const int ntake = min(max(kk - tie0, 0), neq);
    const int pos0 = block_exclusive_scan(ngt + ntake, scan_scratch, &tot);
    int32_t* ids_out = out_ids + ((int64_t)bi * p.Hkv + h) * p.k;
    float* sc_out = out_scores ? out_scores + ((int64_t)bi * p.Hkv + h) * p.k : nullptr;
    int pos = pos0, tie = tie0;
#pragma unroll 1
    for (int c = 0; c < reps; ++c) {
        if (reps > 1) load(c);
        const int64_t b0 = ((int64_t)tid * reps + c) * KPT;
#pragma unroll
        for (int i = 0; i < KPT; ++i) {
            if (!((cm >> i) & 1u)) continue;
            bool take = key[i] > T;
            if (key[i] == T) take = tie++ < kk;
            if (take) {
                ids_out[pos] = (int32_t)(b0 + i);
                if (sc_out) sc_out[pos] = sc[b0 + i];
                ++pos;
            }
        }
    }
}

template <int V>
static cudaError_t launch_score(kvd_cache* c, const StepParams& p, const uint16_t* q, cudaStream_t s) {
    const unsigned tiles = (unsigned)((c->nb_pad + kScoreThreads * V - 1) / (kScoreThreads * V));
    return launch_pdl(score_kernel<V>, dim3(tiles, p.Hkv, p.B), dim3(kScoreThreads), 0, s, p, q,
                      (const uint16_t*)c->summ, c->scores, (const int32_t*)c->ntok_dev);
}

template <int KPT>
static cudaError_t launch_topk(kvd_cache* c, const StepParams& p, int reps, int32_t* out_ids, float* out_scores,
                               cudaStream_t s) {
    return launch_pdl(topk_kernel<KPT>, dim3(p.Hkv, p.B), dim3(kTopkThreads), 0, s, p, (const float*)c->scores,
                      (const int32_t*)c->ntok_dev, reps, out_ids, out_scores);
}

cudaError_t launch_select(kvd_cache* c, const StepParams& p, const uint16_t* q, int32_t* out_ids, float* out_scores,
                          cudaStream_t s) {
    // V: largest of 8, 4, 2 blocks per thread that still gives >= 2 CTAs per SM
    const int64_t segs = (int64_t)p.B * p.Hkv;
    auto ctas = [&](int V) { return segs * ((c->nb_pad + kScoreThreads * V - 1) / (kScoreThreads * V)); };
    cudaError_t e;
    if (ctas(8) >= 2 * 148) e = launch_score<8>(c, p, q, s);
    else if (ctas(4) >= 2 * 148) e = launch_score<4>(c, p, q, s);
    else e = launch_score<2>(c, p, q, s);
    if (e != cudaSuccess) return e;
    const int64_t per = (c->nb_pad + kTopkThreads - 1) / kTopkThreads;   // blocks per thread
    if (per <= 1) e = launch_topk<1>(c, p, 1, out_ids, out_scores, s);
    else if (per <= 2) e = launch_topk<2>(c, p, 1, out_ids, out_scores, s);
    else if (per <= 4) e = launch_topk<4>(c, p, 1, out_ids, out_scores, s);
    else if (per <= 8) e = launch_topk<8>(c, p, 1, out_ids, out_scores, s);
    else if (per <= 16) e = launch_topk<16>(c, p, 1, out_ids, out_scores, s);
    else e = launch_topk<16>(c, p, (int)((per + 15) / 16), out_ids, out_scores, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace kvd
