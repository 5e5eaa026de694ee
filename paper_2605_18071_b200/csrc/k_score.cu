// k_score.cu — row (a1) summary scoring as a pure streaming kernel.
//
// "identifying critical KV entries via the index": every block's score is the
// dot product of the KV head's group query with the block's mean-key summary,
// one fp32 FMA chain over the 128 dims in order (DESIGN.md §3 R3, R5) so that the ids the
// select kernel derives are bit-exact.  With Quest min/max summaries (R30) the
// chain is acc = acc + max(q_j mn_j, q_j mx_j), products rounded, sequential in j.
//
// HBM-bound: 256 B of summary per block (512 B for min/max), 1 flop per byte.  The summaries
// are dim-major, so a thread owning V consecutive blocks reads one V*2-byte vector per dim row
// and a warp reads 64*V contiguous bytes per row (coalesced).  No shared-memory staging: each
// thread keeps 2R rows of its blocks in flight (two ping-pong register batches) and runs V
// independent chains.  Small CTAs (256 threads) over the whole (tile, KV head, request) grid
// put every SM on the stream whatever the number of segments; rows of the first batch are
// requested before griddepcontrol.wait (summaries are immutable during a step), overlapping the
// previous kernel's tail.  Scores go to the cache's score array (4 B per 256 B read), where the
// select kernel ranks them from L2 and the lookahead policy reads them.
#include "common.cuh"
#include "internal.h"

namespace kvd {

constexpr int kScoreThreads = 256;

template <int V>
struct SVec;
template <>
struct SVec<2> {
    using T = uint32_t;
    static __device__ __forceinline__ uint32_t word(const T& x, int) { return x; }
};
template <>
struct SVec<4> {
    using T = uint2;
    static __device__ __forceinline__ uint32_t word(const T& x, int i) { return i ? x.y : x.x; }
};

// grid (tiles, Hkv, B); a CTA scores 256*V consecutive blocks (or centroids: p.sel_mode 1) of
// one segment.  mat: [seg][128][pitch] bf16 (pitch = p.nb_pad); mat2: the maxima (QUEST).
template <int V, int R, bool QUEST>
__global__ void __launch_bounds__(kScoreThreads, R * V > 32 ? 2 : 4)
    score_kernel(StepParams p, const uint16_t* __restrict__ q, const uint16_t* __restrict__ mat,
                 const uint16_t* __restrict__ mat2, float* __restrict__ scores, const int32_t* __restrict__ ntok) {
    using Vec = typename SVec<V>::T;
    __shared__ float qbar[kHeadDim];
    const int bi = blockIdx.z, h = p.h0 + blockIdx.y;
    const int r = p.req[bi];
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    // blocks (centroids) of the segment: token counts change only in kvd_load_prefix and
    // kvd_append_token, which complete before a dependent step kernel starts
    const int64_t nb = p.sel_mode == 1 ? (int64_t)p.sel_count[seg] : ((int64_t)ntok[r] + p.P - 1) / p.P;
    const int64_t t0 = (int64_t)blockIdx.x * kScoreThreads * V;
    if (t0 >= nb) {                               // whole CTA past this segment's end
        if (p.kt_slots && threadIdx.x == 0)
            kt_end(p.kt_slots, p.kt_acc, p.kt_base + kKtScore, kKtScore, (unsigned long long)gridDim.x * gridDim.y * gridDim.z);
        return;
    }
    const int64_t b0 = t0 + (int64_t)threadIdx.x * V;
    const bool ld = b0 < nb;                      // V-groups never straddle the pitch (V | 128)
    const int64_t pitch = p.nb_pad;
    const Vec* src = reinterpret_cast<const Vec*>(mat + seg * kHeadDim * pitch + (ld ? b0 : 0));
    const Vec* src2 = QUEST ? reinterpret_cast<const Vec*>(mat2 + seg * kHeadDim * pitch + (ld ? b0 : 0)) : nullptr;
    const int64_t rstride = pitch / V;            // Vec elements per dim row
    Vec bufA[R], bufB[R];
#pragma unroll
    for (int u = 0; u < R; ++u)
        if (ld) bufA[u] = __ldcs(src + u * rstride);
#pragma unroll
    for (int u = 0; u < R; ++u)
        if (ld) bufB[u] = QUEST ? __ldcs(src2 + u * rstride) : __ldcs(src + (R + u) * rstride);
    griddep_wait();                               // q may come from an earlier kernel of the step
    if (p.early_trigger) griddep_launch();
    if (threadIdx.x == 0) kt_begin(p.kt_slots, p.kt_base + kKtScore);
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
    if constexpr (QUEST) {
        // rows j0 .. j0+R-1 of the minima (bufA) and of the maxima (bufB), R rows per step
#pragma unroll 1
        for (int j0 = 0; j0 < kHeadDim; j0 += R) {
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const float qj = qbar[j0 + u];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const uint32_t wn = SVec<V>::word(bufA[u], v >> 1), wx = SVec<V>::word(bufB[u], v >> 1);
                    const float a = __fmul_rn(qj, (v & 1) ? bf16_hi(wn) : bf16_lo(wn));
                    const float b = __fmul_rn(qj, (v & 1) ? bf16_hi(wx) : bf16_lo(wx));
                    acc[v] = __fadd_rn(acc[v], fmaxf(a, b));   // sequential in j (R30)
                }
            }
            if (ld && j0 + R < kHeadDim) {
#pragma unroll
                for (int u = 0; u < R; ++u) {
                    bufA[u] = __ldcs(src + (j0 + R + u) * rstride);
                    bufB[u] = __ldcs(src2 + (j0 + R + u) * rstride);
                }
            }
        }
    } else {
        auto consume = [&](const Vec (&buf)[R], int j0) {
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const float qj = qbar[j0 + u];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const uint32_t w = SVec<V>::word(buf[u], v >> 1);
                    acc[v] = __fmaf_rn(qj, (v & 1) ? bf16_hi(w) : bf16_lo(w), acc[v]);   // sequential in j (R5)
                }
            }
        };
#pragma unroll 1
        for (int j0 = 0; j0 < kHeadDim; j0 += 2 * R) {
            consume(bufA, j0);
            if (ld && j0 + 2 * R < kHeadDim) {
#pragma unroll
                for (int u = 0; u < R; ++u) bufA[u] = __ldcs(src + (j0 + 2 * R + u) * rstride);
            }
            consume(bufB, j0 + R);
            if (ld && j0 + 3 * R < kHeadDim) {
#pragma unroll
                for (int u = 0; u < R; ++u) bufB[u] = __ldcs(src + (j0 + 3 * R + u) * rstride);
            }
        }
    }
    griddep_launch();                             // dependents still wait for this grid's completion
    if (ld) {
        float* out = scores + seg * pitch + b0;
        if (b0 + V <= nb) {
#pragma unroll
            for (int v = 0; v < V; v += 2) *reinterpret_cast<float2*>(out + v) = make_float2(acc[v], acc[v + 1]);
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v)
                if (b0 + v < nb) out[v] = acc[v];
        }
    }
    if (p.kt_slots) {
        __syncthreads();
        if (threadIdx.x == 0)
            kt_end(p.kt_slots, p.kt_acc, p.kt_base + kKtScore, kKtScore, (unsigned long long)gridDim.x * gridDim.y * gridDim.z);
    }
}

// Scores of every block (centroid) of the launch's segments into `scores` ([seg][p.nb_pad]).
cudaError_t launch_score(kvd_cache* c, const StepParams& p, const uint16_t* q, const uint16_t* mat,
                         const uint16_t* mat2, float* scores, cudaStream_t s) {
    constexpr int V = 2, R = 16;                 // 512 blocks per CTA, 32 rows (16 KiB) in flight per warp
    const unsigned tiles = (unsigned)((p.nb_pad + kScoreThreads * V - 1) / (kScoreThreads * V));
    const int32_t* ntok = c->ntok_dev + (int64_t)p.layer * c->R;
    cudaError_t e = p.sel_mode == 2
        ? launch_pdl(score_kernel<V, R / 2, true>, dim3(tiles, p.nh, p.B), dim3(kScoreThreads), 0, s, p, q, mat, mat2,
                     scores, ntok)
        : launch_pdl(score_kernel<V, R, false>, dim3(tiles, p.nh, p.B), dim3(kScoreThreads), 0, s, p, q, mat, mat2,
                     scores, ntok);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace kvd
