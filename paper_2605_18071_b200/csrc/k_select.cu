// k_select.cu — rows (a1) summary scoring and (a2) top-k block selection.
//
// (a1) "identifying critical KV entries via the index": every
// block's score is the dot product of the KV head's group query with the
// block's mean-key summary, computed as one fp32 FMA chain
// over the 128 dims in order (DESIGN.md §3 R3, R5) so that ids are bit-exact.
// HBM-bound: 256 B of summary per block.  The summaries are dim-major, so a
// CTA tile = 128 rows x kScoreCols blocks, staged into shared memory with bulk
// async copies (TMA engine) in 4 chunks of 32 rows, each on its own mbarrier,
// while one thread per block runs the chain.
//
// (a2) "retrieving only the Top-K important chunks": per
// segment, a 4-pass 8-bit radix select on the monotone 32-bit score key finds
// the k-th largest key T; keys > T are taken and ties at T go to the lowest
// block ids (R10).  Selected ids are emitted ascending via a bitmap scan.
#include "common.cuh"
#include "internal.h"

namespace kvd {

constexpr int kScoreChunks = 4;
constexpr int kScoreRowsPerChunk = kHeadDim / kScoreChunks;   // 32

__global__ void __launch_bounds__(kScoreCols) score_kernel(StepParams p, const uint16_t* __restrict__ q,
                                                           const uint16_t* __restrict__ summ,
                                                           float* __restrict__ scores,
                                                           const int32_t* __restrict__ ntok) {
    __shared__ __align__(128) uint16_t tile[kHeadDim][kScoreCols];
    __shared__ float qbar[kHeadDim];
    __shared__ __align__(8) uint64_t bar[kScoreChunks];
    const int bi = blockIdx.z, h = blockIdx.y;
    const int r = p.req[bi];
    const int64_t col0 = (int64_t)blockIdx.x * kScoreCols;
    const int n = ntok[r];
    const int64_t nb = (n + p.P - 1) / p.P;
    if (col0 >= nb) return;                                   // whole tile past this request's end
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    const uint16_t* rows = summ + seg * kHeadDim * p.nb_pad + col0;
    const int tid = threadIdx.x;

    if (tid < 32) {
        if (tid == 0) {
            for (int c = 0; c < kScoreChunks; ++c) mbar_init(&bar[c], 1);
            fence_mbar_init();
        }
        __syncwarp();
        const uint32_t row_bytes = kScoreCols * 2;
        for (int c = 0; c < kScoreChunks; ++c) {
            if (tid == 0) mbar_arrive_expect_tx(&bar[c], row_bytes * kScoreRowsPerChunk);
            __syncwarp();
            const int j = c * kScoreRowsPerChunk + tid;
            bulk_g2s(&tile[j][0], rows + (int64_t)j * p.nb_pad, row_bytes, &bar[c]);
        }
    }
    // group query: qbar[j] = ((+0 + q_0[j]) + q_1[j]) + ... (fp32, g ascending; R3)
    {
        const uint16_t* qh = q + ((int64_t)bi * p.Hq + (int64_t)h * p.G) * kHeadDim;
        float a = 0.0f;
        for (int g = 0; g < p.G; ++g) a = __fadd_rn(a, bf16_bits(qh[g * kHeadDim + tid]));
        qbar[tid] = a;
    }
    __syncthreads();

    float acc = 0.0f;
#pragma unroll
    for (int c = 0; c < kScoreChunks; ++c) {
        mbar_wait(&bar[c], 0);
#pragma unroll 8
        for (int jj = 0; jj < kScoreRowsPerChunk; ++jj) {
            const int j = c * kScoreRowsPerChunk + jj;
            acc = __fmaf_rn(qbar[j], bf16_bits(tile[j][tid]), acc);
        }
    }
    const int64_t b = col0 + tid;
    if (b < nb) scores[seg * p.nb_pad + b] = acc;
}

constexpr int kTopkThreads = 512;

// One CTA per segment.  Shared memory: hist[256] + 2 bitmaps of nb_pad bits.
__global__ void __launch_bounds__(kTopkThreads) topk_kernel(StepParams p, const float* __restrict__ scores,
                                                            const int32_t* __restrict__ ntok,
                                                            int32_t* __restrict__ out_ids,
                                                            float* __restrict__ out_scores) {
    extern __shared__ uint32_t sm[];
    __shared__ int hist[256];
    __shared__ int scan_scratch[33];
    __shared__ uint32_t s_digit;
    __shared__ int s_above;
    const int bi = blockIdx.y, h = blockIdx.x;
    const int r = p.req[bi];
    const SegGeom g = seg_geom(ntok[r], p.P, p.sink_tokens, p.local_tokens);
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    const float* sc = scores + seg * p.nb_pad;
    const int nwords = (g.nb + 31) >> 5;
    uint32_t* selw = sm;                 // [nwords]
    uint32_t* eqw = sm + nwords;         // [nwords]
    const int tid = threadIdx.x;
    int32_t* ids_out = out_ids + ((int64_t)bi * p.Hkv + h) * p.k;
    if (p.k == 0) return;

    // ---- radix select: T = k-th largest key among candidates
    uint32_t prefix = 0, mask = 0;
    int kk = p.k;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int b = tid; b < g.nb; b += blockDim.x) {
            if (b < g.sink_end || b >= g.local_begin) continue;
            const uint32_t key = score_key32(sc[b]);
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
        }
        __syncthreads();
        if (tid < 32) {
            // lane L owns digits 255-8L .. 248-8L (descending)
            int cnt[8], tot = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                cnt[i] = hist[255 - 8 * tid - i];
                tot += cnt[i];
            }
            int incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += y;
            }
            int above = incl - tot;     // keys with a higher digit than this lane's first digit
            bool mine = above < kk && kk <= incl;
            if (mine) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (above + cnt[i] >= kk) {
                        s_digit = (uint32_t)(255 - 8 * tid - i);
                        s_above = above;
                        break;
                    }
                    above += cnt[i];
                }
            }
        }
        __syncthreads();
        prefix |= s_digit << shift;
        mask |= 0xFFu << shift;
        kk -= s_above;
        __syncthreads();
    }
    const uint32_t T = prefix;          // kk = number of keys == T to take (lowest ids)

    // ---- bitmaps: sel = key > T, eq = key == T (candidates only)
    for (int w = tid; w < nwords; w += blockDim.x) {
        uint32_t s = 0, e = 0;
        for (int i = 0; i < 32; ++i) {
            const int b = w * 32 + i;
            if (b >= g.nb || b < g.sink_end || b >= g.local_begin) continue;
            const uint32_t key = score_key32(sc[b]);
            s |= (uint32_t)(key > T) << i;
            e |= (uint32_t)(key == T) << i;
        }
        selw[w] = s;
        eqw[w] = e;
    }
    __syncthreads();
    // ---- ties: the kk lowest ids with key == T.  Threads own contiguous word ranges.
    const int wpt = (nwords + blockDim.x - 1) / blockDim.x;
    const int w0 = tid * wpt, w1 = min(nwords, w0 + wpt);
    {
        int local = 0;
        for (int w = w0; w < w1; ++w) local += __popc(eqw[w]);
        int total;
        int base = block_exclusive_scan(local, scan_scratch, &total);
        for (int w = w0; w < w1; ++w) {
            uint32_t e = eqw[w];
            while (e) {
                const int bit = __ffs(e) - 1;
                if (base < kk) selw[w] |= 1u << bit;
                ++base;
                e &= e - 1;
            }
        }
    }
    __syncthreads();
    // ---- emit ascending ids
    {
        int local = 0;
        for (int w = w0; w < w1; ++w) local += __popc(selw[w]);
        int total;
        int base = block_exclusive_scan(local, scan_scratch, &total);
        for (int w = w0; w < w1; ++w) {
            uint32_t s = selw[w];
            while (s) {
                const int bit = __ffs(s) - 1;
                const int b = w * 32 + bit;
                if (base < p.k) {
                    ids_out[base] = b;
                    if (out_scores) out_scores[((int64_t)bi * p.Hkv + h) * p.k + base] = sc[b];
                }
                ++base;
                s &= s - 1;
            }
        }
    }
}

cudaError_t launch_select(kvd_cache* c, const StepParams& p, const uint16_t* q, int32_t* out_ids, float* out_scores,
                          cudaStream_t s) {
    dim3 sg((unsigned)(c->nb_pad / kScoreCols), p.Hkv, p.B);
    score_kernel<<<sg, kScoreCols, 0, s>>>(p, q, c->summ, c->scores, c->ntok_dev);
    const size_t smem = 2 * sizeof(uint32_t) * (size_t)((c->nb_pad + 31) / 32);
    topk_kernel<<<dim3(p.Hkv, p.B), kTopkThreads, smem, s>>>(p, c->scores, c->ntok_dev, out_ids, out_scores);
    return cudaGetLastError();
}

}  // namespace kvd
