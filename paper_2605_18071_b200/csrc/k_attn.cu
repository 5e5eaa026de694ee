// k_attn.cu — rows (a5) split-K sparse decode attention and (a6) LSE merge.
//
// "executing attention ... over the union of the newly fetched and resident KV
// entries".  Per (request, KV head, split) one CTA of 4 warps.
// The attention list (selected + pinned blocks, from resolve) is cut into
// 16-token tiles (E = 16/P list entries, 8 KiB); each warp streams its tiles
// from the slot pool into a private 3-stage shared-memory ring with bulk async
// copies (TMA engine) completing on mbarriers, then runs the two contractions
// on tensor cores (mma.sync m16n8k16 bf16 -> fp32, swap-AB so the 16 tokens
// fill M and the G <= 8 query heads of the KV head fill N):
//     S^T[16 tok][8 h] = K[16][128] . Q^T            (8 MMAs)
//     O^T[128][8 h]   += V^T[128][16] . (P_hi + P_lo)^T  (16 MMAs)
// P is split into bf16 hi + lo parts so P.V keeps ~16 mantissa bits (a single
// bf16 P misses the 2e-3 bar, SURVEY §7 hard part 4).  The S^T accumulator is
// turned into the P^T B-fragment with movmatrix.trans.  Online softmax in the
// log2 domain (exp2), warp-shuffle max/sum.  Warps merge through shared
// memory; splits merge (a6) in the last-arriving CTA of the segment:
//     m = max_s m_s;  l = sum_s l_s 2^(m_s-m);  o = sum_s 2^(m_s-m) o~_s / l;
//     lse = (m + log2 l) ln 2.
// HBM-bound: 8 KiB per 16-token tile; 4*G flop per 4 B of K/V.
#include "common.cuh"
#include "internal.h"

namespace kvd {

struct AttnBufs {
    const uint8_t* slots;
    const int32_t* ntok;
    const uint8_t* zero_rec;
    float* part_o;      // [R][Hkv][max_splits][8][128]
    float* part_ml;     // [R][Hkv][max_splits][8][2]
    uint32_t* ctr;      // [R][Hkv]
    int32_t max_splits;
};

constexpr int kAttnThreads = kAttnWarps * 32;
constexpr size_t kAttnSmem = (size_t)kAttnWarps * kAttnStages * kTileBytes;

__global__ void __launch_bounds__(kAttnThreads) attn_kernel(StepParams p, AttnBufs ab, const uint16_t* __restrict__ q,
                                                            const int32_t* __restrict__ attn,
                                                            float* __restrict__ out, float* __restrict__ out_lse) {
    extern __shared__ __align__(1024) uint8_t stage[];
    __shared__ __align__(8) uint64_t bar[kAttnWarps][kAttnStages];
    __shared__ float red_m[kAttnWarps][8], red_l[kAttnWarps][8];
    __shared__ int s_last;
    __shared__ int2 s_list[kSplitTiles * 16];          // (block, slot) of the split's entries
    const int split = blockIdx.x, h = blockIdx.y, bi = blockIdx.z;
    const int r = p.req[bi];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const SegGeom g = seg_geom(ab.ntok[r], p.P, p.sink_tokens, p.local_tokens);
    const int pr = g.sink_end + (g.nb - g.local_begin);
    const int nvalid = min(p.W, p.k + pr);
    const int ntiles = (nvalid + p.E - 1) / p.E;
    const int t0 = split * kSplitTiles;
    const int t1 = min(ntiles, t0 + kSplitTiles);
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    const int64_t rs = (int64_t)r * p.Hkv + h;
    const int32_t* lst = attn + ((int64_t)bi * p.Hkv + h) * (int64_t)p.W * 2;
    const uint8_t* seg_slots = ab.slots + seg * p.C * (int64_t)p.rec_bytes;
    const int rec = p.rec_bytes;

    // this warp's tiles: t0 + warp + 4 i
    const int nt_w = (t1 - t0 - warp + kAttnWarps - 1) / kAttnWarps > 0 ? (t1 - t0 - warp + kAttnWarps - 1) / kAttnWarps : 0;
    uint8_t* my_stage = stage + (size_t)warp * kAttnStages * kTileBytes;
    uint64_t* my_bar = bar[warp];
    if (lane == 0) {
        for (int s = 0; s < kAttnStages; ++s) mbar_init(&my_bar[s], 1);
        fence_mbar_init();
    }
    const uint64_t pol = l2_evict_first_policy();
    // everything below reads what resolve / gather (the previous kernels) wrote
    griddep_wait();
    // the split's (block, slot) entries -> shared memory, so issuing a tile's copy
    // never waits on a dependent global load
    const int e0 = t0 * p.E, ne = max(0, min(nvalid, t1 * p.E) - e0);
    for (int i = tid; i < ne; i += kAttnThreads) s_list[i] = reinterpret_cast<const int2*>(lst)[e0 + i];
    __syncthreads();
    auto issue = [&](int i) {
        if (lane == 0) {
            const int t = t0 + warp + kAttnWarps * i;
            uint64_t* b = &my_bar[i % kAttnStages];
            uint8_t* dst = my_stage + (size_t)(i % kAttnStages) * kTileBytes;
            mbar_arrive_expect_tx(b, (uint32_t)(p.E * rec));
            for (int e = 0; e < p.E; ++e) {
                const int idx = t * p.E + e;
                const uint8_t* src = ab.zero_rec;
                if (idx < nvalid) {
                    const int32_t slot = s_list[idx - e0].y;
                    if (slot >= 0) src = seg_slots + (int64_t)slot * rec;
                }
                bulk_g2s_hint(dst + e * rec, src, (uint32_t)rec, b, pol);
            }
        }
    };
    for (int i = 0; i < kAttnStages && i < nt_w; ++i) issue(i);

    // Q^T B-fragments: head = lane/4 (< G), dims 16 kk + 2 (lane%4) + {0,1} and +8
    uint32_t qf[8][2];
    {
        const int hd = lane >> 2;
        const uint16_t* qh = q + ((int64_t)bi * p.Hq + (int64_t)h * p.G + hd) * kHeadDim + 2 * (lane & 3);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            qf[kk][0] = hd < p.G ? *reinterpret_cast<const uint32_t*>(qh + 16 * kk) : 0u;
            qf[kk][1] = hd < p.G ? *reinterpret_cast<const uint32_t*>(qh + 16 * kk + 8) : 0u;
        }
    }
    // per-lane ldmatrix row offsets.  K (non-trans): matrix i = lane/8 -> row (lane&7) + 8 (i&1),
    // chunk 2kk + (i>>1).  V (trans): row (lane&7) + 8 (i>>1), chunk 2mt + (i&1).
    const int mi = lane >> 3;
    const int rk = (lane & 7) + 8 * (mi & 1), rv = (lane & 7) + 8 * (mi >> 1);
    const uint32_t koff = (uint32_t)((rk / p.P) * rec + (rk % p.P) * kRowBytes);
    const uint32_t kswz = (uint32_t)((rk % p.P) & 7);
    const uint32_t voff = (uint32_t)((rv / p.P) * rec + p.P * kRowBytes + (rv % p.P) * kRowBytes);
    const uint32_t vswz = (uint32_t)((rv % p.P) & 7);
    const int kchunk_hi = mi >> 1, vchunk_hi = mi & 1;
    // the two token rows this thread's accumulators hold
    const int row_lo = lane >> 2, row_hi = row_lo + 8;

    float oacc[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;   // heads h0 = 2 (lane%4), h1 = h0 + 1

    for (int i = 0; i < nt_w; ++i) {
        const int t = t0 + warp + kAttnWarps * i;
        // token validity of this thread's two rows
        bool vlo, vhi;
        {
            const int e_lo = row_lo / p.P, e_hi = row_hi / p.P;
            const int idx_lo = t * p.E + e_lo, idx_hi = t * p.E + e_hi;
            vlo = idx_lo < nvalid && (int64_t)p.P * s_list[idx_lo - e0].x + (row_lo % p.P) < g.n;
            vhi = idx_hi < nvalid && (int64_t)p.P * s_list[idx_hi - e0].x + (row_hi % p.P) < g.n;
        }
        mbar_wait(&my_bar[i % kAttnStages], (uint32_t)((i / kAttnStages) & 1));
        const uint32_t sbase = smem_u32(my_stage + (size_t)(i % kAttnStages) * kTileBytes);

        float sacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            uint32_t a0, a1, a2, a3;
            const uint32_t c = (uint32_t)(2 * kk + kchunk_hi);
            ldsm_x4(sbase + koff + ((c ^ kswz) << 4), a0, a1, a2, a3);
            mma_bf16_16816(sacc, a0, a1, a2, a3, qf[kk][0], qf[kk][1]);
        }
        // online softmax (log2 domain)
        const float x0 = vlo ? sacc[0] * p.scale_log2 : -INFINITY;   // row_lo, h0
        const float x1 = vlo ? sacc[1] * p.scale_log2 : -INFINITY;   // row_lo, h1
        const float x2 = vhi ? sacc[2] * p.scale_log2 : -INFINITY;   // row_hi, h0
        const float x3 = vhi ? sacc[3] * p.scale_log2 : -INFINITY;   // row_hi, h1
        float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
        }
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float ms0 = mn0 == -INFINITY ? 0.f : mn0, ms1 = mn1 == -INFINITY ? 0.f : mn1;
        const float al0 = fast_exp2(m0 - ms0), al1 = fast_exp2(m1 - ms1);
        const float p0 = fast_exp2(x0 - ms0), p1 = fast_exp2(x1 - ms1);
        const float p2 = fast_exp2(x2 - ms0), p3 = fast_exp2(x3 - ms1);
        m0 = mn0;
        m1 = mn1;
        l0 = l0 * al0 + (p0 + p2);
        l1 = l1 * al1 + (p1 + p3);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            oacc[mt][0] *= al0;
            oacc[mt][1] *= al1;
            oacc[mt][2] *= al0;
            oacc[mt][3] *= al1;
        }
        // P^T B-fragments (hi and lo bf16 parts) via movmatrix.trans
        const uint32_t hlo = pack_bf16x2(p0, p1), hhi = pack_bf16x2(p2, p3);
        const uint32_t llo = pack_bf16x2(p0 - bf16_lo(hlo), p1 - bf16_hi(hlo));
        const uint32_t lhi = pack_bf16x2(p2 - bf16_lo(hhi), p3 - bf16_hi(hhi));
        const uint32_t bh0 = movmatrix_t(hlo), bh1 = movmatrix_t(hhi);
        const uint32_t bl0 = movmatrix_t(llo), bl1 = movmatrix_t(lhi);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            uint32_t a0, a1, a2, a3;
            const uint32_t c = (uint32_t)(2 * mt + vchunk_hi);
            ldsm_x4_t(sbase + voff + ((c ^ vswz) << 4), a0, a1, a2, a3);
            mma_bf16_16816(oacc[mt], a0, a1, a2, a3, bh0, bh1);
            mma_bf16_16816(oacc[mt], a0, a1, a2, a3, bl0, bl1);
        }
        __syncwarp();
        if (i + kAttnStages < nt_w) {
            fence_proxy_async();
            issue(i + kAttnStages);
        }
    }
    griddep_launch();
    // full row sums per head
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    }
    // ---- merge the 4 warps through shared memory (reuse the stage ring)
    __syncthreads();
    float* red_o = reinterpret_cast<float*>(stage);   // [warp][8 heads][128 dims]
    {
        const int h0 = 2 * (lane & 3), h1 = h0 + 1, d = lane >> 2;
        float* ro = red_o + (size_t)warp * 8 * kHeadDim;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
            ro[h0 * kHeadDim + 16 * mt + d] = oacc[mt][0];
            ro[h1 * kHeadDim + 16 * mt + d] = oacc[mt][1];
            ro[h0 * kHeadDim + 16 * mt + 8 + d] = oacc[mt][2];
            ro[h1 * kHeadDim + 16 * mt + 8 + d] = oacc[mt][3];
        }
        if (lane < 4) {
            red_m[warp][h0] = m0;
            red_m[warp][h1] = m1;
            red_l[warp][h0] = l0;
            red_l[warp][h1] = l1;
        }
    }
    __syncthreads();
    const int dim = tid;   // kAttnThreads == 128 == head_dim
    const float kLn2 = 0.69314718055994531f;
    if (p.nsplit == 1) {
        for (int hh = 0; hh < p.G; ++hh) {
            float M = -INFINITY;
            for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, red_m[w][hh]);
            float o = 0.f, l = 0.f;
            if (M != -INFINITY) {
                for (int w = 0; w < kAttnWarps; ++w) {
                    const float sc = fast_exp2(red_m[w][hh] - M);
                    o += sc * red_o[((size_t)w * 8 + hh) * kHeadDim + dim];
                    l += sc * red_l[w][hh];
                }
            }
            const int64_t oh = (int64_t)bi * p.Hq + (int64_t)h * p.G + hh;
            out[oh * kHeadDim + dim] = l > 0.f ? o / l : 0.f;
            if (out_lse && dim == 0) out_lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : -INFINITY;
        }
        return;
    }
    float* po = ab.part_o + ((rs * ab.max_splits + split) * 8) * (int64_t)kHeadDim;
    float* pml = ab.part_ml + ((rs * ab.max_splits + split) * 8) * 2;
    for (int hh = 0; hh < p.G; ++hh) {
        float M = -INFINITY;
        for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, red_m[w][hh]);
        float o = 0.f, l = 0.f;
        if (M != -INFINITY) {
            for (int w = 0; w < kAttnWarps; ++w) {
                const float sc = fast_exp2(red_m[w][hh] - M);
                o += sc * red_o[((size_t)w * 8 + hh) * kHeadDim + dim];
                l += sc * red_l[w][hh];
            }
        }
        po[hh * kHeadDim + dim] = o;
        if (dim == 0) {
            pml[hh * 2] = M;
            pml[hh * 2 + 1] = l;
        }
    }
    // ---- (a6) split merge in the last-arriving CTA of this segment.  The barrier
    // orders the CTA's partial writes before thread 0's gpu-scope fence (fence
    // cumulativity), so one fence per CTA suffices.
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        s_last = (atomicAdd(&ab.ctr[rs], 1u) == (uint32_t)(p.nsplit - 1));
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) return;
    const float* po0 = ab.part_o + (rs * ab.max_splits * 8) * (int64_t)kHeadDim;
    const float* pml0 = ab.part_ml + (rs * ab.max_splits * 8) * 2;
    for (int hh = 0; hh < p.G; ++hh) {
        float M = -INFINITY;
        for (int s = 0; s < p.nsplit; ++s) M = fmaxf(M, __ldcg(&pml0[(s * 8 + hh) * 2]));
        float o = 0.f, l = 0.f;
        if (M != -INFINITY) {
            for (int s = 0; s < p.nsplit; ++s) {
                const float ms = __ldcg(&pml0[(s * 8 + hh) * 2]);
                const float sc = fast_exp2(ms - M);
                o += sc * __ldcg(&po0[(s * 8 + hh) * kHeadDim + dim]);
                l += sc * __ldcg(&pml0[(s * 8 + hh) * 2 + 1]);
            }
        }
        const int64_t oh = (int64_t)bi * p.Hq + (int64_t)h * p.G + hh;
        out[oh * kHeadDim + dim] = l > 0.f ? o / l : 0.f;
        if (out_lse && dim == 0) out_lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : -INFINITY;
    }
    if (tid == 0) ab.ctr[rs] = 0u;
}

cudaError_t launch_attention(kvd_cache* c, const StepParams& p, const uint16_t* q, const int32_t* attn, float* out,
                             float* out_lse, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAttnSmem);
        attr_set = true;
    }
    AttnBufs ab{c->slots, c->ntok_dev, c->zero_rec, c->part_o, c->part_ml, c->split_ctr, c->max_splits};
    cudaError_t e = launch_pdl(attn_kernel, dim3(p.nsplit, p.Hkv, p.B), dim3(kAttnThreads), kAttnSmem, s, p, ab, q,
                               attn, out, out_lse);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace kvd
