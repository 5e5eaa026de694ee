// k_attn.cu — rows (a5) split-K sparse decode attention and (a6) LSE merge.
//
// "executing attention ... over the union of the newly fetched and resident KV
// entries".  The attention lists from resolve (selected +
// pinned blocks, ascending) are cut into 16-token tiles (E = 16/P list
// entries, 8 KiB).  The call's S = B*Hkv segments give T = S*TS tiles (TS =
// ceil(W/E) per segment, uniform; entries past a segment's valid length read a
// zero record and are masked).  The tile sequence is split evenly over NW warp
// workers (stream-K: worker w owns tiles [w*T/NW, (w+1)*T/NW)), so every SM
// streams the same number of tiles whatever B, Hkv and k are; a worker whose
// range crosses a segment boundary produces one partial per segment piece.
//
// Per worker (one warp; 8 per SM by default): a private STAGES-deep ring of 8 KiB tiles in shared
// memory fed by bulk async copies (TMA engine) completing on mbarriers; the
// (block, slot) entries are staged through shared memory 128 at a time so a
// copy is never issued behind a dependent global load.  Per tile, on tensor
// cores (mma.sync m16n8k16 bf16 -> fp32, swap-AB: 16 tokens fill M, heads N):
//     S^T[16 tok][8] = K[16][128] . Q^T                   (8 MMAs)
//     O^T[128][8]   += V^T[128][16] . P^T                  (8 or 16 MMAs)
// P^T holds P = P_hi + P_lo (two bf16 parts; a single bf16 P misses the 2e-3
// bar, R26).  For G <= 4 both parts share one MMA: columns 0-3 carry
// P_hi of heads 0-3 and columns 4-7 P_lo of the same heads (Q^T columns 4-7
// duplicate heads 0-3, so those lanes see identical softmax statistics); the
// two output columns are summed in the epilogue.  For 4 < G <= 8 the hi and lo
// parts take two MMAs.  The S^T accumulator becomes the P^T B-fragment with
// movmatrix.trans.  Online softmax in the log2 domain (exp2).
//
// (a6) A segment handled by one worker is finalised in place; otherwise each
// piece writes its unnormalised partial (o~_j, m_j, l_j) and merge_kernel,
// launched behind attn_kernel (PDL, so no fences or arrival counters on the
// streaming path), combines them with one warp per query head:
//     m = max_j m_j;  l = sum_j l_j 2^(m_j-m);  o = sum_j 2^(m_j-m) o~_j / l;
//     lse = (m + log2 l) ln 2.
// HBM-bound: 8 KiB per 16-token tile; 4*G flop per 4 B of K/V.
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>
#include <cstdio>

#include "common.cuh"
#include "internal.h"

namespace kvd {

struct AttnBufs {
    const uint8_t* slots;
    const int32_t* ntok;
    const uint8_t* zero_rec;
    float* part_o;      // [R][Hkv][kMaxPieces][8][128]
    float* part_ml;     // [R][Hkv][kMaxPieces][8][2]
};

constexpr int kEntChunk = 128;                      // list entries staged per chunk (>= STAGES * 16)

struct Work {
    int32_t T;          // total tiles of the call (< 2^31: B <= 256, Hkv * TS small)
    int32_t TS;         // tiles per segment
    int32_t NW;         // workers
    int32_t xflags;     // timing experiments only (KVD_ATTN_X): 1 = skip S MMAs, 2 = skip P.V MMAs
    unsigned long long* trace;   // KVD_ATTN_TRACE: per-warp globaltimer stamps [NW][8] (experiments only)
};

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define ATTN_STAMP(i)                                                         \
    do {                                                                      \
        if (wk.trace && lane == 0 && w < wk.NW) wk.trace[(int64_t)w * 8 + (i)] = gtime(); \
    } while (0)

__device__ __forceinline__ int tile_begin(int w, const Work& wk) { return (int)((int64_t)w * wk.T / wk.NW); }
__device__ __forceinline__ int worker_of(int t, const Work& wk) {
    return (int)(((int64_t)(t + 1) * wk.NW - 1) / wk.T);
}

template <int STAGES, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) attn_kernel(StepParams p, AttnBufs ab, Work wk,
                                                               const uint16_t* __restrict__ q,
                                                               const int32_t* __restrict__ attn,
                                                               float* __restrict__ out, float* __restrict__ out_lse) {
    extern __shared__ __align__(1024) uint8_t stage[];
    __shared__ __align__(8) uint64_t bar[WARPS][STAGES];
    __shared__ int2 s_ent[WARPS][2][kEntChunk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int w = blockIdx.x * WARPS + warp;
    uint8_t* my_stage = stage + (size_t)warp * STAGES * kTileBytes;
    uint64_t* my_bar = bar[warp];
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&my_bar[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int ta = w < wk.NW ? tile_begin(w, wk) : 0, tb = w < wk.NW ? tile_begin(w + 1, wk) : 0;
    const int nt = tb - ta;
    const int s_first = ta / wk.TS, i_first = ta - s_first * wk.TS;   // segment / tile-in-segment of tile ta
    // P, E = 16/P and CT = kEntChunk/E >= STAGES (tiles per entry chunk) are powers of two: shifts, no divisions
    const int logP = __ffs(p.P) - 1, logE = 4 - logP, logCT = 7 - logE;
    const int E = 1 << logE, rec = p.rec_bytes, CT = 1 << logCT;
    const uint64_t pol = l2_evict_first_policy();
    const bool packed = p.G <= 4;
    ATTN_STAMP(0);
    griddep_wait();                                // lists / slots / q come from earlier kernels
    ATTN_STAMP(1);
    if (nt <= 0) return;

    // stage entry chunk c (tiles ta + c*CT ..) into buffer c & 1: (block, slot), or (-1, -1).
    // resolve pads each list past its valid length with (-1, -1); entries j >= W are tile padding.
    auto load_chunk = [&](int c) {
        for (int i = lane; i < kEntChunk; i += 32) {
            const int k = (c << logCT) + (i >> logE);   // worker-relative tile
            int2 v = make_int2(-1, -1);
            if (k < nt) {
                const int x = i_first + k;              // tile-in-segment relative to s_first
                const int ds = x / wk.TS;
                const int j = ((x - ds * wk.TS) << logE) + (i & (E - 1));
                if (j < p.W) v = reinterpret_cast<const int2*>(attn)[(int64_t)(s_first + ds) * p.W + j];
            }
            s_ent[warp][c & 1][i] = v;
        }
        __syncwarp();
    };
    // issue side: tile ik goes to stage ist; its segment's slot base is tracked incrementally
    int ik = 0, ist = 0, is_seg = s_first - 1, is_left = 0;
    const uint8_t* is_slots = nullptr;
    auto issue = [&]() {
        if (is_left == 0) {
            ++is_seg;
            is_left = is_seg == s_first ? wk.TS - i_first : wk.TS;
            const int bi = is_seg / p.Hkv, h = is_seg - bi * p.Hkv;
            is_slots = ab.slots + (((int64_t)p.layer * p.R + p.req[bi]) * p.Hkv + h) * p.C * (int64_t)rec;
        }
        if (lane == 0) {
            uint64_t* b = &my_bar[ist];
            uint8_t* dst = my_stage + (size_t)ist * kTileBytes;
            mbar_arrive_expect_tx(b, (uint32_t)(E * rec));
            const int2* ent = &s_ent[warp][(ik >> logCT) & 1][(ik & (CT - 1)) << logE];
            for (int e = 0; e < E; ++e) {
                const int32_t slot = ent[e].y;
                const uint8_t* src = slot >= 0 ? is_slots + (int64_t)slot * rec : ab.zero_rec;
                bulk_g2s_hint(dst + e * rec, src, (uint32_t)rec, b, pol);
            }
        }
        --is_left;
        ++ik;
        ist = ist + 1 == STAGES ? 0 : ist + 1;
    };
    load_chunk(0);
    while (ik < STAGES && ik < nt) issue();

    // per-lane ldmatrix row offsets.  K (non-trans): matrix i = lane/8 -> row (lane&7) + 8 (i&1),
    // chunk 2kk + (i>>1).  V (trans): row (lane&7) + 8 (i>>1), chunk 2mt + (i&1).
    const int mi = lane >> 3;
    const int rk = (lane & 7) + 8 * (mi & 1), rv = (lane & 7) + 8 * (mi >> 1);
    const int pm = p.P - 1;
    const uint32_t koff = (uint32_t)((rk >> logP) * rec + (rk & pm) * kRowBytes);
    const uint32_t kswz = (uint32_t)((rk & pm) & 7);
    const uint32_t voff = (uint32_t)((rv >> logP) * rec + p.P * kRowBytes + (rv & pm) * kRowBytes);
    const uint32_t vswz = (uint32_t)((rv & pm) & 7);
    const int kchunk_hi = mi >> 1, vchunk_hi = mi & 1;
    const int row_lo = lane >> 2, row_hi = row_lo + 8;     // token rows of this lane's accumulators
    const int quad = lane & 3;                              // accumulator columns 2 quad, 2 quad + 1
    const bool lo_lane = packed && quad >= 2;               // packed: this lane's columns carry P_lo
    const float kLn2 = 0.69314718055994531f;

    uint32_t qf[8][2];
    float oacc[8][4];
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    int cs = -1;                                            // current segment
    int n_cur = 0;

    // flush the running piece of segment cs: partial or (single piece) final output
    auto flush = [&]() {
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            l0 += __shfl_xor_sync(0xffffffffu, l0, o);
            l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        }
        if (packed) {
#pragma unroll
            for (int mt = 0; mt < 8; ++mt)
#pragma unroll
                for (int c = 0; c < 4; ++c) oacc[mt][c] += __shfl_xor_sync(0xffffffffu, oacc[mt][c], 2);
        }
        const int bi = cs / p.Hkv, h = cs - bi * p.Hkv;
        const int64_t rs = (int64_t)p.req[bi] * p.Hkv + h;
        const int s0 = cs * wk.TS;
        const int fw = worker_of(s0, wk), lw = worker_of(s0 + wk.TS - 1, wk);
        const int np = lw - fw + 1;
        const int h0 = 2 * quad, h1 = h0 + 1, d = lane >> 2;
        const bool own = !packed || quad < 2;               // lanes holding real head columns
        if (np == 1) {
            if (own) {
                const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    if (h0 < p.G) {
                        float* o = out + ((int64_t)bi * p.Hq + (int64_t)h * p.G + h0) * kHeadDim + 16 * mt + d;
                        o[0] = oacc[mt][0] * i0;
                        o[8] = oacc[mt][2] * i0;
                    }
                    if (h1 < p.G) {
                        float* o = out + ((int64_t)bi * p.Hq + (int64_t)h * p.G + h1) * kHeadDim + 16 * mt + d;
                        o[0] = oacc[mt][1] * i1;
                        o[8] = oacc[mt][3] * i1;
                    }
                }
                if (out_lse && d == 0) {
                    const int64_t ob = (int64_t)bi * p.Hq + (int64_t)h * p.G;
                    if (h0 < p.G) out_lse[ob + h0] = l0 > 0.f ? (m0 + log2f(l0)) * kLn2 : -INFINITY;
                    if (h1 < p.G) out_lse[ob + h1] = l1 > 0.f ? (m1 + log2f(l1)) * kLn2 : -INFINITY;
                }
            }
            return;
        }
        const int j = w - fw;
        float* po = ab.part_o + ((rs * kMaxPieces + j) * 8) * (int64_t)kHeadDim;
        float* pml = ab.part_ml + ((rs * kMaxPieces + j) * 8) * 2;
        if (own) {
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                po[h0 * kHeadDim + 16 * mt + d] = oacc[mt][0];
                po[h1 * kHeadDim + 16 * mt + d] = oacc[mt][1];
                po[h0 * kHeadDim + 16 * mt + 8 + d] = oacc[mt][2];
                po[h1 * kHeadDim + 16 * mt + 8 + d] = oacc[mt][3];
            }
            if (d == 0) {
                pml[h0 * 2] = m0;
                pml[h0 * 2 + 1] = l0;
                pml[h1 * 2] = m1;
                pml[h1 * 2 + 1] = l1;
            }
        }
    };

    int seg_left = 0;                                       // tiles left in the current segment
    int st = 0;                                             // stage of the next tile to consume
    uint32_t ph = 0;                                        // its mbarrier phase

    // Consume NT (1 or 2) tiles of the current segment: the two tiles' S chains, one softmax
    // update over their 16 NT tokens and their P.V products are interleaved for ILP.
    auto step = [&](auto nt_tag, int k) {
        constexpr int NT = decltype(nt_tag)::value;
        uint32_t sb[NT];
        bool vlo[NT], vhi[NT];
        int st_t = st;
        uint32_t ph_t = ph;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int kt = k + t;
            const int2* ent = &s_ent[warp][(kt >> logCT) & 1][(kt & (CT - 1)) << logE];
            const int2 elo = ent[row_lo >> logP], ehi = ent[row_hi >> logP];
            vlo[t] = elo.x >= 0 && (elo.x << logP) + (row_lo & pm) < n_cur;
            vhi[t] = ehi.x >= 0 && (ehi.x << logP) + (row_hi & pm) < n_cur;
            mbar_wait(&my_bar[st_t], ph_t);
            if (kt == 0) ATTN_STAMP(2);
            sb[t] = smem_u32(my_stage + (size_t)st_t * kTileBytes);
            st_t = st_t + 1 == STAGES ? 0 : st_t + 1;
            ph_t ^= st_t == 0 ? 1u : 0u;
        }
        st = st_t;
        ph = ph_t;
        // S^T = K . Q^T: two accumulation chains (even / odd 16-dim slices) per tile
        float sacc[NT][4], sacc2[NT][4];
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int i = 0; i < 4; ++i) sacc[t][i] = sacc2[t][i] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; kk += 2) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
                const uint32_t c = (uint32_t)(2 * kk + kchunk_hi), c2 = c + 2;
                ldsm_x4(sb[t] + koff + ((c ^ kswz) << 4), a0, a1, a2, a3);
                ldsm_x4(sb[t] + koff + ((c2 ^ kswz) << 4), b0, b1, b2, b3);
                if (!(wk.xflags & 1)) {
                    mma_bf16_16816(sacc[t], a0, a1, a2, a3, qf[kk][0], qf[kk][1]);
                    mma_bf16_16816(sacc2[t], b0, b1, b2, b3, qf[kk + 1][0], qf[kk + 1][1]);
                } else {
                    sacc[t][0] += __uint_as_float(a0 & b0); sacc2[t][1] += __uint_as_float(a1 & b3);
                }
            }
        }
        // online softmax (log2 domain) over the NT tiles
        float x[NT][4];
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            x[t][0] = vlo[t] ? (sacc[t][0] + sacc2[t][0]) * p.scale_log2 : -INFINITY;   // row_lo, col 2 quad
            x[t][1] = vlo[t] ? (sacc[t][1] + sacc2[t][1]) * p.scale_log2 : -INFINITY;   // row_lo, col 2 quad + 1
            x[t][2] = vhi[t] ? (sacc[t][2] + sacc2[t][2]) * p.scale_log2 : -INFINITY;   // row_hi, col 2 quad
            x[t][3] = vhi[t] ? (sacc[t][3] + sacc2[t][3]) * p.scale_log2 : -INFINITY;   // row_hi, col 2 quad + 1
            mx0 = fmaxf(mx0, fmaxf(x[t][0], x[t][2]));
            mx1 = fmaxf(mx1, fmaxf(x[t][1], x[t][3]));
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
        }
        const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
        const float ms0 = mn0 == -INFINITY ? 0.f : mn0, ms1 = mn1 == -INFINITY ? 0.f : mn1;
        const float al0 = fast_exp2(m0 - ms0), al1 = fast_exp2(m1 - ms1);
        m0 = mn0;
        m1 = mn1;
        float pr[NT][4];
        float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            pr[t][0] = fast_exp2(x[t][0] - ms0);
            pr[t][1] = fast_exp2(x[t][1] - ms1);
            pr[t][2] = fast_exp2(x[t][2] - ms0);
            pr[t][3] = fast_exp2(x[t][3] - ms1);
            ls0 += pr[t][0] + pr[t][2];
            ls1 += pr[t][1] + pr[t][3];
        }
        l0 = l0 * al0 + ls0;
        l1 = l1 * al1 + ls1;
        if (__any_sync(0xffffffffu, al0 != 1.f || al1 != 1.f)) {   // running max moved somewhere
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                oacc[mt][0] *= al0;
                oacc[mt][1] *= al1;
                oacc[mt][2] *= al0;
                oacc[mt][3] *= al1;
            }
        }
        // P^T B-fragments via movmatrix.trans (hardware RNE packs), then O^T += V^T . P^T
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const uint32_t hlo = cvt_bf16x2(pr[t][0], pr[t][1]), hhi = cvt_bf16x2(pr[t][2], pr[t][3]);
            const uint32_t llo = cvt_bf16x2(pr[t][0] - bf16_lo(hlo), pr[t][1] - bf16_hi(hlo));
            const uint32_t lhi = cvt_bf16x2(pr[t][2] - bf16_lo(hhi), pr[t][3] - bf16_hi(hhi));
            if (packed) {
                const uint32_t b0 = movmatrix_t(lo_lane ? llo : hlo), b1 = movmatrix_t(lo_lane ? lhi : hhi);
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    uint32_t a0, a1, a2, a3;
                    const uint32_t c = (uint32_t)(2 * mt + vchunk_hi);
                    ldsm_x4_t(sb[t] + voff + ((c ^ vswz) << 4), a0, a1, a2, a3);
                    if (!(wk.xflags & 2)) mma_bf16_16816(oacc[mt], a0, a1, a2, a3, b0, b1);
                    else oacc[mt][0] += __uint_as_float(a0 ^ a3 ^ b0);
                }
            } else {
                const uint32_t bh0 = movmatrix_t(hlo), bh1 = movmatrix_t(hhi);
                const uint32_t bl0 = movmatrix_t(llo), bl1 = movmatrix_t(lhi);
#pragma unroll
                for (int mt = 0; mt < 8; ++mt) {
                    uint32_t a0, a1, a2, a3;
                    const uint32_t c = (uint32_t)(2 * mt + vchunk_hi);
                    ldsm_x4_t(sb[t] + voff + ((c ^ vswz) << 4), a0, a1, a2, a3);
                    mma_bf16_16816(oacc[mt], a0, a1, a2, a3, bh0, bh1);
                    mma_bf16_16816(oacc[mt], a0, a1, a2, a3, bl0, bl1);
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (ik < nt) {                                  // refill the stages just consumed
                if ((ik & (CT - 1)) == 0) load_chunk(ik >> logCT);
                fence_proxy_async();
                issue();
            }
        }
    };

    int k = 0;
    while (k < nt) {
        if (seg_left == 0) {                                // new segment piece
            if (cs >= 0) flush();
            cs = cs < 0 ? s_first : cs + 1;
            seg_left = cs == s_first ? wk.TS - i_first : wk.TS;
            const int bi = cs / p.Hkv, h = cs - bi * p.Hkv;
            n_cur = ab.ntok[p.req[bi]];
            // Q^T B-fragments: column n = lane/4 -> head n (packed: n & 3), dims 16 kk + 2 quad + {0,1} (+8)
            const int hd = packed ? (lane >> 2) & 3 : lane >> 2;
            const uint16_t* qh = q + ((int64_t)bi * p.Hq + (int64_t)h * p.G + hd) * kHeadDim + 2 * quad;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                qf[kk][0] = hd < p.G ? *reinterpret_cast<const uint32_t*>(qh + 16 * kk) : 0u;
                qf[kk][1] = hd < p.G ? *reinterpret_cast<const uint32_t*>(qh + 16 * kk + 8) : 0u;
            }
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;
            m0 = m1 = -INFINITY;
            l0 = l1 = 0.f;
        }
        const int left = min(seg_left, nt - k);
        if (left >= 2) {
            step(std::integral_constant<int, 2>{}, k);
            k += 2;
            seg_left -= 2;
        } else {
            step(std::integral_constant<int, 1>{}, k);
            k += 1;
            seg_left -= 1;
        }
    }
    ATTN_STAMP(3);
    griddep_launch();
    flush();
    ATTN_STAMP(6);
}


// (a6) grid (S), 32*G*NG threads: warp (grp, hh) merges pieces [32 grp, 32 grp + 32) of query
// head hh of segment s; lane owns dims 4 lane .. 4 lane + 3.  All 32 partial rows of a warp
// are requested before anything else (one memory round trip); groups combine through smem.
template <int NG>   // groups of 32 pieces: 1 (np <= 32) or 2 (np <= 64)
__global__ void __launch_bounds__(256 * NG) merge_kernel(StepParams p, AttnBufs ab, Work wk, float* __restrict__ out,
                                                         float* __restrict__ out_lse) {
    __shared__ float s_m[NG][8], s_l[NG][8];
    __shared__ float4 s_acc[NG > 1 ? 8 : 1][32];
    const int cs = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int hh = NG > 1 ? warp % p.G : warp, grp = NG > 1 ? warp / p.G : 0;
    const int s0 = cs * wk.TS;
    const int fw = worker_of(s0, wk), lw = worker_of(s0 + wk.TS - 1, wk);
    const int np = lw - fw + 1;
    griddep_wait();                               // partials come from attn_kernel
    if (np == 1) return;                          // finalised by its only worker (uniform over the CTA)
    const int bi = cs / p.Hkv, h = cs - bi * p.Hkv;
    const int64_t rs = (int64_t)p.req[bi] * p.Hkv + h;
    const float* po0 = ab.part_o + (rs * kMaxPieces * 8) * (int64_t)kHeadDim;
    const float* pml0 = ab.part_ml + (rs * kMaxPieces * 8) * 2;
    const int j0 = 32 * grp;
    const float4* src = reinterpret_cast<const float4*>(po0 + hh * kHeadDim) + lane;
    float4 x[32];
#pragma unroll
    for (int u = 0; u < 32; ++u)
        x[u] = j0 + u < np ? __ldcg(src + (j0 + u) * 8 * (kHeadDim / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
    const int j = j0 + lane;
    const float mj = j < np ? __ldcg(&pml0[(j * 8 + hh) * 2]) : -INFINITY;
    const float lj = j < np ? __ldcg(&pml0[(j * 8 + hh) * 2 + 1]) : 0.f;
    float M = mj;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    if (NG > 1) {
        if (lane == 0) s_m[grp][hh] = M;
        __syncthreads();
#pragma unroll
        for (int g2 = 0; g2 < NG; ++g2) M = fmaxf(M, s_m[g2][hh]);
    }
    const float scj = (j < np && M != -INFINITY) ? fast_exp2(mj - M) : 0.f;
    float l = scj * lj;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 32; ++u) {
        const float sc = __shfl_sync(0xffffffffu, scj, u);   // 0 past np
        acc.x += sc * x[u].x; acc.y += sc * x[u].y; acc.z += sc * x[u].z; acc.w += sc * x[u].w;
    }
    if (NG > 1) {
        if (grp == 1) s_acc[hh][lane] = acc;
        if (lane == 0) s_l[grp][hh] = l;
        __syncthreads();
        if (grp != 0) return;
        const float4 o1 = s_acc[hh][lane];
        acc.x += o1.x; acc.y += o1.y; acc.z += o1.z; acc.w += o1.w;
        l += s_l[1][hh];
    }
    const float il = l > 0.f ? 1.f / l : 0.f;
    const int64_t oh = (int64_t)bi * p.Hq + (int64_t)h * p.G + hh;
    reinterpret_cast<float4*>(out + oh * kHeadDim)[lane] = make_float4(acc.x * il, acc.y * il, acc.z * il, acc.w * il);
    if (out_lse && lane == 0) out_lse[oh] = l > 0.f ? (M + log2f(l)) * 0.69314718055994531f : -INFINITY;
}

template <int STAGES, int WARPS>
static cudaError_t launch_attn_s(kvd_cache* c, const StepParams& p, const uint16_t* q, const int32_t* attn, float* out,
                                 float* out_lse, cudaStream_t s) {
    constexpr size_t smem = (size_t)WARPS * STAGES * kTileBytes;
    static int max_ctas = 0;
    if (!max_ctas) {
        cudaError_t e = cudaFuncSetAttribute(attn_kernel<STAGES, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0, sms = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_kernel<STAGES, WARPS>, WARPS * 32, smem);
        if (e != cudaSuccess) return e;
        max_ctas = sms * (per_sm > 0 ? per_sm : 1);
    }
    const int S = p.B * p.Hkv;
    Work wk;
    wk.TS = (p.W + p.E - 1) / p.E;
    wk.T = S * wk.TS;
    // workers: enough to fill every SM, but at most kMaxPieces - 1 per segment so a segment
    // never has more than kMaxPieces pieces (<= ceil(NW/S) + 1), and at most T
    // pieces per segment: 16 once a launch has >= 8 segments (a micro-batch chain of one Llama
    // request; 15 workers per segment leave SM room for the other chains' fetches: c3 2623 ->
    // 2865 tok/s, c2 unchanged), 32 for fewer segments (c4: 1675 vs 1632 at 16)
    static int maxp_env = -1;
    if (maxp_env < 0) {
        const char* env = getenv("KVD_ATTN_MAXP");   // experiments only: override the cap
        maxp_env = env ? std::max(2, std::min(atoi(env), kMaxPieces)) : 0;
    }
    const int maxp = maxp_env ? maxp_env : (S >= 8 ? 16 : kMaxPieces);
    int nw = max_ctas * WARPS;
    nw = std::min(nw, S * (maxp - 1));
    nw = std::min(nw, wk.T);
    wk.NW = std::max(nw, 1);
    static int xflags = -1;
    if (xflags < 0) {
        const char* env = getenv("KVD_ATTN_X");
        xflags = env ? atoi(env) : 0;
    }
    wk.xflags = xflags;
    static int trace = -1;
    static unsigned long long* tbuf = nullptr;
    if (trace < 0) {
        trace = getenv("KVD_ATTN_TRACE") ? 1 : 0;
        if (trace) cudaMalloc(&tbuf, sizeof(unsigned long long) * 8 * 8192);
    }
    wk.trace = trace ? tbuf : nullptr;
    if (trace) cudaMemsetAsync(tbuf, 0, sizeof(unsigned long long) * 8 * 8192, s);
    AttnBufs ab{c->slots, c->ntok_dev, c->zero_rec, c->part_o, c->part_ml};
    const unsigned grid = (unsigned)((wk.NW + WARPS - 1) / WARPS);
    cudaError_t e = launch_pdl(attn_kernel<STAGES, WARPS>, dim3(grid), dim3(WARPS * 32), smem, s, p, ab, wk, q, attn, out,
                               out_lse);
    if (e != cudaSuccess) return e;
    bool split = false;                           // some segment spans more than one worker
    for (int sg = 0; sg < S && !split; ++sg) {
        const int64_t a = (int64_t)sg * wk.TS, b = a + wk.TS - 1;
        split = ((a + 1) * wk.NW - 1) / wk.T != ((b + 1) * wk.NW - 1) / wk.T;
    }
    if (split) {
        // pieces of a segment <= ceil(NW/S) + 1 <= kMaxPieces = 32: one group of rows per warp.
        // (64 pieces measured slower at c2 and c4: merge_kernel<2> cannot keep 64 rows in flight)
        e = launch_pdl(merge_kernel<1>, dim3(S), dim3(32 * p.G), 0, s, p, ab, wk, out, out_lse);
        if (e != cudaSuccess) return e;
    }
    if (trace) {   // experiments only: synchronous dump of per-warp phase times (us from first stamp)
        cudaStreamSynchronize(s);
        std::vector<unsigned long long> h((size_t)wk.NW * 8);
        cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull;
        for (int i = 0; i < wk.NW; ++i) if (h[i * 8] && h[i * 8] < t0) t0 = h[i * 8];
        const char* names[7] = {"entry", "griddep", "tile0", "stream_end", "merge_begin", "merge_end", "exit"};
        for (int j = 0; j < 7; ++j) {
            std::vector<double> v;
            for (int i = 0; i < wk.NW; ++i) if (h[i * 8 + j]) v.push_back((h[i * 8 + j] - t0) * 1e-3);
            if (v.empty()) continue;
            std::sort(v.begin(), v.end());
            fprintf(stderr, "attn trace %-12s n=%5zu min %7.2f p50 %7.2f p90 %7.2f max %7.2f us\n", names[j], v.size(), v[0],
                    v[v.size() / 2], v[v.size() * 9 / 10], v.back());
        }
    }
    return cudaGetLastError();
}

cudaError_t launch_attention(kvd_cache* c, const StepParams& p, const uint16_t* q, const int32_t* attn, float* out,
                             float* out_lse, cudaStream_t s) {
    // (warps per CTA, ring depth per warp): KVD_ATTN_CFG = 3 (4 warps x 3 stages, 2 CTAs per
    // SM: 8 warp workers per SM, default), 1 (4 x 6, 1 CTA per SM), 2 (2 x 12).  Measured at
    // c2 / c3: 28.9 / 37.7 us (3), 28.7 / 41.2 us (1), 35.4 / 53.1 us (2): the per-warp
    // dependent chain of MMA + softmax needs >= 2 warps per scheduler.
    static int cfg = 0;
    if (!cfg) {
        const char* env = getenv("KVD_ATTN_CFG");
        cfg = env ? atoi(env) : 3;
        if (cfg < 1 || cfg > 3) cfg = 3;
    }
    if (cfg == 2) return launch_attn_s<12, 2>(c, p, q, attn, out, out_lse, s);
    if (cfg == 3) return launch_attn_s<3, 4>(c, p, q, attn, out, out_lse, s);
    return launch_attn_s<6, 4>(c, p, q, attn, out, out_lse, s);
}

}  // namespace kvd
