// k_attn.cu — rows (a5) split-K sparse decode attention and (a6) LSE merge, one kernel.
//
// "executing attention ... over the union of the newly fetched and resident KV
// entries".  The attention lists from resolve (selected +
// pinned blocks, ascending) are cut into 16-token tiles (E = 16/P list
// entries, 8 KiB).  Every segment has TS = ceil(W/E) tiles (uniform in a call;
// entries past a segment's valid length read a zero record and are masked).
//
// Split plan.  A segment's tiles are cut into NP = attn_pieces(TS) pieces of
// >= 8 tiles (internal.h).  The plan depends on TS (i.e. on k) only, never on
// how many segments share the launch, so outputs are bit-identical however the
// requests are batched, chained or sharded over GPUs.  The call's S*NP pieces
// are dealt to NW warp workers in contiguous ranges (stream-K over pieces:
// worker w owns pieces [w*Ptot/NW, (w+1)*Ptot/NW)); consecutive pieces are
// consecutive tiles, so a worker streams one contiguous tile range and its
// copy pipeline runs across piece and segment boundaries without a break.
//
// Per worker (one warp; 8 per SM): a private STAGES-deep ring of 8 KiB tiles in
// shared memory fed by bulk async copies (TMA engine) completing on mbarriers;
// the (block, slot) entries are staged through shared memory 128 at a time so
// a copy is never issued behind a dependent global load.  Per tile, on tensor
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
// (a6) At the end of each piece the worker writes its unnormalised partial
// (o~_j, m_j, l_j) with plain stores; merge_kernel, launched behind attn_kernel
// with programmatic dependent launch (its CTAs are resident before the
// attention grid drains, and griddepcontrol.wait orders the partials: no
// fences or arrival counters on the streaming path), combines the NP partials
// of every segment in piece order j = 0 .. NP-1:
//     m = max_j m_j;  l = sum_j l_j 2^(m_j-m);  o = sum_j 2^(m_j-m) o~_j / l;
//     lse = (m + log2 l) ln 2.
// One CTA per segment, one warp per query head; each lane requests all NP of
// its partial rows at once (one memory round trip).  A segment of one piece is
// finalised in place by its worker.  HBM-bound: 8 KiB per 16-token tile; 4*G
// flop per 4 B of K/V.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

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
    int32_t TS;         // tiles per segment
    int32_t NP;         // pieces per segment (attn_pieces(TS))
    int32_t Ptot;       // pieces of the call (S * NP)
    int32_t NW;         // workers
};

// first tile of global piece gp (pieces of a segment are balanced: i*TS/NP)
__device__ __forceinline__ int piece_tile(int gp, const Work& wk) {
    const int s = gp / wk.NP, i = gp - s * wk.NP;
    return s * wk.TS + (i * wk.TS) / wk.NP;
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
    const int pa = w < wk.NW ? (int)((int64_t)w * wk.Ptot / wk.NW) : 0;
    const int pb = w < wk.NW ? (int)((int64_t)(w + 1) * wk.Ptot / wk.NW) : 0;
    const int ta = piece_tile(pa, wk);
    const int nt = piece_tile(pb, wk) - ta;
    const int s_first = ta / wk.TS, i_first = ta - s_first * wk.TS;   // segment / tile-in-segment of tile ta
    // P, E = 16/P and CT = kEntChunk/E >= STAGES (tiles per entry chunk) are powers of two: shifts, no divisions
    const int logP = __ffs(p.P) - 1, logE = 4 - logP, logCT = 7 - logE;
    const int E = 1 << logE, rec = p.rec_bytes, CT = 1 << logCT;
    const uint64_t pol = l2_evict_first_policy();
    const bool packed = p.G <= 4;
    if (lane == 0) EXP_STAMP(p.exp_trace, w, 0);
    griddep_wait();                                // lists / slots / q come from earlier kernels
    if (lane == 0) EXP_STAMP(p.exp_trace, w, 1);
    // kernel timer (kvd.h): one start / end per CTA; the CTA's last warp to finish ends it
    __shared__ int kt_warps_done;
    if (threadIdx.x == 0) {
        kt_warps_done = 0;
        kt_begin(p.kt_slots, p.kt_base + kKtAttn);
    }
    __syncthreads();
    auto kt_warp_exit = [&]() {
        if (p.kt_slots && lane == 0 && atomicAdd(&kt_warps_done, 1) == WARPS - 1)
            kt_end(p.kt_slots, p.kt_acc, p.kt_base + kKtAttn, kKtAttn, gridDim.x);
    };
    if (nt <= 0) {
        kt_warp_exit();
        return;
    }

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
    int cp = pa - 1;                                        // current piece (global index)
    int n_cur = 0;

    // flush piece cp of segment cs: final output (one-piece segment) or partial + arrival
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
        const int h0 = 2 * quad, h1 = h0 + 1, d = lane >> 2;
        const bool own = !packed || quad < 2;               // lanes holding real head columns
        if (wk.NP == 1) {
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
        const int j = cp - cs * wk.NP;                      // piece index within the segment
        float* po = ab.part_o + ((rs * kMaxPieces + j) * 8) * (int64_t)kHeadDim;
        float* pml = ab.part_ml + ((rs * kMaxPieces + j) * 8) * 2;
        if (own) {
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                __stcg(&po[h0 * kHeadDim + 16 * mt + d], oacc[mt][0]);
                __stcg(&po[h1 * kHeadDim + 16 * mt + d], oacc[mt][1]);
                __stcg(&po[h0 * kHeadDim + 16 * mt + 8 + d], oacc[mt][2]);
                __stcg(&po[h1 * kHeadDim + 16 * mt + 8 + d], oacc[mt][3]);
            }
            if (d == 0) {
                __stcg(&pml[h0 * 2], m0);
                __stcg(&pml[h0 * 2 + 1], l0);
                __stcg(&pml[h1 * 2], m1);
                __stcg(&pml[h1 * 2 + 1], l1);
            }
        }
    };

    int piece_left = 0;                                     // tiles left in the current piece
    int st = 0;                                             // stage of the next tile to consume
    uint32_t ph = 0;                                        // its mbarrier phase

    // Consume NT (1 or 2) tiles of the current piece: the two tiles' S chains, one softmax
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
            if (kt == 0 && lane == 0) EXP_STAMP(p.exp_trace, w, 2);
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
                mma_bf16_16816(sacc[t], a0, a1, a2, a3, qf[kk][0], qf[kk][1]);
                mma_bf16_16816(sacc2[t], b0, b1, b2, b3, qf[kk + 1][0], qf[kk + 1][1]);
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
                    mma_bf16_16816(oacc[mt], a0, a1, a2, a3, b0, b1);
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
        if (piece_left == 0) {                              // next piece
            if (cp >= pa) flush();
            ++cp;
            const int s = cp / wk.NP, i = cp - s * wk.NP;
            piece_left = ((i + 1) * wk.TS) / wk.NP - (i * wk.TS) / wk.NP;
            if (s != cs) {                                  // new segment: its query fragments
                cs = s;
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
            }
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;
            m0 = m1 = -INFINITY;
            l0 = l1 = 0.f;
        }
        const int left = min(piece_left, nt - k);
        if (left >= 2) {
            step(std::integral_constant<int, 2>{}, k);
            k += 2;
            piece_left -= 2;
        } else {
            step(std::integral_constant<int, 1>{}, k);
            k += 1;
            piece_left -= 1;
        }
    }
    if (lane == 0) EXP_STAMP(p.exp_trace, w, 3);
    griddep_launch();
    flush();
    __syncwarp();
    if (lane == 0) EXP_STAMP(p.exp_trace, w, 4);
    kt_warp_exit();
}

// (a6) grid (S), 32*G threads: warp hh merges query head hh of segment blockIdx.x; lane owns dims
// 4 lane .. 4 lane + 3.  Thread 0 copies the segment's NP partial blocks (G rows of 512 B each,
// contiguous per piece) into shared memory with bulk async copies on one mbarrier while lane j
// loads (m_j, l_j): one memory round trip for everything.  The sums run in piece order j.
__global__ void __launch_bounds__(32 * KVD_MAX_GROUP) merge_kernel(StepParams p, AttnBufs ab, Work wk,
                                                                 float* __restrict__ out, float* __restrict__ out_lse) {
    extern __shared__ __align__(128) float4 s_part[];   // [NP][G][32] float4
    __shared__ __align__(8) uint64_t bar;
    const int cs = blockIdx.x;
    const int lane = threadIdx.x & 31, hh = threadIdx.x >> 5;
    const int NP = wk.NP, G = p.G;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    griddep_wait();                               // partials come from attn_kernel
    if (threadIdx.x == 0) kt_begin(p.kt_slots, p.kt_base + kKtMerge);
    const int bi = cs / p.Hkv, h = cs - bi * p.Hkv;
    const int64_t rs = (int64_t)p.req[bi] * p.Hkv + h;
    const float* po = ab.part_o + rs * kMaxPieces * 8 * (int64_t)kHeadDim;
    if (threadIdx.x == 0) {
        const uint32_t row = (uint32_t)(G * kHeadDim * 4);
        mbar_arrive_expect_tx(&bar, row * (uint32_t)NP);
        for (int j = 0; j < NP; ++j) bulk_g2s(s_part + j * G * 32, po + (int64_t)j * 8 * kHeadDim, row, &bar);
    }
    const float* pml = ab.part_ml + (rs * kMaxPieces * 8 + hh) * 2;
    const float mj = lane < NP ? pml[lane * 16] : -INFINITY;   // a new kernel: plain loads see the
    const float lj = lane < NP ? pml[lane * 16 + 1] : 0.f;     // partials (griddepcontrol.wait)
    float M = mj;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    const float scj = (lane < NP && M != -INFINITY) ? fast_exp2(mj - M) : 0.f;
    mbar_wait(&bar, 0);
    float l = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < NP; ++j) {                // sequential in j
        const float sc = __shfl_sync(0xffffffffu, scj, j);
        const float lu = __shfl_sync(0xffffffffu, lj, j);
        const float4 x = s_part[(j * G + hh) * 32 + lane];
        l = __fmaf_rn(sc, lu, l);
        acc.x = __fmaf_rn(sc, x.x, acc.x);
        acc.y = __fmaf_rn(sc, x.y, acc.y);
        acc.z = __fmaf_rn(sc, x.z, acc.z);
        acc.w = __fmaf_rn(sc, x.w, acc.w);
    }
    const float il = l > 0.f ? 1.f / l : 0.f;
    const int64_t oh = (int64_t)bi * p.Hq + (int64_t)h * G + hh;
    reinterpret_cast<float4*>(out + oh * kHeadDim)[lane] = make_float4(acc.x * il, acc.y * il, acc.z * il, acc.w * il);
    if (out_lse && lane == 0) out_lse[oh] = l > 0.f ? (M + log2f(l)) * 0.69314718055994531f : -INFINITY;
    if (p.kt_slots) {
        __syncthreads();
        if (threadIdx.x == 0) kt_end(p.kt_slots, p.kt_acc, p.kt_base + kKtMerge, kKtMerge, gridDim.x);
    }
}

template <int STAGES, int WARPS>
static cudaError_t launch_attn_s(kvd_cache* c, const StepParams& p, const uint16_t* q, const int32_t* attn, float* out,
                                 float* out_lse, cudaStream_t s) {
    constexpr size_t smem = (size_t)WARPS * STAGES * kTileBytes;
    static int max_ctas[64] = {};                 // per device ordinal
    const int dev = c->cfg.device & 63;
    if (!max_ctas[dev]) {
        cudaError_t e = cudaFuncSetAttribute(attn_kernel<STAGES, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int per_sm = 0, sms = 0;
        e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->cfg.device);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_kernel<STAGES, WARPS>, WARPS * 32, smem);
        if (e != cudaSuccess) return e;
        max_ctas[dev] = sms * (per_sm > 0 ? per_sm : 1);
    }
    Work wk;
    wk.TS = (p.W + p.E - 1) / p.E;
    wk.NP = attn_pieces(wk.TS);
#ifdef KVD_EXPERIMENTS
    if (const char* e = getenv("KVD_ATTN_PIECE_TILES")) {   // experiment builds only
        const int pt = std::max(1, atoi(e));
        wk.NP = std::max(1, std::min(kMaxPieces, (wk.TS + pt - 1) / pt));
    }
#endif
    wk.Ptot = p.B * p.Hkv * wk.NP;
    // workers: every warp slot of the device at most, with an even number of pieces each
    // (ppw = ceil(Ptot / slots); NW = ceil(Ptot / ppw)), so no worker has a piece more than
    // the others -- the assignment never changes the arithmetic (the plan is per segment)
    const int slots = max_ctas[dev] * WARPS;
    const int ppw = (wk.Ptot + slots - 1) / slots;
    wk.NW = std::max(1, (wk.Ptot + ppw - 1) / ppw);
    AttnBufs ab{c->slots, c->ntok_dev, c->zero_rec, c->part_o, c->part_ml};
    const unsigned grid = (unsigned)((wk.NW + WARPS - 1) / WARPS);
    cudaError_t e = launch_pdl(attn_kernel<STAGES, WARPS>, dim3(grid), dim3(WARPS * 32), smem, s, p, ab, wk, q, attn,
                               out, out_lse);
    if (e != cudaSuccess) return e;
    if (wk.NP > 1) {                              // split segments: LSE merge behind it (PDL)
        const size_t msmem = (size_t)wk.NP * p.G * kHeadDim * 4;   // <= 32 x 8 x 512 B = 128 KiB
        static size_t msmem_set[64] = {};
        if (msmem > msmem_set[dev]) {
            e = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem);
            if (e != cudaSuccess) return e;
            msmem_set[dev] = msmem;
        }
        e = launch_pdl(merge_kernel, dim3(p.B * p.Hkv), dim3(32 * p.G), msmem, s, p, ab, wk, out, out_lse);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

cudaError_t launch_attention(kvd_cache* c, const StepParams& p, const uint16_t* q, const int32_t* attn, float* out,
                             float* out_lse, cudaStream_t s) {
    // 4 warps x 3 stages of 8 KiB per CTA, 2 CTAs per SM: 8 warp workers per SM (the per-warp
    // dependent chain of MMA + softmax needs >= 2 warps per scheduler; measured round 1:
    // 4 x 6 stages at 1 CTA/SM and 2 x 12 stages were slower at c2 / c3)
    return launch_attn_s<3, 4>(c, p, q, attn, out, out_lse, s);
}

}  // namespace kvd
