// k_attn.cu — rows (a5) split-K sparse decode attention and (a6) LSE merge, one kernel.
//
// "executing attention ... over the union of the newly fetched and resident KV
// entries".  The attention lists from resolve (selected +
// pinned blocks, ascending) are cut into 16-token tiles (E = 16/P list
// entries, 8 KiB).  Every segment has TS = ceil(W/E) tiles (uniform in a call;
// entries past a segment's valid length read a zero record and are masked).
//
// Split plan.  A segment's tiles are cut into NP = attn_pieces(TS) pieces
// (internal.h; 4..32, about 8 tiles each), piece j = tiles [j*TS/NP,
// (j+1)*TS/NP).  The plan depends on TS (i.e. on k) only, never on how many
// segments share the launch, so outputs are bit-identical however the requests
// are batched, chained or sharded over GPUs.  One thread-block cluster of
// NP/4 CTAs x 4 warps serves one segment: warp w of CTA rank r computes piece
// 4r + w.
//
// Per warp: a private STAGES-deep ring of 8 KiB tiles in shared memory fed by
// bulk async copies (TMA engine) completing on mbarriers; the (block, slot)
// entries are staged through shared memory 128 at a time so a copy is never
// issued behind a dependent global load.  Per tile, on tensor cores (mma.sync
// m16n8k16 bf16 -> fp32, swap-AB: 16 tokens fill M, heads N):
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
// (a6) Each warp leaves its unnormalised partial (o~_j, m_j, l_j) in its own
// shared memory; after a cluster barrier the cluster's warps read the NP
// partials of the segment through distributed shared memory (one (head, 32-dim
// quarter) slice each, every load issued at once) and combine them in piece
// order j = 0 .. NP-1:
//     m = max_j m_j;  l = sum_j l_j 2^(m_j-m);  o = sum_j 2^(m_j-m) o~_j / l;
//     lse = (m + log2 l) ln 2.
// No partial touches global memory and there is no second kernel.  HBM-bound:
// 8 KiB per 16-token tile; 4*G flop per 4 B of K/V.
#include <algorithm>
#include <cooperative_groups.h>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace kvd {

struct AttnBufs {
    const uint8_t* slots;
    const int32_t* ntok;
    const uint8_t* zero_rec;
};

constexpr int kEntChunk = 128;                      // list entries staged per chunk (>= STAGES * 16)
constexpr int kAttnWarpsPerCta = 4;                 // pieces per CTA of a segment's cluster

struct Work {
    int32_t TS;         // tiles per segment
    int32_t NP;         // pieces per segment (attn_pieces(TS)), 4 * cluster size
};

// partial of one warp (piece) in its stage ring: o~[8 heads][128] fp32 then (m, l)[8 heads]
constexpr int kPartFloats = 8 * kHeadDim + 16;

template <int STAGES>
__global__ void __launch_bounds__(kAttnWarpsPerCta * 32, STAGES == 2 ? 3 : 1) attn_kernel(StepParams p, AttnBufs ab, Work wk,
                                                                         const uint16_t* __restrict__ q,
                                                                         const int32_t* __restrict__ attn,
                                                                         float* __restrict__ out,
                                                                         float* __restrict__ out_lse) {
    constexpr int WARPS = kAttnWarpsPerCta;
    extern __shared__ __align__(1024) uint8_t stage[];
    __shared__ __align__(8) uint64_t bar[WARPS][STAGES];
    __shared__ int2 s_ent[WARPS][2][kEntChunk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int crank = (int)cg::this_cluster().block_rank();
    const int ncl = (int)cg::this_cluster().num_blocks();
    const int cs = blockIdx.y;                                 // segment (request bi, KV head h)
    const int bi = cs / p.nh, h = p.h0 + (cs - bi * p.nh);
    const int j = crank * WARPS + warp;                         // this warp's piece
    const int ta = (j * wk.TS) / wk.NP, nt = ((j + 1) * wk.TS) / wk.NP - ta;
    uint8_t* my_stage = stage + (size_t)warp * STAGES * kTileBytes;
    uint64_t* my_bar = bar[warp];
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&my_bar[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    // P, E = 16/P and CT = kEntChunk/E >= STAGES (tiles per entry chunk) are powers of two: shifts, no divisions
    const int logP = __ffs(p.P) - 1, logE = 4 - logP, logCT = 7 - logE;
    const int E = 1 << logE, rec = p.rec_bytes, CT = 1 << logCT;
    const uint64_t pol = l2_evict_first_policy();
    const uint8_t* seg_slots = ab.slots + (((int64_t)p.layer * p.R + p.req[bi]) * p.Hkv + h) * p.C * (int64_t)rec;
    const int2* seg_list = reinterpret_cast<const int2*>(attn) + ((int64_t)bi * p.Hkv + h) * p.W;
    if (lane == 0) EXP_STAMP(p.exp_trace, cs * 32 + j, 0);
    const bool packed = p.G <= 4;
    const int quad = lane & 3;                              // accumulator columns 2 quad, 2 quad + 1
    // Q^T B-fragments: column n = lane/4 -> head n (packed: n & 3), dims 16 kk + 2 quad + {0,1} (+8).
    // q is the query the select call read, two kernels back in the stream (every step kernel waits
    // on its predecessor before triggering this one), so it is loaded before the wait.
    uint32_t qf[8][2];
    {
        const int hd = packed ? (lane >> 2) & 3 : lane >> 2;
        const uint16_t* qh = q + ((int64_t)bi * p.Hq + (int64_t)h * p.G + hd) * kHeadDim + 2 * quad;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            qf[kk][0] = hd < p.G ? *reinterpret_cast<const uint32_t*>(qh + 16 * kk) : 0u;
            qf[kk][1] = hd < p.G ? *reinterpret_cast<const uint32_t*>(qh + 16 * kk + 8) : 0u;
        }
    }
    griddep_wait();                                // lists / slots come from the select call
    if (p.early_trigger) griddep_launch();
    if (lane == 0) EXP_STAMP(p.exp_trace, cs * 32 + j, 1);
    if (threadIdx.x == 0) kt_begin(p.kt_slots, p.kt_base + kKtAttn);

    // stage entry chunk c (tiles ta + c*CT ..) into buffer c & 1: (block, slot), or (-1, -1).
    // resolve pads each list past its valid length with (-1, -1); entries >= W are tile padding.
    auto load_chunk = [&](int c) {
        for (int i = lane; i < kEntChunk; i += 32) {
            const int k = (c << logCT) + (i >> logE);   // piece-relative tile
            int2 v = make_int2(-1, -1);
            if (k < nt) {
                const int e = ((ta + k) << logE) + (i & (E - 1));
                if (e < p.W) v = seg_list[e];
            }
            s_ent[warp][c & 1][i] = v;
        }
        __syncwarp();
    };
    int ik = 0, ist = 0;                                        // issue side: tile ik -> stage ist
    auto issue = [&]() {
        if (lane == 0) {
            uint64_t* b = &my_bar[ist];
            uint8_t* dst = my_stage + (size_t)ist * kTileBytes;
            mbar_arrive_expect_tx(b, (uint32_t)(E * rec));
            const int2* ent = &s_ent[warp][(ik >> logCT) & 1][(ik & (CT - 1)) << logE];
            for (int e = 0; e < E; ++e) {
                const int32_t slot = ent[e].y;
                const uint8_t* src = slot >= 0 ? seg_slots + (int64_t)slot * rec : ab.zero_rec;
                bulk_g2s_hint(dst + e * rec, src, (uint32_t)rec, b, pol);
            }
        }
        ++ik;
        ist = ist + 1 == STAGES ? 0 : ist + 1;
    };
    if (nt > 0) {
        load_chunk(0);
        while (ik < STAGES && ik < nt) issue();
    }

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
    const bool lo_lane = packed && quad >= 2;               // packed: this lane's columns carry P_lo
    const float kLn2 = 0.69314718055994531f;
    const int n_cur = ab.ntok[p.req[bi]];

    float oacc[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    int st = 0;                                             // stage of the next tile to consume
    uint32_t ph = 0;                                        // its mbarrier phase

    // Consume NT (1 or 2) tiles: the two tiles' S chains, one softmax
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
            if (kt == 0 && lane == 0) EXP_STAMP(p.exp_trace, cs * 32 + j, 2);
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
        if (nt - k >= 2) {
            step(std::integral_constant<int, 2>{}, k);
            k += 2;
        } else {
            step(std::integral_constant<int, 1>{}, k);
            k += 1;
        }
    }
    if (lane == 0) EXP_STAMP(p.exp_trace, cs * 32 + j, 3);
    griddep_launch();

    // ---- this piece's partial -> this warp's stage ring (its tiles are all consumed)
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
    float* part = reinterpret_cast<float*>(my_stage);
    {
        const int h0 = 2 * quad, h1 = h0 + 1, d = lane >> 2;
        if (!packed || quad < 2) {                          // lanes holding real head columns
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                part[h0 * kHeadDim + 16 * mt + d] = oacc[mt][0];
                part[h1 * kHeadDim + 16 * mt + d] = oacc[mt][1];
                part[h0 * kHeadDim + 16 * mt + 8 + d] = oacc[mt][2];
                part[h1 * kHeadDim + 16 * mt + 8 + d] = oacc[mt][3];
            }
            if (d == 0) {
                part[8 * kHeadDim + 2 * h0] = m0;
                part[8 * kHeadDim + 2 * h0 + 1] = l0;
                part[8 * kHeadDim + 2 * h1] = m1;
                part[8 * kHeadDim + 2 * h1 + 1] = l1;
            }
        }
    }
    cg::this_cluster().sync();                              // every partial of the segment is in place

    // ---- (a6) merge: item = (head hh, 32-dim quarter qd); lane owns dim 32 qd + lane.  Every
    // partial value of the item is requested at once (distributed shared memory), then summed in
    // piece order j.
    const int nwarps = ncl * WARPS;
    auto part_of = [&](int jj) {                            // piece jj's partial (remote shared memory)
        return cg::this_cluster().map_shared_rank(
            reinterpret_cast<float*>(stage + (size_t)(jj % WARPS) * STAGES * kTileBytes), jj / WARPS);
    };
    for (int item = j; item < p.G * 4; item += nwarps) {
        const int hh = item >> 2, dd = (item & 3) * 32 + lane;
        // lane jj holds piece jj's (m, l) of head hh (one load per lane); every lane then loads its
        // dim of every piece (coalesced 128-byte rows): all requests in flight at once
        const float* pl = lane < wk.NP ? part_of(lane) : nullptr;
        const float mjl = pl ? pl[8 * kHeadDim + 2 * hh] : -INFINITY;
        const float ljl = pl ? pl[8 * kHeadDim + 2 * hh + 1] : 0.f;
        float x[kMaxPieces];
#pragma unroll
        for (int jj = 0; jj < kMaxPieces; ++jj)
            if (jj < wk.NP) x[jj] = part_of(jj)[hh * kHeadDim + dd];
        float M = mjl;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float scl = (mjl != -INFINITY && M != -INFINITY) ? fast_exp2(mjl - M) : 0.f;
        float l = 0.f, acc = 0.f;
#pragma unroll
        for (int jj = 0; jj < kMaxPieces; ++jj) {           // sequential in j
            const float sc = __shfl_sync(0xffffffffu, scl, jj);
            const float lu = __shfl_sync(0xffffffffu, ljl, jj);
            if (jj < wk.NP) {
                l = __fmaf_rn(sc, lu, l);
                acc = __fmaf_rn(sc, x[jj], acc);
            }
        }
        const int64_t oh = (int64_t)bi * p.Hq + (int64_t)h * p.G + hh;
        out[oh * kHeadDim + dd] = l > 0.f ? acc * (1.f / l) : 0.f;
        if (out_lse && (item & 3) == 0 && lane == 0) out_lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : -INFINITY;
    }
    if (lane == 0) EXP_STAMP(p.exp_trace, cs * 32 + j, 4);
    cg::this_cluster().sync();                              // remote reads done before any CTA exits
    if (p.kt_slots && threadIdx.x == 0)
        kt_end(p.kt_slots, p.kt_acc, p.kt_base + kKtAttn, kKtAttn, (unsigned long long)gridDim.x * gridDim.y);
}

template <int STAGES>
static cudaError_t launch_attn_s(kvd_cache* c, const StepParams& p, const uint16_t* q, const int32_t* attn, float* out,
                                 float* out_lse, cudaStream_t s) {
    constexpr size_t smem = (size_t)kAttnWarpsPerCta * STAGES * kTileBytes;
    static_assert(STAGES * kTileBytes >= kPartFloats * 4, "a warp's partial fits its stage ring");
    static bool attr_set[64] = {};
    const int dev = c->cfg.device & 63;
    if (!attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(attn_kernel<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    Work wk;
    wk.TS = (p.W + p.E - 1) / p.E;
    wk.NP = attn_pieces(wk.TS);
#ifdef KVD_EXPERIMENTS
    if (const char* e = getenv("KVD_ATTN_NP")) wk.NP = std::max(4, std::min(kMaxPieces, atoi(e) / 4 * 4));   // tuning only
#endif
    AttnBufs ab{c->slots, c->ntok_dev + (int64_t)p.layer * c->R, c->zero_rec};   // token counts of this layer
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(wk.NP / kAttnWarpsPerCta), (unsigned)(p.B * p.nh));
    cfg.blockDim = dim3(kAttnWarpsPerCta * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = wk.NP / kAttnWarpsPerCta;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    count_launch();
    cudaError_t e = cudaLaunchKernelEx(&cfg, attn_kernel<STAGES>, p, ab, wk, q, attn, out, out_lse);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_attention(kvd_cache* c, const StepParams& p, const uint16_t* q, const int32_t* attn, float* out,
                             float* out_lse, cudaStream_t s) {
    // 4 warps x 3 stages of 8 KiB per CTA, 2 CTAs per SM (the per-warp dependent chain of MMA +
    // softmax needs >= 2 warps per scheduler; measured round 1).  KVD_ATTN_STAGES=2 (experiment
    // builds): 2 stages, 3 CTAs per SM (167 registers, no spills).
#ifdef KVD_EXPERIMENTS
    if (const char* e = getenv("KVD_ATTN_STAGES"))
        if (atoi(e) == 2) return launch_attn_s<2>(c, p, q, attn, out, out_lse, s);
#endif
    return launch_attn_s<3>(c, p, q, attn, out, out_lse, s);
}

}  // namespace kvd
