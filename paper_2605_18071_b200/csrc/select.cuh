// select.cuh — rows (a1) summary scoring and (a2) top-k block selection, in one
// kernel (plus, fused, rows (a3) resolve and (a4) miss fetch).
//
// (a1) "identifying critical KV entries via the index": every
// block's score is the dot product of the KV head's group query with the
// block's mean-key summary, computed as one fp32 FMA chain
// over the 128 dims in order (DESIGN.md §3 R3, R5) so that ids are bit-exact.
// HBM-bound: 256 B of summary per block.  select_kernel runs one thread-block
// cluster of CL CTAs x NT threads per segment; CTA rank c scores its span of
// NT*kpt blocks straight into shared memory as monotone keys.  The summaries
// are dim-major, so a thread owning V consecutive blocks reads one V*2-byte
// vector per dim row and a warp reads 64*V contiguous bytes per row
// (coalesced); each thread keeps 2R rows in flight (two ping-pong register
// batches) and runs V independent FMA chains.  The first batch is requested
// before griddepcontrol.wait (summaries are immutable during a step), so it
// overlaps the previous kernel's tail.  Scores also go to HBM (4 B per 256 B
// read) for the lookahead policy and out_scores.
//
// (a2) "retrieving only the Top-K important chunks": the same
// CTAs then select.  First digit: 256 bins linear in the score value over the
// candidates' [min, max]; per-CTA histograms are summed over the cluster
// through distributed shared memory; the threshold bin's members (and the keys
// above it) are compacted; then 8-bit radix digits of the members' keys from
// the highest differing bit (warp-aggregated shared histogram adds).  The digit
// loop stops as soon as the threshold bin is taken whole, holds <= 32 keys
// (ranked directly: key desc, id asc), or is a single key value (equal keys:
// lowest ids first).  Emission: ids come out ascending with no sort.
#pragma once
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "resolve.cuh"
#include "topk.cuh"

namespace cg = cooperative_groups;

namespace kvd {

constexpr int kTieList = 32;                  // threshold bins up to this size are ranked directly

// V consecutive bf16 summary values of one dim row (one vector load per row per thread)
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
// R rows per register batch (two batches in flight): about 128 KiB of summary rows in flight per
// CTA, 2R*V*2 B per thread -- one SM streams ~140 GB/s at that depth, 32 GB/s at a quarter of it
// (tools/micro/score_stream.cu, in-kernel timing)
template <int NT, int V>
struct ScoreRows {
    static constexpr int R0 = 32768 / (NT * V);
    static constexpr int Rmax = (NT <= 512 ? 48 : 32) / V;   // register budget of the two batches
    static constexpr int Rc = R0 > Rmax ? Rmax : R0;
    // a power of two (2R divides the 128 rows)
    static constexpr int R = Rc >= 32 ? 32 : Rc >= 16 ? 16 : Rc >= 8 ? 8 : 4;
    static_assert(kHeadDim % (2 * R) == 0, "two batches of R rows must tile the 128 dims");
};

// ------------------------------------------------------------------ (a2) top-k
constexpr int kListCap = 4096;                // compacted threshold-bin members per CTA
constexpr int kTakeMax = 512;                 // list emission for k up to this

struct TopkShared {
    int hist[2][256];                 // per-pass digit histograms (double-buffered: read remotely)
    int tot[256];                     // cluster-summed histogram
    int wcnt[2][32];                  // per-warp counts of the emission pre-pass (above, bin)
    int woff[2][32];                  // their cluster-wide exclusive offsets
    uint32_t wred[2][32];
    uint32_t cmin[2], cmax[2];        // this CTA's key ranges: candidates, threshold-bin members (read remotely)
    int mm_slot;                      // next cmin/cmax slot
    int digit, above, cnt;            // pass decision (broadcast)
    int ctot[2];                      // CTA totals of the emission counts (read remotely)
    int ncomp;                        // compacted members of the first threshold bin (this CTA)
    int lcount;                       // threshold-bin members of this CTA (LIST mode)
    int ntake;                        // taken ids of this CTA (list emission)
    int32_t take[kTakeMax];
    uint32_t lkey[kTieList];
    int32_t lid[kTieList];
};

template <int CL>
__device__ __forceinline__ void cl_sync() {
    if constexpr (CL == 1) __syncthreads();
    else cg::this_cluster().sync();
}
template <int CL, class T>
__device__ __forceinline__ T* cl_remote(T* p, int rank) {
    if constexpr (CL == 1) return p;
    else return cg::this_cluster().map_shared_rank(p, rank);
}

enum { kModeWhole = 0, kModeList = 1, kModeEqual = 2 };

// cluster-wide min / max of (kmn, kmx); every thread returns the cluster values
template <int CL>
__device__ __forceinline__ void cta_minmax(uint32_t& kmn, uint32_t& kmx, TopkShared& sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    kmn = __reduce_min_sync(0xffffffffu, kmn);
    kmx = __reduce_max_sync(0xffffffffu, kmx);
    if (lane == 0) {
        sm.wred[0][warp] = kmn;
        sm.wred[1][warp] = kmx;
    }
    __syncthreads();
    if (warp == 0) {
        const bool v = lane < (int)(blockDim.x >> 5);
        const uint32_t a = __reduce_min_sync(0xffffffffu, v ? sm.wred[0][lane] : 0xFFFFFFFFu);
        const uint32_t b = __reduce_max_sync(0xffffffffu, v ? sm.wred[1][lane] : 0u);
        if (lane == 0) {
            sm.cmin[sm.mm_slot] = a;
            sm.cmax[sm.mm_slot] = b;
        }
    }
    cl_sync<CL>();
    const int slot = sm.mm_slot;
    kmn = 0xFFFFFFFFu;
    kmx = 0u;
#pragma unroll
    for (int c = 0; c < CL; ++c) {
        kmn = min(kmn, cl_remote<CL>(sm.cmin, c)[slot]);
        kmx = max(kmx, cl_remote<CL>(sm.cmax, c)[slot]);
    }
    __syncthreads();                              // everyone read mm_slot before it advances
    if (threadIdx.x == 0) sm.mm_slot = slot + 1;
    __syncthreads();
}

// warp 0: find the bin (descending) holding the kk-th largest member; lane l owns bins
// d = nbins-1-(8l+j), j < 8.  Writes sm.digit / sm.above (members in higher bins) / sm.cnt.
__device__ __forceinline__ void pick_digit(TopkShared& sm, int nbins, int kk, int lane) {
    int c8[8], t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int d = nbins - 1 - (8 * lane + j);
        c8[j] = d >= 0 ? sm.tot[d] : 0;
        t += c8[j];
    }
    int incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    int above = incl - t;
    if (above < kk && kk <= incl) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (above + c8[j] >= kk) {
                sm.digit = nbins - 1 - (8 * lane + j);
                sm.above = above;
                sm.cnt = c8[j];
                break;
            }
            above += c8[j];
        }
    }
}

// grid (CL, Hkv, B), cluster (CL, 1, 1), NT threads.  CTA rank c owns blocks
// [c*span, (c+1)*span), span = NT*kpt, staged as monotone keys in shared memory.
// Candidates = [sink_end, local_begin) (not pinned, < nb).  Every phase walks the keys in
// 32-wide strips (conflict-free shared loads); warp w owns the contiguous strip range
// [w*span/32, (w+1)*span/32) for the ordered emission.
// Fused variant (RESOLVE): after the selection, CTA rank 0 resolves the segment against the
// cache (a3, resolve.cuh) and copies its misses from the host store (a4) in the same CTA,
// reusing the dynamic shared memory: select -> resolve -> fetch without kernel boundaries.

// Selection after scoring, the default path (fa.fast): every CTA finds the K-th largest rank key
// of its own candidates (topk.cuh, CTA barriers only) and emits its top min(K, candidates) in id
// order -- straight to the output when the segment has one CTA; otherwise as rank keys into
// rank 0's candidate area (distributed shared memory), whose offset every rank derives from the
// geometry.  One cluster barrier; rank 0 then selects K of the <= CL*K candidates (already in
// ascending id order: rank c's span precedes rank c+1's) and emits them.  The global top-k is
// contained in the union of the per-CTA top-k sets, so the result is the exact top-k.
template <int CL, bool RESOLVE>
__device__ __forceinline__ void select_fast(const FuseArgs& fa, const StepParams& p, const SegGeom& g, int K,
                                            int ostride, int64_t base, int span, int crank, int c_lo, int c_hi,
                                            uint32_t kmn, uint32_t kmx, uint32_t* skey, int64_t seg, int bi, int h,
                                            int r, const float* __restrict__ scores, int32_t* __restrict__ out_ids,
                                            float* __restrict__ out_scores, ResolveShared& rsm) {
    __shared__ KthShared ks;
    const int tid = threadIdx.x;
    uint64_t* list = reinterpret_cast<uint64_t*>(skey + span);      // [kRankList] threshold-bin members
    uint64_t* cand = list + kRankList;                              // [CL * min(K, span)] (rank 0)
    uint8_t* smraw = reinterpret_cast<uint8_t*>(skey);
    int32_t* sel = reinterpret_cast<int32_t*>(smraw + fa.sel_off);  // fused: the selection, past everything
    // stage 1 (index) writes per request id: concurrent chains of one step never share rows
    int32_t* ids_out = out_ids + ((int64_t)(p.sel_mode == 1 ? r : bi) * p.Hkv + h) * ostride;
    float* sc_out = out_scores ? out_scores + ((int64_t)bi * p.Hkv + h) * ostride : nullptr;
    const float* sc_seg = scores + seg * p.nb_pad;
    auto put = [&](uint32_t id, int pos) {
        ids_out[pos] = (int32_t)id;
        if (sc_out) sc_out[pos] = __ldcg(sc_seg + id);
        if (RESOLVE) sel[pos] = (int32_t)id;
    };
    const int unit = (bi * gridDim.y + blockIdx.y) * CL + crank;
    (void)unit;
    if (tid == 0) EXP_STAMP(p.exp_trace, unit, 2);
    const SpanView sv{skey, c_lo, c_hi, (uint32_t)base};
    uint64_t T = 0ull;                                              // 0: every candidate
    if (K > 0 && c_hi - c_lo > K) T = kth_largest(sv, K, kmn, kmx, list, ks, p.exp_trace, unit);
    if (tid == 0) EXP_STAMP(p.exp_trace, unit, 5);
    if constexpr (CL == 1) {
        if (K > 0) emit_ordered(sv, T, ks, [&](int i, int pos) { put((uint32_t)(base + i), pos); });
    } else {
        auto ncand_of = [&](int c) {
            const int64_t b0 = (int64_t)c * span;
            const int64_t nbv = min(max((int64_t)g.nb - b0, (int64_t)0), (int64_t)span);
            const int64_t lo = min(max((int64_t)g.sink_end - b0, (int64_t)0), nbv);
            const int64_t hi = min(max((int64_t)g.local_begin - b0, (int64_t)0), nbv);
            return (int)(hi - lo);
        };
        int off = 0, n = 0;
#pragma unroll
        for (int c = 0; c < CL; ++c) {
            const int m = min(K, ncand_of(c));
            off += c < crank ? m : 0;
            n += m;
        }
        uint64_t* cand0 = cg::this_cluster().map_shared_rank(cand, 0);
        if (K > 0)
            emit_ordered(sv, T, ks, [&](int i, int pos) { cand0[off + pos] = rank_key(skey[i], (uint32_t)(base + i)); });
        cl_sync<CL>();              // release / acquire: every CTA's candidates and scores reach rank 0
        if (crank != 0) {
            if constexpr (!RESOLVE) griddep_launch();
            return;
        }
        const ListView lv{cand, 0, n};
        uint64_t T2 = 0ull;
        if (K > 0 && n > K) {
            uint32_t mn = 0xFFFFFFFFu, mx = 0u;
            for (int i = tid; i < n; i += blockDim.x) {
                const uint32_t k = lv.k32(i);
                if (k) {
                    mn = min(mn, k);
                    mx = max(mx, k);
                }
            }
            T2 = kth_largest(lv, K, mn, mx, list, ks);
        }
        if (K > 0) emit_ordered(lv, T2, ks, [&](int i, int pos) { put(rank_id(cand[i]), pos); });
    }
    if (tid == 0) EXP_STAMP(p.exp_trace, unit, 6);
    if constexpr (!RESOLVE) {
        griddep_launch();
    } else {
        // the sorted selection -> the resolve's S[] (sel lies past the resolve's working set);
        // resolve_main starts with a barrier
        int32_t* S = reinterpret_cast<int32_t*>(reinterpret_cast<uint64_t*>(smraw) + fa.rb.nkeys);
        for (int j = tid; j < K; j += blockDim.x) S[j] = sel[j];
        const int nm = resolve_main(p, fa.rb, bi, h, out_ids, fa.out_attn, smraw, rsm, true, true);
        if (nm > 0 && fa.host_store) {
            const int32_t* Sx = reinterpret_cast<const int32_t*>(reinterpret_cast<uint64_t*>(smraw) + fa.rb.nkeys);
            gather_segment(p, bi, h, Sx + 2 * fa.rb.kmax, Sx + 3 * fa.rb.kmax, nm, fa.host_store, fa.slots, 0, 1);
        }
    }
}

template <int CL, int NT, int V, bool RESOLVE>
__device__ __forceinline__ void select_body(const FuseArgs& fa, const StepParams& p, const uint16_t* __restrict__ q,
                                            const uint16_t* __restrict__ summ, float* __restrict__ scores,
                                            const int32_t* __restrict__ ntok, int kpt,
                                            int32_t* __restrict__ out_ids, float* __restrict__ out_scores) {
    using Vec = typename VecOf<V>::T;
    extern __shared__ __align__(16) uint32_t skey[];   // [span] keys | [kListCap] compacted pairs | [span] bins
    __shared__ TopkShared sm;
    __shared__ float qbar[kHeadDim];
    const int crank = CL > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int h = p.h0 + blockIdx.y, bi = blockIdx.z;
    const int r = p.req[bi];
    const int span = NT * kpt;
    uint2* comp = reinterpret_cast<uint2*>(skey + span);
    uint8_t* sbin = reinterpret_cast<uint8_t*>(comp + kListCap);   // first-digit bin of every key
    const int64_t base = (int64_t)crank * span;
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    // the launch's view: the segment's blocks (pinned excluded, k = p.k), or -- stage 1 of the
    // hierarchical index (R27) -- its centroids (no pinned; K = min(nc, max(ceil(4k/ratio),
    // k + pinned)), ids written with stride sel_stride)
    SegGeom g = seg_geom(ntok[r], p.P, p.sink_tokens, p.local_tokens);   // ntok: setup only
    int K = p.k, ostride = p.k;
    if (p.sel_mode == 1) {
        const int nc = p.sel_count[seg];
        const int pin = g.sink_end + (g.nb - g.local_begin);
        const int f = (kIdxFanout * p.k + p.sel_ratio - 1) / p.sel_ratio;
        K = min(nc, max(f, p.k + pin));
        ostride = p.sel_stride;
        g.n = nc;
        g.nb = nc;
        g.sink_end = 0;
        g.local_begin = nc;
    }
    auto clampi = [](int64_t x, int64_t lo_, int64_t hi_) { return (int)(x < lo_ ? lo_ : x > hi_ ? hi_ : x); };
    const int nbv = clampi((int64_t)g.nb - base, 0, span);       // positions of this CTA holding a block
    const int c_lo = clampi(g.sink_end - base, 0, nbv);
    const int c_hi = clampi(g.local_begin - base, 0, nbv);
    const int ncand = g.local_begin - g.sink_end;
    float* sc = scores + seg * p.nb_pad + base;
    __shared__ ResolveShared rsm;
    if (RESOLVE && crank == 0) resolve_pre(p, fa.rb, bi, h, rsm);
    if (tid == 0) {
        sm.lcount = 0;
        sm.ncomp = 0;
        sm.mm_slot = 0;
    }
    // ---- (a1) score this CTA's blocks straight into shared memory as monotone keys, and take
    // the candidates' key range (NaN keys are 0; every other key is >= 1).  Thread tid of group
    // gi owns the V blocks at local positions (gi*NT + tid)*V ..; dim row j of the segment's
    // summaries is contiguous (dim-major), so a warp's loads of one row are coalesced.  Two
    // ping-pong register batches of R rows keep 2R rows of every thread's blocks in flight.
    // (Measured, tools/micro/score_stream.cu: a ring of bulk async row copies into shared memory
    // streams no faster per SM than these loads, and costs the shared memory of the top-k.)
    constexpr int R = ScoreRows<NT, V>::R;
    const Vec* srow = reinterpret_cast<const Vec*>(summ + seg * kHeadDim * p.nb_pad + base);
    const int64_t rstride = p.nb_pad / V;         // Vec elements per dim row (nb_pad % 128 == 0)
    uint32_t kmn = 0xFFFFFFFFu, kmx = 0u;
#pragma unroll 1
    for (int gi = 0; gi * V < kpt; ++gi) {
        const int i0 = (gi * NT + tid) * V;
        const bool ld = i0 < nbv;                 // V-groups never straddle nb_pad
        const Vec* src = srow + (ld ? i0 / V : 0);
        Vec bufA[R], bufB[R];
#pragma unroll
        for (int u = 0; u < R; ++u)
            if (ld) bufA[u] = __ldcs(src + u * rstride);
#pragma unroll
        for (int u = 0; u < R; ++u)
            if (ld) bufB[u] = __ldcs(src + (R + u) * rstride);
        if (gi == 0) {
            griddep_wait();                       // summaries are immutable; q may come from an earlier kernel
            if (tid == 0) kt_begin(p.kt_slots, p.kt_base + kKtSelect);
            if (tid == 0) EXP_STAMP(p.exp_trace, ((bi * gridDim.y + blockIdx.y) * CL + crank), 1);
            if (tid < kHeadDim) {
                // group query: qbar[j] = ((+0 + q_0[j]) + q_1[j]) + ... (fp32, g ascending; R3)
                const uint16_t* qh = q + ((int64_t)bi * p.Hq + (int64_t)h * p.G) * kHeadDim;
                float a = 0.0f;
                for (int gq = 0; gq < p.G; ++gq) a = __fadd_rn(a, bf16_bits(qh[gq * kHeadDim + tid]));
                qbar[tid] = a;
            }
            __syncthreads();
        }
        float acc[V];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = 0.0f;
        if (p.sel_mode == 2) {
            // Quest min/max (R30): acc = acc + max(q mn, q mx), products rounded, sequential in j.
            // The minimum rows were loaded above (bufA / bufB hold rows 0 .. 2R-1 of the minima);
            // here the rows are streamed in pairs (minimum, maximum) R/2 at a time.
            const Vec* src2 = reinterpret_cast<const Vec*>(p.summ2 + seg * kHeadDim * p.nb_pad + base) + (ld ? i0 / V : 0);
#pragma unroll 1
            for (int j0 = 0; j0 < kHeadDim; j0 += R) {
                Vec mnv[R], mxv[R];
#pragma unroll
                for (int u = 0; u < R; ++u) {
                    if (ld) mnv[u] = __ldcs(src + (j0 + u) * rstride);
                    if (ld) mxv[u] = __ldcs(src2 + (j0 + u) * rstride);
                }
#pragma unroll
                for (int u = 0; u < R; ++u) {
                    const float qj = qbar[j0 + u];
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        const uint32_t wn = VecOf<V>::word(mnv[u], v >> 1), wx = VecOf<V>::word(mxv[u], v >> 1);
                        const float a = __fmul_rn(qj, (v & 1) ? bf16_hi(wn) : bf16_lo(wn));
                        const float b2 = __fmul_rn(qj, (v & 1) ? bf16_hi(wx) : bf16_lo(wx));
                        acc[v] = __fadd_rn(acc[v], fmaxf(a, b2));
                    }
                }
            }
        }
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
        for (int j0 = 0; j0 < (p.sel_mode == 2 ? 0 : kHeadDim); j0 += 2 * R) {
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
        if (ld) {
            uint32_t key[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                key[v] = score_key32(acc[v]);
                const int i = i0 + v;
                if (i >= c_lo && i < c_hi && key[v] != 0u) {
                    kmn = min(kmn, key[v]);
                    kmx = max(kmx, key[v]);
                }
            }
#pragma unroll
            for (int v = 0; v < V; v += 2) *reinterpret_cast<uint2*>(&skey[i0 + v]) = make_uint2(key[v], key[v + 1]);
            if (i0 + V <= nbv) {
#pragma unroll
                for (int v = 0; v < V; v += 2) *reinterpret_cast<float2*>(sc + i0 + v) = make_float2(acc[v], acc[v + 1]);
            } else {
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (i0 + v < nbv) sc[i0 + v] = acc[v];
            }
        }
    }
    if (fa.fast) {
        select_fast<CL, RESOLVE>(fa, p, g, K, ostride, base, span, crank, c_lo, c_hi, kmn, kmx, skey, seg, bi, h, r,
                                 scores, out_ids, out_scores, rsm);
        return;
    }
    // ---- general path (a cluster whose candidates do not fit rank 0's candidate area: K large)
    cta_minmax<CL>(kmn, kmx, sm);
    if (tid == 0) EXP_STAMP(p.exp_trace, ((bi * gridDim.y + blockIdx.y) * CL + crank), 2);
    if (K == 0) {
        // nothing to select (the scores are still kept: lookahead victims, kvd_read_scores).  The
        // cluster barrier ends the remote min/max reads and publishes the scores to rank 0.
        cl_sync<CL>();
        if constexpr (RESOLVE) {
            if (crank == 0) {
                uint8_t* smraw = reinterpret_cast<uint8_t*>(skey);
                resolve_main(p, fa.rb, bi, h, out_ids, fa.out_attn, smraw, rsm, true, true);
            }
        } else {
            griddep_launch();
        }
        return;
    }
    // ---- first digit: 256 bins linear in the score value over [vmin, vmax] (monotone: fp32
    // subtract, multiply by a positive scale and truncate never invert an order; equal scores
    // share a bin; NaN -> bin 0).  Float keys crowd a few leading bits, linear bins do not,
    // so plain shared atomics suffice.  Skipped (single "bin") for non-finite or equal ends.
    int kk = K, cnt = ncand;                    // still to take / members of the threshold bin
    const float vmin = key_to_score(kmn), vmax = key_to_score(kmx);
    const bool lin = kmn <= kmx && isfinite(vmin) && isfinite(vmax) && vmax > vmin && isfinite(vmax - vmin) &&
                     kk != cnt && cnt > kTieList;
    const float scale = lin ? 256.0f / (vmax - vmin) : 0.f;
    auto bin_of = [&](uint32_t key) {
        if (!lin || key == 0u) return 0;
        const int b = (int)((key_to_score(key) - vmin) * scale);
        return b > 255 ? 255 : b;
    };
    auto bin_at = [&](int i) { return lin ? (int)sbin[i] : 0; };   // i in [c_lo, c_hi)
    int bstar = 0;
    if (lin) {
        int* hb = sm.hist[1];
        if (tid < 256) hb[tid] = 0;
        __syncthreads();
        for (int i = c_lo + tid; i < c_hi; i += NT) {
            const int b = bin_of(skey[i]);
            sbin[i] = (uint8_t)b;
            atomicAdd(&hb[b], 1);
        }
        cl_sync<CL>();
        if (tid < 256) {
            int t = 0;
#pragma unroll
            for (int c = 0; c < CL; ++c) t += cl_remote<CL>(hb, c)[tid];
            sm.tot[tid] = t;
        }
        __syncthreads();
        if (warp == 0) pick_digit(sm, 256, kk, lane);
        __syncthreads();
        bstar = sm.digit;
        if (tid == 0) EXP_STAMP(p.exp_trace, ((bi * gridDim.y + blockIdx.y) * CL + crank), 3);
        kk -= sm.above;
        cnt = sm.cnt;
    }
    // ---- compact the threshold bin's members and the keys above it (when they fit; bit 31 of
    // the index marks "above") and take the members' key range
    kmn = 0xFFFFFFFFu;
    kmx = 0u;
    for (int i0 = (c_lo & ~31) + warp * 32; i0 < c_hi; i0 += NT) {
        const int i = i0 + lane;
        const bool inr = i >= c_lo && i < c_hi;
        const uint32_t key = inr ? skey[i] : 0u;
        const int b = inr ? bin_at(i) : -1;
        const bool in = inr && b >= bstar;
        if (inr && b == bstar) {
            kmn = min(kmn, key);
            kmx = max(kmx, key);
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, in);
        int wbase = 0;
        if (lane == 0 && bal) wbase = atomicAdd(&sm.ncomp, __popc(bal));
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
        const int slot = wbase + __popc(bal & ((1u << lane) - 1u));
        if (in && slot < kListCap) comp[slot] = make_uint2(key, (uint32_t)i | (b > bstar ? 0x80000000u : 0u));
    }
    cta_minmax<CL>(kmn, kmx, sm);                 // contains the barriers that publish ncomp
    if (tid == 0) EXP_STAMP(p.exp_trace, ((bi * gridDim.y + blockIdx.y) * CL + crank), 4);
    bool compacted = sm.ncomp <= kListCap;        // uniform over the CTA
    // ---- clusters: when the cluster's compacted lists fit one list, rank 0 gathers them (ids
    // made cluster-global) and finishes alone, with no further cluster barriers
    bool local = false;
    int64_t gbase = base;                         // id of local position 0 in the current lists
    if constexpr (CL > 1) {
        int tot_c = 0;
        bool fit = true;
#pragma unroll
        for (int c = 0; c < CL; ++c) {
            const int m = *cl_remote<CL>(&sm.ncomp, c);
            tot_c += m;
            fit = fit && m <= kListCap;
        }
        // every later branch reads the other ranks' shared memory under the same layout, so
        // "compacted" must be one decision for the whole cluster: all ranks' lists fit
        compacted = fit;
        if (fit && tot_c <= kListCap && K <= kTakeMax) {   // uniform over the cluster
            if (crank == 0) {
                int o = sm.ncomp;                 // rank 0's own entries stay (its base is 0)
                for (int c = 1; c < CL; ++c) {
                    const uint2* rc = cg::this_cluster().map_shared_rank(comp, c);
                    const int m = *cl_remote<CL>(&sm.ncomp, c);
                    const uint32_t add = (uint32_t)c * (uint32_t)span;   // ids < 2^31: flag bit kept
                    for (int j = tid; j < m; j += NT) {
                        uint2 e = rc[j];
                        e.y += add;
                        comp[o + j] = e;
                    }
                    o += m;
                }
            }
            cl_sync<CL>();                        // remote lists read: the other ranks are done
            if (crank != 0) return;
            if (tid == 0) sm.ncomp = tot_c;
            __syncthreads();
            local = true;
            compacted = true;
            gbase = 0;
        }
    }
    const int ncl = local ? 1 : CL;               // CTAs whose shared memory is still consulted
    auto csync = [&]() {
        if (local) __syncthreads();
        else cl_sync<CL>();
    };
    const uint32_t diff = kmn ^ kmx;
    int lo = (kk != cnt && cnt > kTieList && diff) ? 32 - __clz(diff) : 0;   // bits [0, lo) still to resolve
    uint32_t mask = lo == 32 ? 0u : ~((1u << lo) - 1u);
    uint32_t prefix = kmn & mask;
    if (kk == cnt || cnt <= kTieList) {           // the bin decides by itself: no key digits
        mask = 0u;
        prefix = 0u;
    }
    int mode;
    // ---- radix digits of the members' keys, most significant first
#pragma unroll 1
    for (int pass = 0;; ++pass) {
        if (kk == cnt) { mode = kModeWhole; break; }
        if (cnt <= kTieList) { mode = kModeList; break; }
        if (lo == 0) { mode = kModeEqual; break; }
        const int width = min(8, lo), shift = lo - width, nbins = 1 << width;
        int* hb = sm.hist[pass & 1];
        if (tid < 256) hb[tid] = 0;
        __syncthreads();
        if (compacted) {
            const int nc = sm.ncomp;
            for (int j0 = warp * 32; j0 < nc; j0 += NT) {
                const int j = j0 + lane;
                const uint2 e = j < nc ? comp[j] : make_uint2(0u, 0x80000000u);
                warp_hist_add(hb, (e.x >> shift) & (uint32_t)(nbins - 1), !(e.y >> 31) && (e.x & mask) == prefix);
            }
        } else {
            for (int i0 = (c_lo & ~31) + warp * 32; i0 < c_hi; i0 += NT) {
                const int i = i0 + lane;
                const uint32_t key = skey[i];
                warp_hist_add(hb, (key >> shift) & (uint32_t)(nbins - 1),
                              i >= c_lo && i < c_hi && bin_at(i) == bstar && (key & mask) == prefix);
            }
        }
        csync();
        if (tid < nbins) {
            int t = 0;
#pragma unroll
            for (int c = 0; c < ncl; ++c) t += cl_remote<CL>(hb, c)[tid];
            sm.tot[tid] = t;
        }
        __syncthreads();
        if (warp == 0) pick_digit(sm, nbins, kk, lane);
        __syncthreads();
        prefix |= (uint32_t)sm.digit << shift;
        mask |= (uint32_t)(nbins - 1) << shift;
        kk -= sm.above;
        cnt = sm.cnt;
        lo = shift;
    }
    if (tid == 0) EXP_STAMP(p.exp_trace, ((bi * gridDim.y + blockIdx.y) * CL + crank), 5);
    // ---- LIST: the <= 32 threshold-bin members of the cluster, ranked by (key desc, id asc)
    if (mode == kModeList) {
        auto add = [&](uint32_t key, int i) {
            const int slot = atomicAdd(&sm.lcount, 1);
            sm.lkey[slot] = key;
            sm.lid[slot] = (int32_t)(gbase + i);
        };
        if (compacted) {
            for (int j = tid; j < sm.ncomp; j += NT)
                if (!(comp[j].y >> 31) && (comp[j].x & mask) == prefix) add(comp[j].x, (int)comp[j].y);
        } else {
            for (int i = c_lo + tid; i < c_hi; i += NT)
                if (bin_at(i) == bstar && (skey[i] & mask) == prefix) add(skey[i], i);
        }
        csync();
    }
    auto bin_rank = [&](uint32_t key, int32_t id) {   // members beating (key, id)
        int rank = 0;
#pragma unroll 1
        for (int c = 0; c < ncl; ++c) {
            TopkShared* rs = cl_remote<CL>(&sm, c);
            const int m = rs->lcount;
            for (int j = 0; j < m; ++j) {
                const uint32_t kj = rs->lkey[j];
                rank += (kj > key || (kj == key && rs->lid[j] < id)) ? 1 : 0;
            }
        }
        return rank;
    };
    // stage 1 (index) writes per request id: concurrent chains of one step never share rows
    int32_t* ids_out = out_ids + ((int64_t)(p.sel_mode == 1 ? r : bi) * p.Hkv + h) * ostride;
    float* sc_out = out_scores ? out_scores + ((int64_t)bi * p.Hkv + h) * ostride : nullptr;
    bool s_ready = false;                         // fused: S[] of the resolve already in smem
    if (compacted && (mode != kModeEqual || local) && K <= kTakeMax) {
        // ---- emission from the compacted list: every taken id is in it (above the bin, or a
        // taken member); its output position = number of taken ids (cluster-wide) below it
        if (tid == 0) sm.ntake = 0;
        __syncthreads();
        const int nc = sm.ncomp;
        for (int j = tid; j < nc; j += NT) {
            const uint2 e = comp[j];
            const int i = (int)(e.y & 0x7FFFFFFFu);
            bool take = e.y >> 31;
            if (!take) {
                const uint32_t km = e.x & mask;
                if (km > prefix || (km == prefix && mode == kModeWhole)) {
                    take = true;
                } else if (km == prefix && mode == kModeList) {
                    take = bin_rank(e.x, (int32_t)(gbase + i)) < kk;
                } else if (km == prefix) {        // kModeEqual (local finish only): lowest ids first
                    int r = 0;
                    for (int u = 0; u < nc; ++u) {
                        const uint2 f = comp[u];
                        r += (!(f.y >> 31) && (f.x & mask) == prefix && (int)(f.y & 0x7FFFFFFFu) < i) ? 1 : 0;
                    }
                    take = r < kk;
                }
            }
            if (take) sm.take[atomicAdd(&sm.ntake, 1)] = (int32_t)(gbase + i);
        }
        csync();
        // gather the cluster's taken ids locally (K of them), then rank by id
        int off = 0, tot = 0;
#pragma unroll
        for (int c = 0; c < ncl; ++c) {
            const int m = *cl_remote<CL>(&sm.ntake, c);
            off += c < crank ? m : 0;
            tot += m;
        }
        int32_t* all = reinterpret_cast<int32_t*>(comp);   // comp is no longer needed
        __syncthreads();
        {
            int o = 0;
            for (int c = 0; c < ncl; ++c) {
                const TopkShared* rs = cl_remote<CL>(&sm, c);
                const int m = rs->ntake;
                for (int j = tid; j < m; j += NT) all[o + j] = rs->take[j];
                o += m;
            }
        }
        __syncthreads();
        for (int j = tid; j < sm.ntake; j += NT) {
            const int32_t id = all[off + j];
            int pos = 0;
            for (int u = 0; u < tot; ++u) pos += all[u] < id ? 1 : 0;
            ids_out[pos] = id;
            if (sc_out) sc_out[pos] = __ldcg(sc + (id - base));
        }
        if (RESOLVE && crank == 0 && 2 * (int)fa.rb.nkeys + K <= span) {
            // hand the sorted selection to the resolve in shared memory (its S[] slot; the
            // keys are dead, `all` lies beyond it): no global re-read, no validation needed
            int32_t* S = reinterpret_cast<int32_t*>(skey) + 2 * fa.rb.nkeys;
            for (int j = tid; j < tot; j += NT) {
                const int32_t id = all[j];
                int pos = 0;
                for (int u = 0; u < tot; ++u) pos += all[u] < id ? 1 : 0;
                S[pos] = id;
            }
            s_ready = true;
        }
    } else {
    // ---- emission.  Warp w owns positions [w0, w1) and walks them in 32-wide strips: pre-pass
    // counts (above, bin members), cluster-wide exclusive offsets in position order, then
    // ballots place every taken id at its ascending output position.
    const int per_w = span / (NT / 32);
    const int w0 = max(warp * per_w, c_lo), w1 = min((warp + 1) * per_w, c_hi);
    auto classify = [&](int i, bool& gt, bool& eq) {   // above the threshold / in it
        const bool in = i >= w0 && i < w1;
        const uint32_t key = in ? skey[i] : 0u;
        const int b = in ? bin_at(i) : 0;
        gt = in && (b > bstar || (b == bstar && (key & mask) > prefix));
        eq = in && b == bstar && (key & mask) == prefix;
    };
    int cgt = 0, ceq = 0;
    for (int i0 = warp * per_w; i0 < w1; i0 += 32) {
        bool gt, eq;
        classify(i0 + lane, gt, eq);
        cgt += __popc(__ballot_sync(0xffffffffu, gt));
        ceq += __popc(__ballot_sync(0xffffffffu, eq));
    }
    if (lane == 0) {
        sm.wcnt[0][warp] = cgt;
        sm.wcnt[1][warp] = ceq;
    }
    __syncthreads();
    if (warp < 2) {                               // warp 0: "above" offsets, warp 1: bin offsets
        const int v = lane < NT / 32 ? sm.wcnt[warp][lane] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        sm.woff[warp][lane] = incl - v;
        if (lane == 31) sm.ctot[warp] = incl;
    }
    csync();
    int before_gt = 0, before_eq = 0;
#pragma unroll
    for (int c = 0; c < ncl; ++c) {
        if (c < crank) {
            before_gt += *cl_remote<CL>(&sm.ctot[0], c);
            before_eq += *cl_remote<CL>(&sm.ctot[1], c);
        }
    }
    // position of a taken id: ids above the bin before it + taken bin members before it
    int gt_before = before_gt + sm.woff[0][warp];     // above-bin keys before this strip
    int eq_before = before_eq + sm.woff[1][warp];     // bin members before this strip (position order)
    int taken_eq_before = 0;                          // LIST mode: taken bin members before this strip
    if (mode == kModeList) {
        // taken bin members at positions before this warp's range (ids ascend with positions)
        int t = 0;
        for (int c = 0; c < ncl; ++c) {
            TopkShared* rs = cl_remote<CL>(&sm, c);
            for (int j = lane; j < rs->lcount; j += 32) {
                const int32_t id = rs->lid[j];
                if (id < base + warp * per_w && bin_rank(rs->lkey[j], id) < kk) ++t;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        taken_eq_before = t;
    }
    for (int i0 = warp * per_w; i0 < w1; i0 += 32) {
        const int i = i0 + lane;
        bool gt, eq;
        classify(i, gt, eq);
        const uint32_t bgt = __ballot_sync(0xffffffffu, gt), beq = __ballot_sync(0xffffffffu, eq);
        const uint32_t lt = (1u << lane) - 1u;
        bool take_eq = false;
        if (mode == kModeWhole) take_eq = eq;
        else if (mode == kModeEqual) take_eq = eq && eq_before + __popc(beq & lt) < kk;
        else if (eq) take_eq = bin_rank(skey[i], (int32_t)(gbase + i)) < kk;
        const uint32_t btk = __ballot_sync(0xffffffffu, take_eq);
        const int eq_taken_before = mode == kModeWhole ? eq_before
                                  : mode == kModeEqual ? min(eq_before, kk)
                                                       : taken_eq_before;
        if (gt || take_eq) {
            const int pos = gt_before + eq_taken_before + __popc((bgt | btk) & lt);
            ids_out[pos] = (int32_t)(gbase + i);
            if (sc_out) sc_out[pos] = __ldcg(sc + i);
        }
        gt_before += __popc(bgt);
        eq_before += __popc(beq);
        taken_eq_before += __popc(btk);
    }
    }
    if (tid == 0) EXP_STAMP(p.exp_trace, ((bi * gridDim.y + blockIdx.y) * CL + crank), 6);
    if constexpr (!RESOLVE) {
        griddep_launch();
        if (CL > 1 && !local) cl_sync<CL>();     // remote readers of this CTA's shared memory are done
    } else {
        // every CTA's ids are written (cluster barrier: release / acquire) and no CTA reads
        // another's shared memory any more; rank 0 resolves and fetches
        csync();
        if (crank != 0) return;
        uint8_t* smraw = reinterpret_cast<uint8_t*>(skey);
        const int nm = resolve_main(p, fa.rb, bi, h, out_ids, fa.out_attn, smraw, rsm, true, s_ready);
        if (nm > 0 && fa.host_store) {
            const int32_t* S = reinterpret_cast<const int32_t*>(reinterpret_cast<uint64_t*>(smraw) + fa.rb.nkeys);
            gather_segment(p, bi, h, S + 2 * fa.rb.kmax, S + 3 * fa.rb.kmax, nm, fa.host_store, fa.slots, 0, 1);
        }
    }
}

template <int CL, int NT, int V, bool RESOLVE>
__global__ void __launch_bounds__(NT, 1) select_kernel(FuseArgs fa, StepParams p, const uint16_t* __restrict__ q,
                                                       const uint16_t* __restrict__ summ, float* __restrict__ scores,
                                                       const int32_t* __restrict__ ntok, int kpt,
                                                       int32_t* __restrict__ out_ids, float* __restrict__ out_scores) {
    const int exp_unit = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    if (threadIdx.x == 0) EXP_STAMP(p.exp_trace, exp_unit, 0);
    (void)exp_unit;
    select_body<CL, NT, V, RESOLVE>(fa, p, q, summ, scores, ntok, kpt, out_ids, out_scores);   // CTA-uniform returns
#ifdef KVD_EXPERIMENTS
    __syncthreads();
    if (threadIdx.x == 0) EXP_STAMP(p.exp_trace, exp_unit, 7);
#endif
    if (p.kt_slots) {
        __syncthreads();
        if (threadIdx.x == 0)
            kt_end(p.kt_slots, p.kt_acc, p.kt_base + kKtSelect, kKtSelect, (unsigned long long)gridDim.x * gridDim.y * gridDim.z);
    }
}


// ------------------------------------------------------------------ rank_kernel
// The select call's second kernel (behind score_kernel, PDL): one thread-block cluster of CL
// CTAs x NT threads per segment ranks the segment's scores from L2 -- keys to shared memory,
// select_fast (per-CTA thresholds, one cluster barrier, rank-0 merge), then, fused, the resolve
// and the miss fetch on rank 0.  It carries only that path (no scoring loop, no general top-k):
// every phase is latency-bound, and a kernel of this size keeps its code in the instruction
// cache (the self-scoring select_kernel above is ~350 KiB of SASS; its phases stalled mostly on
// instruction fetch, ncu).
template <int CL, int NT, bool RESOLVE>
__global__ void __launch_bounds__(NT, 1) rank_kernel(FuseArgs fa, StepParams p, float* __restrict__ scores,
                                                     const int32_t* __restrict__ ntok, int kpt,
                                                     int32_t* __restrict__ out_ids, float* __restrict__ out_scores) {
    extern __shared__ __align__(16) uint32_t skey[];   // [span] keys | [kRankList] | [CL * K] candidates
    __shared__ ResolveShared rsm;
    const int crank = CL > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const int tid = threadIdx.x;
    const int h = p.h0 + blockIdx.y, bi = blockIdx.z;
    const int r = p.req[bi];
    const int span = NT * kpt;
    const int64_t base = (int64_t)crank * span;
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    // the launch's view: the segment's blocks (pinned excluded, k = p.k), or -- stage 1 of the
    // hierarchical index (R27) -- its centroids (no pinned; K = min(nc, max(ceil(4k/ratio),
    // k + pinned)), ids written with stride sel_stride)
    SegGeom g = seg_geom(ntok[r], p.P, p.sink_tokens, p.local_tokens);
    int K = p.k, ostride = p.k;
    if (p.sel_mode == 1) {
        const int nc = p.sel_count[seg];
        const int pin = g.sink_end + (g.nb - g.local_begin);
        const int f = (kIdxFanout * p.k + p.sel_ratio - 1) / p.sel_ratio;
        K = min(nc, max(f, p.k + pin));
        ostride = p.sel_stride;
        g.n = nc;
        g.nb = nc;
        g.sink_end = 0;
        g.local_begin = nc;
    }
    auto clampi = [](int64_t x, int64_t lo_, int64_t hi_) { return (int)(x < lo_ ? lo_ : x > hi_ ? hi_ : x); };
    const int nbv = clampi((int64_t)g.nb - base, 0, span);
    const int c_lo = clampi(g.sink_end - base, 0, nbv);
    const int c_hi = clampi(g.local_begin - base, 0, nbv);
    const int unit = (bi * gridDim.y + blockIdx.y) * CL + crank;
    (void)unit;
    if (tid == 0) EXP_STAMP(p.exp_trace, unit, 0);
    if (RESOLVE && crank == 0) resolve_pre(p, fa.rb, bi, h, rsm);
    griddep_wait();                                // the scores come from score_kernel
    if (p.early_trigger == 1) griddep_launch();
    if (tid == 0) kt_begin(p.kt_slots, p.kt_base + kKtSelect);
    if (tid == 0) EXP_STAMP(p.exp_trace, unit, 1);
    // ---- this CTA's scores -> monotone keys in shared memory (16-byte loads; base and the row
    // pitch are multiples of 4), and the candidates' key range
    const float4* s4 = reinterpret_cast<const float4*>(scores + seg * p.nb_pad + base);
    uint32_t kmn = 0xFFFFFFFFu, kmx = 0u;
#pragma unroll 1
    for (int i4 = tid; 4 * i4 < nbv; i4 += NT) {
        const float4 x = __ldcg(s4 + i4);
        const uint4 k4 = make_uint4(score_key32(x.x), score_key32(x.y), score_key32(x.z), score_key32(x.w));
        const uint32_t kv[4] = {k4.x, k4.y, k4.z, k4.w};
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int i = 4 * i4 + v;
            if (i >= c_lo && i < c_hi && kv[v] != 0u) {
                kmn = min(kmn, kv[v]);
                kmx = max(kmx, kv[v]);
            }
        }
        *reinterpret_cast<uint4*>(&skey[4 * i4]) = k4;
    }
    __syncthreads();
    select_fast<CL, RESOLVE>(fa, p, g, K, ostride, base, span, crank, c_lo, c_hi, kmn, kmx, skey, seg, bi, h, r,
                             scores, out_ids, out_scores, rsm);   // CTA-uniform returns
#ifdef KVD_EXPERIMENTS
    __syncthreads();
    if (tid == 0) EXP_STAMP(p.exp_trace, unit, 7);
#endif
    if (p.kt_slots) {
        __syncthreads();
        if (tid == 0)
            kt_end(p.kt_slots, p.kt_acc, p.kt_base + kKtSelect, kKtSelect, (unsigned long long)gridDim.x * gridDim.y * gridDim.z);
    }
}

template <int CL, int NT, bool RESOLVE>
inline cudaError_t launch_rank_k(kvd_cache* c, const StepParams& p, float* scores, int kpt, int32_t* out_ids,
                                 float* out_scores, const FuseArgs& fa, cudaStream_t s) {
    const int64_t kb = p.sel_mode == 1 ? c->m_max : p.k;
    const int64_t span = (int64_t)NT * kpt;
    FuseArgs f2 = fa;
    f2.fast = 1;
    size_t smem = (size_t)span * 4 + (size_t)kRankList * 8 + (CL > 1 ? 8 * (size_t)CL * std::min(kb, span) : 0);
    if (RESOLVE) {
        smem = std::max(smem, resolve_smem_bytes(fa.rb.nkeys, c->kmax, c->nb_pad));
        f2.sel_off = (uint32_t)((smem + 15) / 16 * 16);
        smem = f2.sel_off + 4 * (size_t)kb;
    }
    static size_t smem_set[64] = {};
    const int dev = c->cfg.device & 63;
    if (smem > smem_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(rank_kernel<CL, NT, RESOLVE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        smem_set[dev] = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL, p.nh, p.B);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[3];
    int na = 0;
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
    if (CL > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = CL;
        attr[na].val.clusterDim.y = 1;
        attr[na++].val.clusterDim.z = 1;
    }
    if (RESOLVE && fa.host_store) {               // the host-link fetch is inside: schedule it first
        attr[na].id = cudaLaunchAttributePriority;
        attr[na++].val.priority = c->prio_hi;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    count_launch();
    return cudaLaunchKernelEx(&cfg, rank_kernel<CL, NT, RESOLVE>, f2, p, scores,
                              (const int32_t*)c->ntok_dev + (int64_t)p.layer * c->R, kpt, out_ids, out_scores);
}

template <int NT, bool RESOLVE>
cudaError_t launch_rank_nt(kvd_cache* c, const StepParams& p, float* scores, int cl, int kpt, int32_t* out_ids,
                           float* out_scores, const FuseArgs& fa, cudaStream_t s) {
    switch (cl) {
        case 1: return launch_rank_k<1, NT, RESOLVE>(c, p, scores, kpt, out_ids, out_scores, fa, s);
        case 2: return launch_rank_k<2, NT, RESOLVE>(c, p, scores, kpt, out_ids, out_scores, fa, s);
        case 4: return launch_rank_k<4, NT, RESOLVE>(c, p, scores, kpt, out_ids, out_scores, fa, s);
        default: return launch_rank_k<8, NT, RESOLVE>(c, p, scores, kpt, out_ids, out_scores, fa, s);
    }
}

template <int CL, int NT, int V, bool RESOLVE>
inline cudaError_t launch_select_k(kvd_cache* c, const StepParams& p, const uint16_t* q, const uint16_t* mat,
                                   float* scores, int kpt, int32_t* out_ids, float* out_scores, const FuseArgs& fa,
                                   cudaStream_t s) {
    const int64_t kb = p.sel_mode == 1 ? c->m_max : p.k;          // most ids a segment selects
    FuseArgs f2 = fa;
    f2.fast = select_fast_ok(CL, (int64_t)NT * kpt, kb) ? 1 : 0;
    size_t smem = select_smem_bytes(NT, kpt, CL, kb);
    if (RESOLVE) {
        smem = std::max(smem, resolve_smem_bytes(fa.rb.nkeys, c->kmax, c->nb_pad));
        f2.sel_off = (uint32_t)((smem + 15) / 16 * 16);
        smem = f2.sel_off + 4 * (size_t)kb;
    }
    // opt in to the largest dynamic size this instantiation has been launched with (per device
    // ordinal: the attribute is per device)
    static size_t smem_set[64] = {};
    const int dev = c->cfg.device & 63;
    if (smem > smem_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(select_kernel<CL, NT, V, RESOLVE>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        smem_set[dev] = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL, p.nh, p.B);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[3];
    int na = 0;
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
    if (CL > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = CL;
        attr[na].val.clusterDim.y = 1;
        attr[na++].val.clusterDim.z = 1;
    }
    if (RESOLVE && fa.host_store) {               // the host-link fetch is inside: schedule it first
        attr[na].id = cudaLaunchAttributePriority;
        attr[na++].val.priority = c->prio_hi;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    count_launch();
    return cudaLaunchKernelEx(&cfg, select_kernel<CL, NT, V, RESOLVE>, f2, p, q, mat, scores,
                              (const int32_t*)c->ntok_dev + (int64_t)p.layer * c->R, kpt, out_ids, out_scores);
}

template <int NT, bool RESOLVE>
cudaError_t launch_select_nt(kvd_cache* c, const StepParams& p, const uint16_t* q, const uint16_t* mat, float* scores,
                             int cl, int kpt, int v, int32_t* out_ids, float* out_scores, const FuseArgs& fa,
                             cudaStream_t s) {
#define KVD_SEL_CASE(CLV)                                                                                       \
    case CLV:                                                                                                   \
        return v == 8 ? launch_select_k<CLV, NT, 8, RESOLVE>(c, p, q, mat, scores, kpt, out_ids, out_scores, fa, s)           \
             : v == 4 ? launch_select_k<CLV, NT, 4, RESOLVE>(c, p, q, mat, scores, kpt, out_ids, out_scores, fa, s)           \
                      : launch_select_k<CLV, NT, 2, RESOLVE>(c, p, q, mat, scores, kpt, out_ids, out_scores, fa, s);
    switch (cl) {
        KVD_SEL_CASE(1)
        KVD_SEL_CASE(2)
        KVD_SEL_CASE(4)
        default:
            KVD_SEL_CASE(8)
    }
#undef KVD_SEL_CASE
}

// explicit instantiations: k_select_nt512.cu, k_select_nt1024.cu (compiled in parallel)
extern template cudaError_t launch_select_nt<512, false>(kvd_cache*, const StepParams&, const uint16_t*, const uint16_t*,
    float*, int, int, int, int32_t*, float*, const FuseArgs&, cudaStream_t);
extern template cudaError_t launch_select_nt<512, true>(kvd_cache*, const StepParams&, const uint16_t*, const uint16_t*,
    float*, int, int, int, int32_t*, float*, const FuseArgs&, cudaStream_t);
extern template cudaError_t launch_select_nt<1024, false>(kvd_cache*, const StepParams&, const uint16_t*, const uint16_t*,
    float*, int, int, int, int32_t*, float*, const FuseArgs&, cudaStream_t);
extern template cudaError_t launch_select_nt<1024, true>(kvd_cache*, const StepParams&, const uint16_t*, const uint16_t*,
    float*, int, int, int, int32_t*, float*, const FuseArgs&, cudaStream_t);
// k_rank.cu
extern template cudaError_t launch_rank_nt<512, false>(kvd_cache*, const StepParams&, float*, int, int, int32_t*, float*,
                                                      const FuseArgs&, cudaStream_t);
extern template cudaError_t launch_rank_nt<512, true>(kvd_cache*, const StepParams&, float*, int, int, int32_t*, float*,
                                                     const FuseArgs&, cudaStream_t);
extern template cudaError_t launch_rank_nt<1024, false>(kvd_cache*, const StepParams&, float*, int, int, int32_t*, float*,
                                                       const FuseArgs&, cudaStream_t);
extern template cudaError_t launch_rank_nt<1024, true>(kvd_cache*, const StepParams&, float*, int, int, int32_t*, float*,
                                                      const FuseArgs&, cudaStream_t);

}  // namespace kvd
