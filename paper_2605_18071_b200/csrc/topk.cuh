// topk.cuh — CTA-local building blocks of row (a2) top-k block selection:
// the K-th largest rank key of a set of blocks and the order-preserving emission of every
// block at or above it.
//
// A block's rank key is its 32-bit monotone score key (common.cuh score_key32: -0 == +0,
// NaN lowest) in the high word and ~id in the low word, so one unsigned 64-bit comparison is
// the selection order "score descending, then block id ascending" (R10).  The
// top-k set is then exactly {blocks with rank key >= T}, T the K-th largest rank key, and
// emitting those blocks in position order yields the ids ascending (R25) with no sort.
//
// T is found by a first digit of 256 bins linear in the score value over the blocks'
// [min, max] (float keys crowd a few leading bits; linear bins spread them), then 8-bit
// radix digits of the threshold bin's rank keys from their highest differing bit (exact
// ties between scores resolve on the id bits), until the K-th is isolated: the remaining
// group is taken whole (T = its minimum) or holds <= 32 keys (ranked inside one warp).
#pragma once
#include "common.cuh"

namespace kvd {

__device__ __forceinline__ uint64_t rank_key(uint32_t key, uint32_t id) {
    return ((uint64_t)key << 32) | (uint64_t)(0xFFFFFFFFu - id);
}
__device__ __forceinline__ uint32_t rank_id(uint64_t rk) { return 0xFFFFFFFFu - (uint32_t)rk; }

// inverse of score_key32 for non-NaN keys (key 0 = NaN -> -inf here)
__device__ __forceinline__ float key_to_score(uint32_t key) {
    if (key == 0u) return -INFINITY;
    return __uint_as_float((key >> 31) ? (key & 0x7FFFFFFFu) : ~key);
}

constexpr int kRankList = 4096;     // threshold-bin members compacted per CTA (rank keys, 8 B each)

struct KthShared {
    int hist[2][256];                 // first digit: hist[0]; radix passes alternate
    uint32_t kmin[32], kmax[32];      // per-warp partials of the score-key range
    uint64_t wmin[32], wmax[32];      // per-warp partials of rank-key ranges
    uint64_t small[32];               // a final group of <= 32 rank keys
    int wcnt[33];
    int digit, above, cnt;
    int nlist, nsmall;
    uint64_t T;
};

// The blocks of a CTA's span: position i in [lo, hi) holds score key key[i]; its id is gbase + i.
struct SpanView {
    const uint32_t* key;
    int lo, hi;
    uint32_t gbase;
    __device__ __forceinline__ uint32_t k32(int i) const { return key[i]; }
    __device__ __forceinline__ uint64_t rk(int i) const { return rank_key(key[i], gbase + (uint32_t)i); }
};
// A list of rank keys (the cluster's candidates gathered on rank 0), positions [0, n).
struct ListView {
    const uint64_t* r;
    int lo, hi;
    __device__ __forceinline__ uint32_t k32(int i) const { return (uint32_t)(r[i] >> 32); }
    __device__ __forceinline__ uint64_t rk(int i) const { return r[i]; }
};

// warp 0: the bin d (counted from the top) holding the kk-th largest member of hist[0, nbins);
// lane l owns bins nbins-1-(8l+j), j < 8.  Writes sh.digit, sh.above (members in higher bins),
// sh.cnt.
__device__ __forceinline__ void kth_pick(const int* hist, KthShared& sh, int nbins, int kk) {
    const int lane = threadIdx.x & 31;
    int c8[8], t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int d = nbins - 1 - (8 * lane + j);
        c8[j] = d >= 0 ? hist[d] : 0;
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
                sh.digit = nbins - 1 - (8 * lane + j);
                sh.above = above;
                sh.cnt = c8[j];
                break;
            }
            above += c8[j];
        }
    }
}

__device__ __forceinline__ uint32_t warp_min32(uint32_t x) { return __reduce_min_sync(0xffffffffu, x); }
__device__ __forceinline__ uint32_t warp_max32(uint32_t x) { return __reduce_max_sync(0xffffffffu, x); }
__device__ __forceinline__ uint64_t warp_min64(uint64_t x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = min(x, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)x, o));
    return x;
}
__device__ __forceinline__ uint64_t warp_max64(uint64_t x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = max(x, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)x, o));
    return x;
}

// The K-th largest rank key T of the view's blocks [v.lo, v.hi) (0 < K < hi - lo): exactly K
// blocks have rank key >= T.  kmn / kmx: this thread's partial min / max of the blocks'
// non-NaN score keys (0xFFFFFFFF / 0 if none).  `list`: kRankList rank keys of shared scratch.
// Every thread of the CTA calls it; the result is CTA-uniform.  Barrier phases: key range,
// first-digit histogram, its pick, member compaction (with the members' rank-key range), then
// two per radix digit, and one to rank a final group of <= 32.
template <class View>
__device__ __forceinline__ uint64_t kth_largest(const View v, int K, uint32_t kmn, uint32_t kmx,
                                                uint64_t* __restrict__ list, KthShared& sh,
                                                unsigned long long* trace = nullptr, int unit = 0) {
    (void)trace;
    (void)unit;
    const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = NT >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    // ---- score-key range (one barrier; the histograms are cleared under it)
    kmn = __reduce_min_sync(0xffffffffu, kmn);
    kmx = __reduce_max_sync(0xffffffffu, kmx);
    if (lane == 0) {
        sh.kmin[warp] = kmn;
        sh.kmax[warp] = kmx;
    }
#pragma unroll 1
    for (int i = tid; i < 512; i += NT) (&sh.hist[0][0])[i] = 0;
    if (tid == 0) {
        sh.nlist = 0;
        sh.nsmall = 0;
    }
    __syncthreads();
    kmn = warp_min32(lane < nw ? sh.kmin[lane] : 0xFFFFFFFFu);   // every warp reduces the partials
    kmx = warp_max32(lane < nw ? sh.kmax[lane] : 0u);
    // ---- first digit: 256 bins linear in the score value (fp32 subtract, multiply by a positive
    // scale and truncate are monotone: equal scores share a bin; NaN -> bin 0).  Without a finite
    // non-empty range every block is in one bin.
    const float vmin = key_to_score(kmn), vmax = key_to_score(kmx);
    const bool lin = kmn < kmx && isfinite(vmin) && isfinite(vmax) && vmax > vmin && isfinite(vmax - vmin);
    const float scale = lin ? 256.0f / (vmax - vmin) : 0.f;
    auto bin_of = [&](uint32_t key) -> int {
        if (!lin || key == 0u) return 0;
        const int b = (int)((key_to_score(key) - vmin) * scale);
        return b > 255 ? 255 : b;
    };
    int kk = K, cnt = v.hi - v.lo, bstar = 0;
    if (lin) {
#pragma unroll 4
        for (int i = v.lo + tid; i < v.hi; i += NT) atomicAdd(&sh.hist[0][bin_of(v.k32(i))], 1);
        __syncthreads();
        if (warp == 0) kth_pick(sh.hist[0], sh, 256, kk);
        __syncthreads();
        bstar = sh.digit;
        kk -= sh.above;
        cnt = sh.cnt;
    }
    if (tid == 0) EXP_STAMP(trace, unit, 3);
    // ---- the threshold bin's members: compacted as rank keys when they fit; their range
    const int s0 = v.lo & ~31;
    uint64_t gmn = ~0ull, gmx = 0ull;
#pragma unroll 2
    for (int i0 = s0 + warp * 32; i0 < v.hi; i0 += NT) {
        const int i = i0 + lane;
        const bool m = i >= v.lo && i < v.hi && bin_of(v.k32(i)) == bstar;
        const uint32_t bal = __ballot_sync(0xffffffffu, m);
        if (!bal) continue;
        int wb = 0;
        if (lane == 0) wb = atomicAdd(&sh.nlist, __popc(bal));
        wb = __shfl_sync(0xffffffffu, wb, 0);
        if (m) {
            const uint64_t r = v.rk(i);
            gmn = min(gmn, r);
            gmx = max(gmx, r);
            const int slot = wb + __popc(bal & lt);
            if (slot < kRankList) list[slot] = r;
        }
    }
    gmn = warp_min64(gmn);
    gmx = warp_max64(gmx);
    if (lane == 0) {
        sh.wmin[warp] = gmn;
        sh.wmax[warp] = gmx;
    }
    __syncthreads();
    gmn = warp_min64(lane < nw ? sh.wmin[lane] : ~0ull);
    gmx = warp_max64(lane < nw ? sh.wmax[lane] : 0ull);
    if (tid == 0) EXP_STAMP(trace, unit, 4);
    const bool compacted = cnt <= kRankList;
    const int nl = compacted ? cnt : 0;
    // one pass over the group {members : (rk & mask) == prefix}; every lane of a warp iterates
    // alike (warp-collective bodies).  One loop body for every use keeps the code small.
    enum { kOpMin = 0, kOpMinMax = 1, kOpHist = 2, kOpGather = 3 };
    uint64_t mask = 0ull, prefix = 0ull;
    auto group_pass = [&](int op, int* hb, int shift, int nbins, uint64_t& mn, uint64_t& mx) {
        const int n = compacted ? nl : v.hi - s0;
#pragma unroll 1
        for (int j0 = warp * 32; j0 < n; j0 += NT) {
            const int j = j0 + lane;
            uint64_t r = 0ull;
            bool in = false;
            if (compacted) {
                if (j < nl) {
                    r = list[j];
                    in = true;
                }
            } else {
                const int i = s0 + j;
                if (i >= v.lo && i < v.hi) {
                    r = v.rk(i);
                    in = bin_of((uint32_t)(r >> 32)) == bstar;
                }
            }
            in = in && (r & mask) == prefix;
            if (op == kOpHist) {
                warp_hist_add(hb, (uint32_t)(r >> shift) & (uint32_t)(nbins - 1), in);
            } else if (op == kOpGather) {
                const uint32_t bal = __ballot_sync(0xffffffffu, in);
                if (bal) {
                    int wb = 0;
                    if (lane == 0) wb = atomicAdd(&sh.nsmall, __popc(bal));
                    wb = __shfl_sync(0xffffffffu, wb, 0);
                    if (in) sh.small[wb + __popc(bal & lt)] = r;
                }
            } else if (in) {
                mn = min(mn, r);
                if (op == kOpMinMax) mx = max(mx, r);
            }
        }
    };
    // ---- radix digits of the group, from its highest differing bit down, until the kk-th
    // largest is isolated: the group is taken whole (T = its minimum: known for the members,
    // reduced otherwise) or holds <= 32 keys (ranked in a warp)
    int pass = 0, lo = 64 - __clzll((long long)(gmn ^ gmx));
    uint64_t T;
#pragma unroll 1
    for (;;) {
        if (kk == cnt) {
            if (pass == 0) {
                T = gmn;
            } else {
                uint64_t mn = ~0ull, mx = 0ull;
                group_pass(kOpMin, nullptr, 0, 1, mn, mx);
                mn = warp_min64(mn);
                if (lane == 0) sh.wmin[warp] = mn;
                __syncthreads();
                T = warp_min64(lane < nw ? sh.wmin[lane] : ~0ull);
                __syncthreads();
            }
            break;
        }
        if (cnt <= 32) {
            uint64_t mn = 0ull, mx = 0ull;
            group_pass(kOpGather, nullptr, 0, 1, mn, mx);
            __syncthreads();
            if (warp == 0) {
                const uint64_t r = lane < cnt ? sh.small[lane] : 0ull;
                int above = 0;
#pragma unroll 4
                for (int u = 0; u < 32; ++u) above += (uint64_t)__shfl_sync(0xffffffffu, (unsigned long long)r, u) > r ? 1 : 0;
                if (lane < cnt && above == kk - 1) sh.T = r;
            }
            __syncthreads();
            T = sh.T;
            break;
        }
        // digit of `width` bits below the group's common prefix (bits >= lo)
        const int width = lo < 8 ? lo : 8, shift = lo - width, nbins = 1 << width;
        if (lo < 64) mask |= ~0ull << lo;
        prefix = gmn & mask;
        int* hb = sh.hist[1 - (pass & 1)];       // cleared (pass 0: at the start; later: below)
        {
            uint64_t mn = 0ull, mx = 0ull;
            group_pass(kOpHist, hb, shift, nbins, mn, mx);
        }
        __syncthreads();
        if (warp == 0) kth_pick(hb, sh, nbins, kk);
        else
#pragma unroll 1
            for (int i = tid - 32; i < 256; i += NT - 32) sh.hist[pass & 1][i] = 0;   // the next pass's
        __syncthreads();
        prefix |= (uint64_t)sh.digit << shift;
        mask |= (uint64_t)(nbins - 1) << shift;
        kk -= sh.above;
        cnt = sh.cnt;
        gmn = prefix;                             // the next digit's common-prefix source
        lo = shift;
        ++pass;
        __syncthreads();                          // sh.digit / above / cnt read before the next pick
    }
    return T;
}

// Order-preserving emission of the view's blocks with rank key >= T: warp w walks the
// contiguous positions [lo + w*per, lo + (w+1)*per) in 32-wide strips -- a count pass, an
// exclusive scan of the warp totals, then ballots place every block at its output position
// (ascending position == ascending id).  emit(i, pos) runs once per emitted block.
// Returns the number emitted (CTA-uniform).
template <class View, class Emit>
__device__ __forceinline__ int emit_ordered(const View v, uint64_t T, KthShared& sh, Emit&& emit) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int n = v.hi - v.lo;
    const int per = ((n + nw - 1) / nw + 31) & ~31;
    const int a = v.lo + warp * per, b = min(v.hi, a + per);
    int c = 0;
#pragma unroll 4
    for (int i0 = a; i0 < b; i0 += 32) {
        const int i = i0 + lane;
        c += __popc(__ballot_sync(0xffffffffu, i < b && v.rk(i) >= T));
    }
    if (lane == 0) sh.wcnt[warp] = c;
    __syncthreads();
    if (warp == 0) {
        const int x = lane < nw ? sh.wcnt[lane] : 0;
        int incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane < nw) sh.wcnt[lane] = incl - x;
        if (lane == 31) sh.wcnt[32] = incl;
    }
    __syncthreads();
    int pos = sh.wcnt[warp];
    const int tot = sh.wcnt[32];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll 2
    for (int i0 = a; i0 < b; i0 += 32) {
        const int i = i0 + lane;
        const bool t = i < b && v.rk(i) >= T;
        const uint32_t bal = __ballot_sync(0xffffffffu, t);
        if (t) emit(i, pos + __popc(bal & lt));
        pos += __popc(bal);
    }
    __syncthreads();                              // sh.wcnt reusable
    return tot;
}

}  // namespace kvd
