// resolve.cuh — row (a3) resolve of one segment and row (a4) its miss gather, as device
// functions shared by resolve_kernel (k_resolve.cu) and the fused select + resolve + fetch
// kernel (k_select.cu).  Decisions follow DESIGN.md §3 R12-R13 exactly (the oracle's O6).
#pragma once
#include "common.cuh"
#include "internal.h"

namespace kvd {

constexpr int kResolveThreads = 256;

struct ResolveBufs {
    int32_t* table;
    int32_t* slot_block;
    uint32_t* last_use;
    uint8_t* phase;
    uint32_t* use_count;
    const float* scores;
    const int32_t* ntok;
    int32_t* miss;          // [R][Hkv][kmax][2]
    int32_t* miss_count;    // [R][Hkv]
    int32_t kmax;
    int64_t nkeys;          // victim-key slots in shared memory: C, or 0 for a fully resident cache
    unsigned long long* stats;
    int32_t* err;
    const int32_t* cap;     // [L][Hkv] slots a segment may use (2D window scaling, R28), or NULL: C
    // hierarchical index (R27): a block scored this step (bit set in cbits) has its exact score in
    // `scores`; any other block is ranked by its centroid's score (lookahead victim keys)
    const uint32_t* cbits;  // [seg][nb_pad / 32] this step's candidates, or NULL (flat index)
    const int32_t* cent_of; // [seg][nb_pad]
    const float* cscores;   // [seg][nc_pad]
    int64_t nc_pad;
    unsigned long long* seg_stats;   // [L][Hkv][2] (selected, misses) per layer-head, or NULL
};

__device__ __forceinline__ uint64_t victim_key(int policy, uint32_t lu, uint8_t ph, uint32_t uc, int32_t blk,
                                               float score, int32_t* err) {
    if (policy == KVD_POLICY_LRU) return ((uint64_t)lu << 32) | ((uint64_t)(ph & 1) << 31) | (uint32_t)blk;
    if (policy == KVD_POLICY_LFU) {
        if (uc > 0xFFFFu || lu >= (1u << 24) || blk >= (1 << 23)) atomicOr(err, 2);
        return ((uint64_t)min(uc, 0xFFFFu) << 48) | ((uint64_t)(lu & 0xFFFFFFu) << 24) |
               ((uint64_t)(ph & 1) << 23) | (uint32_t)blk;
    }
    return ((uint64_t)score_key32(score) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)blk);
}

// Shared state of one segment's resolve (static part; the dynamic part is smraw).
ResolveBufs resolve_bufs(kvd_cache* c, int layer);   // k_resolve.cu

struct ResolveShared {
    int scan[33];
    int hist[256];
    int bad, above;
    uint32_t digit;
    int32_t pin_slot[256];            // pinned blocks <= 256 (checked at create)
};

// pre-phase: the pinned blocks' slots (written only by kvd_load_prefix; never evicted), so it
// may run before griddepcontrol.wait and overlap the previous kernel's tail.
__device__ __forceinline__ void resolve_pre(const StepParams& p, const ResolveBufs& rb, int bi, int h,
                                            ResolveShared& rsm) {
    const int r = p.req[bi];
    const SegGeom g = seg_geom(rb.ntok[r], p.P, p.sink_tokens, p.local_tokens);
    const int32_t* table = rb.table + (((int64_t)p.layer * p.R + r) * p.Hkv + h) * p.nb_pad;
    const int ns = g.sink_end, nl = g.nb - g.local_begin;
    for (int t = threadIdx.x; t < ns + nl; t += blockDim.x)
        rsm.pin_slot[t] = table[t < ns ? t : g.local_begin + (t - ns)];
}

// dynamic smem (smraw): keys64[nkeys] | S | hitslot | M | dest | vtmp (kmax each) | inS[nwords].
// All threads of the CTA call it (blockDim a multiple of 32, <= 1024), after resolve_pre and
// griddepcontrol.wait.  Returns the miss count; M[] / dest[] (blocks / slots) stay in smraw.
__device__ inline int resolve_main(const StepParams& p, const ResolveBufs& rb, int bi, int h,
                            const int32_t* __restrict__ ids, int32_t* __restrict__ out_attn, uint8_t* smraw,
                            ResolveShared& rsm, bool launch_dependents, bool s_ready = false) {
    const int r = p.req[bi];
    const int tid = threadIdx.x;
    const SegGeom g = seg_geom(rb.ntok[r], p.P, p.sink_tokens, p.local_tokens);
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    const int64_t rs = (int64_t)r * p.Hkv + h;
    int32_t* table = rb.table + seg * p.nb_pad;
    int32_t* sb = rb.slot_block + seg * p.C;
    uint32_t* lu = rb.last_use + seg * p.C;
    uint8_t* ph = rb.phase + seg * p.C;
    uint32_t* uc = rb.use_count + seg * p.C;
    // 2D window scaling (R28): this layer-head pair's capacity; slots >= Ceff are never used
    const int64_t Ceff = rb.cap ? (int64_t)rb.cap[p.layer * p.Hkv + h] : p.C;
    const float* sc = rb.scores + seg * p.nb_pad;
    const int32_t* S_in = ids + ((int64_t)bi * p.Hkv + h) * p.k;
    int32_t* attn = out_attn + ((int64_t)bi * p.Hkv + h) * (int64_t)p.W * 2;
    const int k = p.k;
    const int nwords = (g.nb + 31) >> 5;

    uint64_t* keys = reinterpret_cast<uint64_t*>(smraw);
    int32_t* S = reinterpret_cast<int32_t*>(keys + rb.nkeys);
    int32_t* hitslot = S + rb.kmax;
    int32_t* M = hitslot + rb.kmax;
    int32_t* dest = M + rb.kmax;
    int32_t* vtmp = dest + rb.kmax;
    uint32_t* inS = reinterpret_cast<uint32_t*>(vtmp + rb.kmax);

    const int ns = g.sink_end, nl = g.nb - g.local_begin;
    // ---- 1. load + validate the selection (ascending, in range, not pinned); s_ready: the
    //         fused kernel already placed its own (valid by construction) ids in S[]
    if (tid == 0) rsm.bad = 0;
    __syncthreads();
    for (int i = s_ready ? k : tid; i < k; i += blockDim.x) {
        const int32_t b = __ldcg(&S_in[i]);
        S[i] = b;
        bool bad = b < g.sink_end || b >= g.local_begin || (i > 0 && __ldcg(&S_in[i - 1]) >= b);
        if (bad) rsm.bad = 1;
    }
    __syncthreads();
    if (rsm.bad) {
        if (tid == 0) atomicOr(rb.err, 1);
        for (int i = tid; i < p.W * 2; i += blockDim.x) attn[i] = -1;
        if (tid == 0) rb.miss_count[rs] = 0;
        return 0;
    }
    if (rb.nkeys == 0) {
        // ---- fully resident (R14): block b lives in slot b and every selected block hits -- no
        //      scans: metadata stores, counters, then the attention list
        const uint32_t step = p.step_dev ? *p.step_dev : p.step;
        for (int i = tid; i < k; i += blockDim.x) {
            const int32_t s = S[i];
            lu[s] = step;
            ph[s] = 0;
            atomicAdd(&uc[s], 1u);
        }
        if (tid == 0) {
            rb.miss_count[rs] = 0;
            atomicAdd(&rb.stats[0], (unsigned long long)k);
            atomicAdd(&rb.stats[1], (unsigned long long)k);
            atomicAdd(&rb.stats[3], (unsigned long long)(ns + nl));
            if (rb.seg_stats) atomicAdd(&rb.seg_stats[((int64_t)p.layer * p.Hkv + h) * 2], (unsigned long long)k);
        }
        if (launch_dependents) griddep_launch();
        for (int i = tid; i < p.W; i += blockDim.x) {
            int32_t b = -1;
            if (i < ns) b = i;
            else if (i < ns + k) b = S[i - ns];
            else if (i < ns + k + nl) b = g.local_begin + (i - ns - k);
            attn[2 * i] = b;
            attn[2 * i + 1] = b;
        }
        return 0;
    }
    // ---- 2. hits / misses (misses compacted in ascending order)
    int nm_total = 0;
    for (int base = 0; base < k; base += blockDim.x) {
        const int i = base + tid;
        int hs = -1;
        if (i < k) {
            hs = rb.nkeys == 0 ? S[i] : table[S[i]];   // fully resident: block b lives in slot b (R14)
            hitslot[i] = hs;
        }
        const int is_miss = (i < k && hs < 0) ? 1 : 0;
        int tot;
        const int pos = block_exclusive_scan(is_miss, rsm.scan, &tot);
        if (is_miss) {
            M[nm_total + pos] = S[i];
            hitslot[i] = -2 - (nm_total + pos);   // miss: its slot will be dest[nm_total + pos]
        }
        nm_total += tot;
    }
    const int nm = nm_total;
    // ---- 3. free slots, ascending: the first nm
    int nf = 0;
    if (nm > 0) {
        for (int base = 0; base < Ceff && nf < nm; base += blockDim.x) {
            const int64_t s = base + tid;
            const int fr = (s < Ceff && sb[s] < 0) ? 1 : 0;
            int tot;
            const int pos = block_exclusive_scan(fr, rsm.scan, &tot);
            if (fr && nf + pos < nm) dest[nf + pos] = (int32_t)s;
            nf = min(nm, nf + tot);
        }
    }
    // ---- 4. victims: the nv smallest policy keys among evictable residents
    const int nv = nm - nf;
    if (nv > 0) {
        for (int w = tid; w < nwords; w += blockDim.x) inS[w] = 0u;
        __syncthreads();
        for (int i = tid; i < k; i += blockDim.x) atomicOr(&inS[S[i] >> 5], 1u << (S[i] & 31));
        __syncthreads();
        for (int64_t s = tid; s < Ceff; s += blockDim.x) {
            const int32_t blk = sb[s];
            uint64_t key = ~0ull;
            if (blk >= 0 && blk >= g.sink_end && blk < g.local_begin && !((inS[blk >> 5] >> (blk & 31)) & 1u)) {
                float score = 0.0f;
                if (p.policy == KVD_POLICY_LOOKAHEAD) {
                    const bool exact = !rb.cbits || ((__ldcg(&rb.cbits[seg * (p.nb_pad >> 5) + (blk >> 5)]) >> (blk & 31)) & 1u);
                    score = exact ? __ldcg(&sc[blk]) : __ldcg(&rb.cscores[seg * rb.nc_pad + rb.cent_of[seg * p.nb_pad + blk]]);
                }
                key = victim_key(p.policy, lu[s], ph[s], uc[s], blk, score, rb.err);
            }
            keys[s] = key;
        }
        __syncthreads();
        // radix select: the nv-th smallest key, T (keys are unique among candidates)
        uint64_t prefix = 0, mask = 0;
        int kk = nv;
#pragma unroll 1
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int i = tid; i < 256; i += blockDim.x) rsm.hist[i] = 0;
            __syncthreads();
            for (int64_t s = tid; s < Ceff; s += blockDim.x) {
                const uint64_t key = keys[s];
                if ((key & mask) == prefix) atomicAdd(&rsm.hist[(key >> shift) & 255], 1);
            }
            __syncthreads();
            if (tid < 32) {
                int cnt[8], tot = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    cnt[i] = rsm.hist[8 * tid + i];
                    tot += cnt[i];
                }
                int incl = tot;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (tid >= o) incl += y;
                }
                int below = incl - tot;
                if (below < kk && kk <= incl) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if (below + cnt[i] >= kk) {
                            rsm.digit = (uint32_t)(8 * tid + i);
                            rsm.above = below;
                            break;
                        }
                        below += cnt[i];
                    }
                }
            }
            __syncthreads();
            prefix |= (uint64_t)rsm.digit << shift;
            mask |= 0xFFull << shift;
            kk -= rsm.above;
            __syncthreads();
        }
        const uint64_t T = prefix;
        // compact victims (key <= T) in slot order, then place them by key rank
        int nvc = 0;
        for (int base = 0; base < Ceff; base += blockDim.x) {
            const int64_t s = base + tid;
            const int isv = (s < Ceff && keys[s] <= T) ? 1 : 0;
            int tot;
            const int pos = block_exclusive_scan(isv, rsm.scan, &tot);
            if (isv && nvc + pos < nv) vtmp[nvc + pos] = (int32_t)s;
            nvc += tot;
        }
        __syncthreads();
        for (int i = tid; i < nv; i += blockDim.x) {
            const int32_t s = vtmp[i];
            const uint64_t ki = keys[s];
            int rank = 0;
            for (int j = 0; j < nv; ++j) rank += keys[vtmp[j]] < ki ? 1 : 0;
            dest[nf + rank] = s;
        }
        __syncthreads();
        for (int i = tid; i < nv; i += blockDim.x) table[sb[dest[nf + i]]] = -1;   // victims leave
    }
    __syncthreads();
    // ---- 5. admit misses, update metadata
    const uint32_t step = p.step_dev ? *p.step_dev : p.step;
    int32_t* miss_out = rb.miss + rs * (int64_t)rb.kmax * 2;
    for (int i = tid; i < nm; i += blockDim.x) {
        const int32_t b = M[i], s = dest[i];
        table[b] = s;
        sb[s] = b;
        lu[s] = step;
        ph[s] = 1;
        uc[s] = 1;
        miss_out[2 * i] = b;
        miss_out[2 * i + 1] = s;
    }
    for (int i = tid; i < k; i += blockDim.x) {
        const int32_t s = hitslot[i];
        if (s >= 0) {                             // stores only: no round trip (slots are unique)
            lu[s] = step;
            ph[s] = 0;
            atomicAdd(&uc[s], 1u);
        }
    }
    if (tid == 0) {
        rb.miss_count[rs] = nm;
        const int pinned = g.sink_end + (g.nb - g.local_begin);
        atomicAdd(&rb.stats[0], (unsigned long long)k);
        atomicAdd(&rb.stats[1], (unsigned long long)(k - nm));
        atomicAdd(&rb.stats[2], (unsigned long long)nm);
        atomicAdd(&rb.stats[3], (unsigned long long)pinned);
        atomicAdd(&rb.stats[4], (unsigned long long)nm * (unsigned long long)p.rec_bytes);
        if (rb.seg_stats) {
            unsigned long long* ss = rb.seg_stats + ((int64_t)p.layer * p.Hkv + h) * 2;
            atomicAdd(&ss[0], (unsigned long long)k);
            atomicAdd(&ss[1], (unsigned long long)nm);
        }
    }
    __syncthreads();
    if (launch_dependents) griddep_launch();
    // ---- 6. attention list: sink blocks ++ S ++ local blocks, ascending, with slots (from
    //         shared memory: hit slots, miss destinations, pinned slots; no table re-read)
    for (int i = tid; i < p.W; i += blockDim.x) {
        int32_t b = -1, s = -1;
        if (i < ns) {
            b = i;
            s = rsm.pin_slot[i];
        } else if (i < ns + k) {
            b = S[i - ns];
            const int32_t hs = hitslot[i - ns];
            s = hs >= 0 ? hs : dest[-2 - hs];
        } else if (i < ns + k + nl) {
            b = g.local_begin + (i - ns - k);
            s = rsm.pin_slot[i - k];
        }
        attn[2 * i] = b;
        attn[2 * i + 1] = s;
    }
    return nm;
}


// Arguments of a select kernel that also resolves and fetches (kvd_select_resolve_fetch).
struct FuseArgs {
    ResolveBufs rb;
    int32_t* out_attn;
    const uint8_t* host_store;    // NULL: fully resident (no misses)
    uint8_t* slots;
    int32_t fast;                 // select_kernel: per-CTA thresholds + rank-0 merge (select_fast)
    uint32_t sel_off;             // select_kernel (fused): byte offset of the selection in shared memory
};

// (a4) inside a segment's CTA: all threads copy the nm missed 8 KiB records host -> slot.
// The (record, 16-byte chunk) space is flattened and cut into nparts equal slices (one per CTA
// of the segment's cluster); every thread keeps up to 8 zero-copy loads in flight, so the whole
// slice is requested in one host-link round trip.
__device__ __forceinline__ void gather_segment(const StepParams& p, int bi, int h, const int32_t* M, const int32_t* dest,
                                               int nm, const uint8_t* __restrict__ host_store,
                                               uint8_t* __restrict__ slots, int part, int nparts) {
    const int r = p.req[bi];
    const int cpr = p.rec_bytes / 16;                       // 16-byte chunks per record (power of two)
    const int lcpr = __ffs(cpr) - 1;
    const int total = nm << lcpr;
    const int xa = (int)((int64_t)part * total / nparts), xb = (int)((int64_t)(part + 1) * total / nparts);
    const uint8_t* hbase = host_store + (((int64_t)p.host_layer * p.R + r) * p.Hkv + h) * p.nb_max * (int64_t)p.rec_bytes;
    uint8_t* sbase = slots + (((int64_t)p.layer * p.R + r) * p.Hkv + h) * p.C * (int64_t)p.rec_bytes;
    for (int x0 = xa + threadIdx.x; x0 < xb; x0 += 8 * blockDim.x) {
        int4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int x = x0 + u * blockDim.x;
            if (x < xb) {
                const int i = x >> lcpr, c = x & (cpr - 1);
                v[u] = ld_host16(reinterpret_cast<const int4*>(hbase + (int64_t)M[i] * p.rec_bytes) + c);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int x = x0 + u * blockDim.x;
            if (x < xb) {
                const int i = x >> lcpr, c = x & (cpr - 1);
                reinterpret_cast<int4*>(sbase + (int64_t)dest[i] * p.rec_bytes)[c] = v[u];
            }
        }
    }
}

}  // namespace kvd
