// k_resolve.cu — rows (a3) resolve against the GPU cache and (a4) miss gather.
//
// (a3) The paper evaluates hit/miss and updates cache metadata on the CPU
// (PAPER.md:530, 537); here it runs on the GPU, one CTA per segment, so the
// step never round-trips to the host.  Decisions follow DESIGN.md §3 R12-R13
// exactly (the oracle's O6): hits = selected blocks already resident; misses
// (ascending) take free slots (ascending), then victims = residents neither
// selected nor pinned, in ascending policy key:
//   LRU  (last_use, phase, block)               packed 32|1|31 bits
//   LFU  (use_count, last_use, phase, block)    packed 16|24|1|23 bits (bounds flagged)
//   LA   (score key ascending, block descending) 32|32 bits — "entries with the
//        lowest current-step attention scores are discarded"
// The nv smallest keys are found by an 8-pass radix select over 64-bit keys.
//
// (a4) "block-level sparse fetching ... only the blocks the queries need"
// (PAPER.md:636-639): each missed 8 KiB record is copied from the pinned,
// mapped host store into its slot by SM zero-copy 16-byte loads over PCIe.
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
    unsigned long long* stats;
    int32_t* err;
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

// dynamic smem: keys64[C] | S | hitslot | M | dest | vtmp (kmax each) | inS[nwords]
__global__ void __launch_bounds__(kResolveThreads) resolve_kernel(StepParams p, ResolveBufs rb,
                                                                  const int32_t* __restrict__ ids,
                                                                  int32_t* __restrict__ out_attn) {
    extern __shared__ __align__(16) uint8_t smraw[];
    __shared__ int scan_scratch[33];
    __shared__ int hist[256];
    __shared__ int s_bad, s_above;
    __shared__ uint32_t s_digit;
    const int bi = blockIdx.y, h = blockIdx.x;
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
    const float* sc = rb.scores + seg * p.nb_pad;
    const int32_t* S_in = ids + ((int64_t)bi * p.Hkv + h) * p.k;
    int32_t* attn = out_attn + ((int64_t)bi * p.Hkv + h) * (int64_t)p.W * 2;
    const int k = p.k;
    const int nwords = (g.nb + 31) >> 5;

    uint64_t* keys = reinterpret_cast<uint64_t*>(smraw);
    int32_t* S = reinterpret_cast<int32_t*>(keys + p.C);
    int32_t* hitslot = S + rb.kmax;
    int32_t* M = hitslot + rb.kmax;
    int32_t* dest = M + rb.kmax;
    int32_t* vtmp = dest + rb.kmax;
    uint32_t* inS = reinterpret_cast<uint32_t*>(vtmp + rb.kmax);

    // ---- 1. load + validate the selection (ascending, in range, not pinned)
    if (tid == 0) s_bad = 0;
    griddep_wait();                               // ids / scores come from select
    __syncthreads();
    for (int i = tid; i < k; i += blockDim.x) {
        const int32_t b = S_in[i];
        S[i] = b;
        bool bad = b < g.sink_end || b >= g.local_begin || (i > 0 && S_in[i - 1] >= b);
        if (bad) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0) atomicOr(rb.err, 1);
        for (int i = tid; i < p.W * 2; i += blockDim.x) attn[i] = -1;
        if (tid == 0) rb.miss_count[rs] = 0;
        return;
    }
    // ---- 2. hits / misses (misses compacted in ascending order)
    int nm_total = 0;
    for (int base = 0; base < k; base += blockDim.x) {
        const int i = base + tid;
        int hs = -1;
        if (i < k) {
            hs = table[S[i]];
            hitslot[i] = hs;
        }
        const int is_miss = (i < k && hs < 0) ? 1 : 0;
        int tot;
        const int pos = block_exclusive_scan(is_miss, scan_scratch, &tot);
        if (is_miss) M[nm_total + pos] = S[i];
        nm_total += tot;
    }
    const int nm = nm_total;
    // ---- 3. free slots, ascending: the first nm
    int nf = 0;
    if (nm > 0) {
        for (int base = 0; base < p.C && nf < nm; base += blockDim.x) {
            const int64_t s = base + tid;
            const int fr = (s < p.C && sb[s] < 0) ? 1 : 0;
            int tot;
            const int pos = block_exclusive_scan(fr, scan_scratch, &tot);
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
        for (int64_t s = tid; s < p.C; s += blockDim.x) {
            const int32_t blk = sb[s];
            uint64_t key = ~0ull;
            if (blk >= 0 && blk >= g.sink_end && blk < g.local_begin && !((inS[blk >> 5] >> (blk & 31)) & 1u))
                key = victim_key(p.policy, lu[s], ph[s], uc[s], blk, sc[blk], rb.err);
            keys[s] = key;
        }
        __syncthreads();
        // radix select: the nv-th smallest key, T (keys are unique among candidates)
        uint64_t prefix = 0, mask = 0;
        int kk = nv;
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
            __syncthreads();
            for (int64_t s = tid; s < p.C; s += blockDim.x) {
                const uint64_t key = keys[s];
                if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
            }
            __syncthreads();
            if (tid < 32) {
                int cnt[8], tot = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    cnt[i] = hist[8 * tid + i];
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
                            s_digit = (uint32_t)(8 * tid + i);
                            s_above = below;
                            break;
                        }
                        below += cnt[i];
                    }
                }
            }
            __syncthreads();
            prefix |= (uint64_t)s_digit << shift;
            mask |= 0xFFull << shift;
            kk -= s_above;
            __syncthreads();
        }
        const uint64_t T = prefix;
        // compact victims (key <= T) in slot order, then place them by key rank
        int nvc = 0;
        for (int base = 0; base < p.C; base += blockDim.x) {
            const int64_t s = base + tid;
            const int isv = (s < p.C && keys[s] <= T) ? 1 : 0;
            int tot;
            const int pos = block_exclusive_scan(isv, scan_scratch, &tot);
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
        if (s >= 0) {
            lu[s] = step;
            ph[s] = 0;
            uc[s] = uc[s] + 1;
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
    }
    __syncthreads();
    griddep_launch();
    // ---- 6. attention list: sink blocks ++ S ++ local blocks, ascending, with slots
    const int ns = g.sink_end, nl = g.nb - g.local_begin;
    for (int i = tid; i < p.W; i += blockDim.x) {
        int32_t b = -1, s = -1;
        if (i < ns) b = i;
        else if (i < ns + k) b = S[i - ns];
        else if (i < ns + k + nl) b = g.local_begin + (i - ns - k);
        if (b >= 0) s = table[b];
        attn[2 * i] = b;
        attn[2 * i + 1] = s;
    }
}

// (a4) grid-stride over (request, head, miss index); one warp per 8 KiB record.
constexpr int kGatherThreads = 128;
__global__ void __launch_bounds__(kGatherThreads) gather_kernel(StepParams p, const int32_t* __restrict__ miss,
                                                                const int32_t* __restrict__ miss_count, int kmax,
                                                                const uint8_t* __restrict__ host_store,
                                                                uint8_t* __restrict__ slots) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t total = (int64_t)p.B * p.Hkv * p.k;
    const int chunks = p.rec_bytes / 16;
    griddep_wait();                               // miss list comes from resolve
    for (int64_t w = warp; w < total; w += nwarps) {
        const int i = (int)(w % p.k);
        const int64_t bh = w / p.k;
        const int h = (int)(bh % p.Hkv), bi = (int)(bh / p.Hkv);
        const int r = p.req[bi];
        const int64_t rs = (int64_t)r * p.Hkv + h;
        if (i >= miss_count[rs]) continue;
        const int32_t blk = miss[(rs * kmax + i) * 2], slot = miss[(rs * kmax + i) * 2 + 1];
        const int4* src = reinterpret_cast<const int4*>(
            host_store + ((((int64_t)p.host_layer * p.R + r) * p.Hkv + h) * p.nb_max + blk) * (int64_t)p.rec_bytes);
        int4* dst = reinterpret_cast<int4*>(
            slots + ((((int64_t)p.layer * p.R + r) * p.Hkv + h) * p.C + slot) * (int64_t)p.rec_bytes);
        for (int c0 = 0; c0 < chunks; c0 += 32 * 8) {
            int4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int c = c0 + u * 32 + lane;
                if (c < chunks) v[u] = ld_host16(src + c);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int c = c0 + u * 32 + lane;
                if (c < chunks) dst[c] = v[u];
            }
        }
    }
}

cudaError_t launch_resolve(kvd_cache* c, const StepParams& p, const int32_t* ids, int32_t* out_attn,
                           cudaStream_t s) {
    ResolveBufs rb{c->table,    c->slot_block, c->last_use, c->phase, c->use_count, c->scores,
                   c->ntok_dev, c->miss,       c->miss_count, c->kmax, c->stats,    c->err};
    const size_t smem = sizeof(uint64_t) * (size_t)c->C + sizeof(int32_t) * (size_t)c->kmax * 5 +
                        sizeof(uint32_t) * (size_t)((c->nb_pad + 31) / 32);
    static size_t smem_set = 48 << 10;
    if (smem > smem_set) {
        cudaError_t e = cudaFuncSetAttribute(resolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        smem_set = smem;
    }
    cudaError_t e = launch_pdl(resolve_kernel, dim3(p.Hkv, p.B), dim3(kResolveThreads), smem, s, p, rb, ids, out_attn);
    if (e != cudaSuccess) return e;
    if (!c->resident) {
        static int prio = 1;
        if (prio == 1) {
            int lo = 0, hi = 0;
            cudaDeviceGetStreamPriorityRange(&lo, &hi);
            prio = hi;                                   // greatest priority (numerically lowest)
        }
        e = launch_pdl_prio(prio, gather_kernel, dim3(148), dim3(kGatherThreads), 0, s, p, (const int32_t*)c->miss,
                       (const int32_t*)c->miss_count, (int)c->kmax, (const uint8_t*)c->host_store, c->slots);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

}  // namespace kvd
