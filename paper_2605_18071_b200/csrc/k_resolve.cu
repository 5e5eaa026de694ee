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
#include <cstdlib>

#include "resolve.cuh"

namespace kvd {


// dynamic smem: keys64[nkeys] | S | hitslot | M | dest | vtmp (kmax each) | inS[nwords]
__global__ void __launch_bounds__(kResolveThreads) resolve_kernel(StepParams p, ResolveBufs rb,
                                                                  const int32_t* __restrict__ ids,
                                                                  int32_t* __restrict__ out_attn) {
    extern __shared__ __align__(16) uint8_t smraw[];
    __shared__ ResolveShared rsm;
    const int bi = blockIdx.y, h = p.h0 + blockIdx.x;
    resolve_pre(p, rb, bi, h, rsm);
    griddep_wait();                               // ids / scores come from select
    if (threadIdx.x == 0) kt_begin(p.kt_slots, p.kt_base + kKtResolve);
    resolve_main(p, rb, bi, h, ids, out_attn, smraw, rsm, true);
    if (p.kt_slots) {
        __syncthreads();
        if (threadIdx.x == 0)
            kt_end(p.kt_slots, p.kt_acc, p.kt_base + kKtResolve, kKtResolve, (unsigned long long)gridDim.x * gridDim.y);
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
    const int64_t total = (int64_t)p.B * p.nh * p.k;
    const int chunks = p.rec_bytes / 16;
    griddep_wait();                               // miss list comes from resolve
    if (threadIdx.x == 0) kt_begin(p.kt_slots, p.kt_base + kKtGather);
    for (int64_t w = warp; w < total; w += nwarps) {
        const int i = (int)(w % p.k);
        const int64_t bh = w / p.k;
        const int h = p.h0 + (int)(bh % p.nh), bi = (int)(bh / p.nh);
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
    if (p.kt_slots) {
        __syncthreads();
        if (threadIdx.x == 0) kt_end(p.kt_slots, p.kt_acc, p.kt_base + kKtGather, kKtGather, gridDim.x);
    }
}

// Host-link probe (kvd_probe_zero_copy): the gather's own access pattern -- 16-byte zero-copy
// loads from mapped pinned memory, 8 in flight per thread -- over a contiguous range.
__global__ void __launch_bounds__(256) zero_copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n16) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n16; i0 += 8 * stride) {
        int4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (i0 + u * stride < n16) v[u] = ld_host16(src + i0 + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (i0 + u * stride < n16) dst[i0 + u * stride] = v[u];
    }
}

cudaError_t launch_zero_copy(const void* host, void* dev, size_t bytes, int ctas, cudaStream_t s) {
    zero_copy_kernel<<<ctas, 256, 0, s>>>(reinterpret_cast<const int4*>(host), reinterpret_cast<int4*>(dev),
                                          (int64_t)(bytes / 16));
    return cudaGetLastError();
}

// kvd_set_segment_capacity: drop the residents of slots >= cap of layer-head (layer, head) in
// every request (pinned blocks live in slots < pinned <= cap).  grid (R), 256 threads.
__global__ void shrink_capacity_kernel(int32_t* table, int32_t* slot_block, int64_t nb_pad, int64_t C, int64_t cap,
                                       int layer, int head, int R, int Hkv) {
    const int r = blockIdx.x;
    const int64_t seg = ((int64_t)layer * R + r) * Hkv + head;
    int32_t* sb = slot_block + seg * C;
    int32_t* tb = table + seg * nb_pad;
    for (int64_t s = cap + threadIdx.x; s < C; s += blockDim.x) {
        const int32_t b = sb[s];
        if (b >= 0) {
            tb[b] = -1;
            sb[s] = -1;
        }
    }
}

cudaError_t launch_shrink_capacity(kvd_cache* c, int layer, int head, int64_t cap, cudaStream_t s) {
    shrink_capacity_kernel<<<c->R, 256, 0, s>>>(c->table, c->slot_block, c->nb_pad, c->C, cap, layer, head, c->R, c->Hkv);
    return cudaGetLastError();
}

size_t resolve_static_smem() { return sizeof(ResolveShared); }

size_t resolve_smem_bytes(int64_t nkeys, int64_t kmax, int64_t nb_pad) {
    return sizeof(uint64_t) * (size_t)nkeys + sizeof(int32_t) * (size_t)kmax * 5 +
           sizeof(uint32_t) * (size_t)((nb_pad + 31) / 32);
}

ResolveBufs resolve_bufs(kvd_cache* c, int layer) {
    ResolveBufs rb{c->table,    c->slot_block, c->last_use, c->phase, c->use_count, c->scores,
                   c->ntok_dev, c->miss,       c->miss_count, c->kmax, 0,           c->stats,    c->err};
    rb.nkeys = c->resident ? 0 : c->C;            // a fully resident cache never evicts
    rb.ntok = c->ntok_dev + (int64_t)layer * c->R;   // token counts of the launch's layer
    rb.cap = c->cap_dev;
    rb.cbits = c->cand_bits;                      // NULL unless the hierarchical index is on
    rb.cent_of = c->cent_of;
    rb.cscores = c->cscores;
    rb.nc_pad = c->nc_pad;
    rb.seg_stats = c->seg_stats;
    return rb;
}

cudaError_t launch_gather(kvd_cache* c, const StepParams& p, cudaStream_t s) {
    // greatest priority (numerically lowest): scheduled ahead of other chains' HBM-bound kernels
    return launch_pdl_prio(c->prio_hi, gather_kernel, dim3(148), dim3(kGatherThreads), 0, s, p, (const int32_t*)c->miss,
                           (const int32_t*)c->miss_count, (int)c->kmax, (const uint8_t*)c->host_store, c->slots);
}

cudaError_t launch_resolve(kvd_cache* c, const StepParams& p, const int32_t* ids, int32_t* out_attn,
                           cudaStream_t s) {
    const ResolveBufs rb = resolve_bufs(c, p.layer);
    const size_t smem = resolve_smem_bytes(rb.nkeys, c->kmax, c->nb_pad);
    static size_t smem_set[64] = {};              // opted-in dynamic size, per device ordinal
    const int dev = c->cfg.device & 63;
    if (smem > smem_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(resolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        smem_set[dev] = smem;
    }
    cudaError_t e = launch_pdl(resolve_kernel, dim3(p.nh, p.B), dim3(kResolveThreads), smem, s, p, rb, ids, out_attn);
    if (e != cudaSuccess) return e;
    if (!c->resident) {
        e = launch_gather(c, p, s);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

}  // namespace kvd
