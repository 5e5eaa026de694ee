// common.cuh — sm_100a device helpers for libkvd: bf16 bit handling, the
// monotone score / victim keys, mbarrier + bulk-copy (TMA engine) wrappers,
// ldmatrix / mma.sync / movmatrix wrappers, block-wide scans.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kvd {

constexpr int kHeadDim = 128;
constexpr int kRowBytes = kHeadDim * 2;         // one token row of K or V (bf16)

// ----------------------------------------------------------------- bf16
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ float bf16_bits(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }
// binary32 -> bf16 round-to-nearest-even (finite inputs; NaN stays NaN)
__device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
    uint32_t u = __float_as_uint(f);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40u);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
// hardware round-to-nearest-even pack (cvt.rn.bf16x2.f32): lo -> bits 0-15, hi -> 16-31
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    return (uint32_t)f32_to_bf16_rne(lo) | ((uint32_t)f32_to_bf16_rne(hi) << 16);
}

// ------------------------------------------------------------- order keys
// Monotone 32-bit key of a score: larger score -> larger key; -0 == +0; NaN -> 0
// (lowest).  DESIGN.md §3 R10.
__device__ __forceinline__ uint32_t score_key32(float s) {
    uint32_t u = __float_as_uint(s);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return 0u;  // NaN
    if ((u << 1) == 0u) u = 0u;                                             // -0 -> +0
    return (u >> 31) ? ~u : (u | 0x80000000u);
}

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    while (!mbar_try_wait(a, parity)) {
    }
}
// Bulk async copy global -> shared (TMA engine, non-tensor form), completion
// signalled on `bar` as transaction bytes.  bytes % 16 == 0, 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Same, with an L2 evict-first policy (streamed once per step).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
// D = A(16x16 bf16, row) * B(16x8 bf16, col) + D, fp32 accumulate.
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 16-byte streaming load from host-mapped memory: no L1 allocation, 256-byte L2
// fetch granularity (fewer, larger host-link read requests for a warp's 512 B).
__device__ __forceinline__ int4 ld_host16(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// 16-byte streaming load that does not allocate in L1 (host-mapped or HBM).
__device__ __forceinline__ int4 ld_stream16(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ------------------------------------------- programmatic dependent launch
// Every step kernel is launched with programmatic stream serialization
// (launch_pdl) so its prologue overlaps the previous kernel's tail; it calls
// griddep_wait() before touching anything an earlier kernel of the step wrote,
// and griddep_launch() once its main loop is done.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------ in-kernel launch timing
// kvd_enable_kernel_timer: every step kernel records its launch's duration on the device, so
// the benchmark can time the kernels of the exact (graph-captured, PDL-chained, multi-stream)
// path it times, with no event node between kernels.  A launch's units (CTAs or warps) take
// the min of their start stamps (after griddepcontrol.wait) in the launch's slot; the unit that
// completes the slot's count adds end - start to the per-kind accumulator and resets the slot.
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void kt_begin(unsigned long long* slots, int slot) {
    if (slots) atomicMin(&slots[2 * slot], global_ns());
}
__device__ __forceinline__ void kt_end(unsigned long long* slots, unsigned long long* acc, int slot, int kind,
                                       unsigned long long units) {
    if (!slots) return;
    unsigned long long* sl = slots + 2 * slot;
    if (atomicAdd(&sl[1], 1ull) == units - 1) {
        const unsigned long long t1 = global_ns();
        const unsigned long long t0 = atomicExch(&sl[0], ~0ull);
        atomicExch(&sl[1], 0ull);
        atomicAdd(&acc[2 * kind], t1 > t0 ? t1 - t0 : 0ull);
        atomicAdd(&acc[2 * kind + 1], 1ull);
    }
}
// Phase stamps for tuning (experiment builds only: -DKVD_EXPERIMENTS; compiled out of the
// product).  EXP_STAMP(buf, unit, i) records %globaltimer for unit (CTA / warp index) and
// phase i into the device buffer StepParams::exp_trace, read back by kvd_exp_read_trace.
constexpr int kExpUnits = 16384, kExpPhases = 8;
#ifdef KVD_EXPERIMENTS
#define EXP_STAMP(buf, unit, i)                                                             \
    do {                                                                                   \
        if ((buf) && (unit) < kExpUnits) (buf)[(unit) * kExpPhases + (i)] = global_ns();    \
    } while (0)
#else
#define EXP_STAMP(buf, unit, i) \
    do {                        \
    } while (0)
#endif
enum { kKtSelect = 0, kKtResolve = 1, kKtGather = 2, kKtAttn = 3, kKtScore = 4, kKtKinds = 5 };

// Process-wide count of step-kernel launches issued by libkvd (kvd_launch_count;
// a launch recorded into a CUDA graph counts once, at capture).
void count_launch();

// `priority` (optional, cudaLaunchAttributePriority): the host-link gather is launched at the
// device's greatest priority so its CTAs are scheduled ahead of concurrent HBM-bound kernels
// of other micro-batch chains (keeps the link busy).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_prio(int priority, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                   cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributePriority;
    attr[1].val.priority = priority;
    cfg.attrs = attr;
    cfg.numAttrs = priority ? 2 : 1;
    count_launch();
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    return launch_pdl_prio(0, kern, grid, block, smem, s, static_cast<Args&&>(args)...);
}

// Shared-memory histogram increment aggregated over the lanes of a warp that
// hit the same bin (the leading key bits are nearly constant, so plain atomics
// would serialise on one bin).  All 32 lanes must call it; `active` = this
// lane contributes.
__device__ __forceinline__ void warp_hist_add(int* hist, uint32_t bin, bool active) {
    const uint32_t act = __ballot_sync(0xffffffffu, active);
    if (!active) return;
    const uint32_t peers = __match_any_sync(act, bin);
    if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&hist[bin], __popc(peers));
}

// ------------------------------------------------------------ block scans
// Exclusive prefix sum of one int per thread over the whole CTA (blockDim.x a
// multiple of 32, <= 1024).  `scratch` >= 33 ints of shared memory.  Returns the
// exclusive prefix; *total receives the CTA sum.  Contains __syncthreads.
__device__ __forceinline__ int block_exclusive_scan(int v, int* scratch, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < nw ? scratch[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) scratch[lane] = w;      // inclusive warp totals
        if (lane == 31) scratch[32] = w;
    }
    __syncthreads();
    int base = warp ? scratch[warp - 1] : 0;
    int t = scratch[32];
    __syncthreads();                           // scratch may be reused right after
    *total = t;
    return base + x - v;
}

}  // namespace kvd
