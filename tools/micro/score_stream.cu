// Microbenchmark: per-SM streaming rate of the block-summary scan (a1) -- one CTA per segment
// scoring 2048 blocks x 128 dims bf16 (dim-major rows of 4 KiB, 512 KiB per CTA) with the
// sequential fp32 FMA chain per block.  Variants: per-thread LDG of V blocks (V = 2, 4, 8) with
// two ping-pong register batches of R rows, and a TMA ring of row copies into shared memory.
// usage: ./score_stream  (prints us and GB/s per SM for 8 / 64 / 148 CTAs)
#include <cstdio>
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_18071_b200/csrc/common.cuh"
using namespace kvd;

constexpr int NB = 2048;          // blocks per segment (row length)

template <int V> struct Vt;
template <> struct Vt<2> { using T = uint32_t; static __device__ uint32_t w(const T& x, int) { return x; } };
template <> struct Vt<4> { using T = uint2; static __device__ uint32_t w(const T& x, int i) { return i ? x.y : x.x; } };
template <> struct Vt<8> { using T = uint4; static __device__ uint32_t w(const T& x, int i) { return i == 0 ? x.x : i == 1 ? x.y : i == 2 ? x.z : x.w; } };

__device__ unsigned long long g_t[2 * 1024];
__device__ __forceinline__ void stamp(int i) { if (threadIdx.x == 0) g_t[2 * blockIdx.x + i] = global_ns(); }

template <int NT, int V, int R>
__global__ void __launch_bounds__(NT, 1) ldg_kernel(const uint16_t* summ, float* out) {
    stamp(0);
    using Vec = typename Vt<V>::T;
    const Vec* src = reinterpret_cast<const Vec*>(summ + (size_t)blockIdx.x * 128 * NB) + threadIdx.x;
    const int64_t rs = NB / V;
    Vec A[R], B[R];
#pragma unroll
    for (int u = 0; u < R; ++u) A[u] = __ldcs(src + u * rs);
#pragma unroll
    for (int u = 0; u < R; ++u) B[u] = __ldcs(src + (R + u) * rs);
    float acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.f;
    const float qj = 1.0001f;
    auto consume = [&](const Vec (&b)[R]) {
#pragma unroll
        for (int u = 0; u < R; ++u)
#pragma unroll
            for (int v = 0; v < V; ++v) { uint32_t w = Vt<V>::w(b[u], v >> 1); acc[v] = __fmaf_rn(qj, (v & 1) ? bf16_hi(w) : bf16_lo(w), acc[v]); }
    };
#pragma unroll 1
    for (int j0 = 0; j0 < 128; j0 += 2 * R) {
        consume(A);
        if (j0 + 2 * R < 128) {
#pragma unroll
            for (int u = 0; u < R; ++u) A[u] = __ldcs(src + (j0 + 2 * R + u) * rs);
        }
        consume(B);
        if (j0 + 3 * R < 128) {
#pragma unroll
            for (int u = 0; u < R; ++u) B[u] = __ldcs(src + (j0 + 3 * R + u) * rs);
        }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) out[(size_t)blockIdx.x * NB + threadIdx.x * V + v] = acc[v];
    __syncthreads();
    stamp(1);
}

// TMA ring: NS stages of RS rows (RS * 4 KiB), thread 0 issues row copies; 1024 threads, V = 2
template <int NS, int RS>
__global__ void __launch_bounds__(1024, 1) tma_kernel(const uint16_t* summ, float* out) {
    stamp(0);
    extern __shared__ __align__(128) uint16_t stg[];
    __shared__ __align__(8) uint64_t bar[NS];
    const uint16_t* seg = summ + (size_t)blockIdx.x * 128 * NB;
    constexpr int NSTG = 128 / RS;
    auto issue = [&](int x) {
        const int b = x % NS;
        mbar_arrive_expect_tx(&bar[b], RS * NB * 2);
        for (int r = 0; r < RS; ++r) bulk_g2s(stg + (b * RS + r) * NB, seg + (size_t)(x * RS + r) * NB, NB * 2, &bar[b]);
    };
    if (threadIdx.x == 0) {
        for (int b = 0; b < NS; ++b) mbar_init(&bar[b], 1);
        fence_mbar_init();
        for (int x = 0; x < NS; ++x) issue(x);
    }
    __syncthreads();
    float a0 = 0.f, a1 = 0.f;
    const float qj = 1.0001f;
    for (int x = 0; x < NSTG; ++x) {
        const int b = x % NS;
        mbar_wait(&bar[b], (x / NS) & 1);
#pragma unroll
        for (int r = 0; r < RS; ++r) {
            const uint32_t w = reinterpret_cast<const uint32_t*>(stg + (b * RS + r) * NB)[threadIdx.x];
            a0 = __fmaf_rn(qj, bf16_lo(w), a0);
            a1 = __fmaf_rn(qj, bf16_hi(w), a1);
        }
        __syncthreads();
        if (threadIdx.x == 0 && x + NS < NSTG) { fence_proxy_async(); issue(x + NS); }
    }
    out[(size_t)blockIdx.x * NB + threadIdx.x * 2] = a0;
    out[(size_t)blockIdx.x * NB + threadIdx.x * 2 + 1] = a1;
    __syncthreads();
    stamp(1);
}

template <class K>
static void bench(const char* name, K kern, int nt, size_t smem, const uint16_t* s, float* o, double cta_bytes = 512.0 * 1024) {
    if (smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int ctas : {8, 64, 148}) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int i = 0; i < 3; ++i) kern<<<ctas, nt, smem>>>(s, o);
        cudaEventRecord(e0);
        const int reps = 20;
        for (int i = 0; i < reps; ++i) kern<<<ctas, nt, smem>>>(s + (size_t)(i % 2) * 148 * 128 * NB, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / reps;
        unsigned long long t[2 * 1024];
        cudaMemcpyFromSymbol(t, g_t, sizeof(unsigned long long) * 2 * ctas);
        unsigned long long t0 = ~0ull, t1 = 0, dmax = 0;
        for (int i = 0; i < ctas; ++i) { t0 = std::min(t0, t[2 * i]); t1 = std::max(t1, t[2 * i + 1]); dmax = std::max(dmax, t[2 * i + 1] - t[2 * i]); }
        const double kus = (t1 - t0) * 1e-3;
        printf("%-28s ctas %3d: launch %6.2f us, in-kernel %6.2f us (slowest CTA %6.2f): %6.1f GB/s per SM %7.1f GB/s total (%s)\n", name, ctas, us,
               kus, dmax * 1e-3, cta_bytes / (dmax * 1e-9) / 1e9, ctas * cta_bytes / (kus * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
}

int main() {
    uint16_t* s; float* o;
    const size_t n = (size_t)2 * 148 * 128 * NB;
    cudaMalloc(&s, n * 2); cudaMalloc(&o, (size_t)148 * NB * 4);
    cudaMemset(s, 0x3f, n * 2);
    bench("ldg V8 NT512 R8 (1 MiB/CTA)", ldg_kernel<512, 8, 8>, 512, 0, s, o, 1024.0 * 1024);
    bench("ldg V8 NT512 R4 (1 MiB/CTA)", ldg_kernel<512, 8, 4>, 512, 0, s, o, 1024.0 * 1024);
    bench("ldg V8 NT256 R8", ldg_kernel<256, 8, 8>, 256, 0, s, o);
    bench("ldg V2 NT1024 R16", ldg_kernel<1024, 2, 16>, 1024, 0, s, o);
    bench("ldg V2 NT1024 R8", ldg_kernel<1024, 2, 8>, 1024, 0, s, o);
    bench("ldg V4 NT512 R16", ldg_kernel<512, 4, 16>, 512, 0, s, o);
    bench("ldg V4 NT512 R8", ldg_kernel<512, 4, 8>, 512, 0, s, o);
    bench("ldg V8 NT256 R16", ldg_kernel<256, 8, 16>, 256, 0, s, o);
    bench("tma NS4 RS8 (4 KiB rows)", tma_kernel<4, 8>, 1024, 4 * 8 * NB * 2, s, o);
    bench("tma NS6 RS4", tma_kernel<6, 4>, 1024, 6 * 4 * NB * 2, s, o);
    bench("tma NS12 RS2", tma_kernel<12, 2>, 1024, 12 * 2 * NB * 2, s, o);
    bench("tma NS3 RS16", tma_kernel<3, 16>, 1024, 3 * 16 * NB * 2, s, o);
    return 0;
}
