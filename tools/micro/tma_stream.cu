// Microbenchmark: stream 8 KiB tiles HBM -> SMEM per warp worker.
// (a) cp.async.bulk ring (STAGES deep) with mbarriers, no compute
// (b) same with 16-byte LDG into registers (baseline)
// usage: ./tma_stream   (prints GB/s per variant)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_18071_b200/csrc/common.cuh"
using namespace kvd;

template <int STAGES, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) tma_kernel(const uint8_t* src, int64_t ntiles, int tiles_per_warp, int hint, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t stage[];
    __shared__ __align__(8) uint64_t bar[WARPS][STAGES];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w = (int64_t)blockIdx.x * WARPS + warp;
    uint8_t* my = stage + (size_t)warp * STAGES * 8192;
    if (lane == 0) { for (int s = 0; s < STAGES; ++s) mbar_init(&bar[warp][s], 1); fence_mbar_init(); }
    __syncwarp();
    const uint64_t pol = l2_evict_first_policy();
    auto issue = [&](int k) {
        if (lane == 0) {
            const int64_t t = (w * tiles_per_warp + k) % ntiles;
            mbar_arrive_expect_tx(&bar[warp][k % STAGES], 8192);
            if (hint) bulk_g2s_hint(my + (k % STAGES) * 8192, src + t * 8192, 8192, &bar[warp][k % STAGES], pol);
            else bulk_g2s(my + (k % STAGES) * 8192, src + t * 8192, 8192, &bar[warp][k % STAGES]);
        }
    };
    for (int k = 0; k < STAGES && k < tiles_per_warp; ++k) issue(k);
    uint32_t acc = 0;
    for (int k = 0; k < tiles_per_warp; ++k) {
        mbar_wait(&bar[warp][k % STAGES], (k / STAGES) & 1);
        acc += reinterpret_cast<uint32_t*>(my + (k % STAGES) * 8192)[lane];
        __syncwarp();
        if (k + STAGES < tiles_per_warp) { fence_proxy_async(); issue(k + STAGES); }
    }
    if (acc == 0x12345678) atomicAdd(sink, 1ull);
}

template <int WARPS, int UNROLL>
__global__ void __launch_bounds__(WARPS * 32) ldg_kernel(const uint8_t* src, int64_t ntiles, int tiles_per_warp, unsigned long long* sink) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w = (int64_t)blockIdx.x * WARPS + warp;
    uint32_t acc = 0;
    for (int k = 0; k < tiles_per_warp; ++k) {
        const int64_t t = (w * tiles_per_warp + k) % ntiles;
        const int4* p = reinterpret_cast<const int4*>(src + t * 8192);
        int4 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldcs(p + u * 32 + lane);
#pragma unroll
        for (int u = 0; u < 16; ++u) acc += v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678) atomicAdd(sink, 1ull);
}

template <typename F>
float timeit(F f) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 10;
}

template <int STAGES, int WARPS>
void run_tma(const uint8_t* src, int64_t ntiles, int ctas_per_sm, int tpw, int hint, unsigned long long* sink) {
    const size_t smem = (size_t)WARPS * STAGES * 8192;
    cudaFuncSetAttribute(tma_kernel<STAGES, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = 148 * ctas_per_sm;
    float ms = timeit([&] { tma_kernel<STAGES, WARPS><<<grid, WARPS * 32, smem>>>(src, ntiles, tpw, hint, sink); });
    const double bytes = (double)grid * WARPS * tpw * 8192;
    printf("TMA stages=%d warps=%d ctas/sm=%d tiles/warp=%d hint=%d: %.1f us  %.0f GB/s  (%s)\n", STAGES, WARPS, ctas_per_sm, tpw, hint,
           ms * 1e3, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int64_t ntiles = (4ll << 30) / 8192;   // 4 GiB source
    uint8_t* src; cudaMalloc(&src, ntiles * 8192); cudaMemset(src, 1, ntiles * 8192);
    unsigned long long* sink; cudaMalloc(&sink, 8);
    for (int tpw : {7, 14, 58, 200}) {
        run_tma<3, 4>(src, ntiles, 2, tpw, 1, sink);
        run_tma<3, 4>(src, ntiles, 2, tpw, 0, sink);
        run_tma<6, 4>(src, ntiles, 1, tpw, 1, sink);
        run_tma<2, 4>(src, ntiles, 3, tpw, 1, sink);
        run_tma<3, 8>(src, ntiles, 1, tpw, 1, sink);
        {
            const int grid = 148 * 4;
            float ms = timeit([&] { ldg_kernel<8, 16><<<grid, 256>>>(src, ntiles, tpw, sink); });
            printf("LDG warps=8 ctas/sm=4 tiles/warp=%d: %.1f us %.0f GB/s\n", tpw, ms * 1e3, (double)grid * 8 * tpw * 8192 / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
