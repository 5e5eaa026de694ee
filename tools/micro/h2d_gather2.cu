// Microbenchmark 2: more host->HBM gather variants for 8 KiB records.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2605_18071_b200/csrc/common.cuh"
using namespace kvd;

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory"); }

// one warp per record stream, NB records in flight per warp (NB * 8 KiB smem per warp)
template <int NB>
__global__ void tma_kernel(const uint8_t* host, uint8_t* dev, const int* ids, int n, int chunk) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[8][NB];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint8_t* buf = sm + wl * NB * 8192;
    if (lane != 0) return;
    for (int b = 0; b < NB; ++b) mbar_init(&bar[wl][b], 1);
    fence_mbar_init();
    // records i = warp, warp + nw, ...; issue NB ahead
    int k = 0;
    int64_t i_issue = warp, i_done = warp;
    for (int b = 0; b < NB && i_issue < n; ++b, i_issue += nw) {
        mbar_arrive_expect_tx(&bar[wl][b], 8192);
        for (int c = 0; c < 8192; c += chunk) bulk_g2s(buf + b * 8192 + c, host + (int64_t)ids[i_issue] * 8192 + c, chunk, &bar[wl][b]);
    }
    for (; i_done < n; i_done += nw, ++k) {
        const int b = k % NB;
        mbar_wait(&bar[wl][b], (k / NB) & 1);
        bulk_s2g(dev + i_done * 8192, buf + b * 8192, 8192);
        bulk_commit();
        if (i_issue < n) {
            bulk_wait_read<0>();
            mbar_arrive_expect_tx(&bar[wl][b], 8192);
            for (int c = 0; c < 8192; c += chunk) bulk_g2s(buf + b * 8192 + c, host + (int64_t)ids[i_issue] * 8192 + c, chunk, &bar[wl][b]);
            i_issue += nw;
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int U>
__global__ void zc256_kernel(const uint8_t* host, uint8_t* dev, const int* ids, int n) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < n; i += nw) {
        const int4* src = reinterpret_cast<const int4*>(host + (int64_t)ids[i] * 8192);
        int4* dst = reinterpret_cast<int4*>(dev + i * 8192);
        for (int c0 = 0; c0 < 512; c0 += 32 * U) {
            int4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int4* a = src + c0 + u * 32 + lane;
                asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(a));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) dst[c0 + u * 32 + lane] = v[u];
        }
    }
}

int main() {
    const int64_t nrec_host = (8ll << 30) / 8192;
    const int n = 4096;
    uint8_t* host; cudaHostAlloc(&host, nrec_host * 8192, cudaHostAllocMapped);
    for (int64_t i = 0; i < nrec_host * 8192; i += 4096) host[i] = (uint8_t)i;
    uint8_t* dev; cudaMalloc(&dev, (int64_t)n * 8192);
    std::vector<int> hid(n);
    uint64_t x = 12345;
    for (int i = 0; i < n; ++i) { x = x * 6364136223846793005ull + 1442695040888963407ull; hid[i] = (int)((x >> 33) % nrec_host); }
    int* ids; cudaMalloc(&ids, n * 4); cudaMemcpy(ids, hid.data(), n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto report = [&](const char* name, auto f) {
        f(); cudaDeviceSynchronize();
        cudaEventRecord(a); for (int r = 0; r < 5; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
        printf("%-48s %8.1f us %6.1f GB/s (%s)\n", name, ms * 1e3, n * 8192.0 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    char nm[128];
    cudaFuncSetAttribute(tma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2 * 8192);
    cudaFuncSetAttribute(tma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * 8192);
    for (int grid : {148, 296}) for (int warps : {4, 8}) for (int chunk : {8192, 2048}) {
        snprintf(nm, sizeof nm, "TMA NB=2 grid=%d warps=%d chunk=%d", grid, warps, chunk);
        report(nm, [&] { tma_kernel<2><<<grid, warps * 32, warps * 2 * 8192>>>(host, dev, ids, n, chunk); });
        snprintf(nm, sizeof nm, "TMA NB=4 grid=%d warps=%d chunk=%d", grid, warps, chunk);
        report(nm, [&] { tma_kernel<4><<<grid, warps * 32, warps * 4 * 8192>>>(host, dev, ids, n, chunk); });
    }
    for (int grid : {148, 296, 592}) {
        snprintf(nm, sizeof nm, "zero-copy L2::256B U=4 grid=%d x128", grid);
        report(nm, [&] { zc256_kernel<4><<<grid, 128>>>(host, dev, ids, n); });
        snprintf(nm, sizeof nm, "zero-copy L2::256B U=8 grid=%d x256", grid);
        report(nm, [&] { zc256_kernel<8><<<grid, 256>>>(host, dev, ids, n); });
    }
    // contiguous DMA reference at several sizes
    for (int64_t mb : {8, 32, 256, 1024}) {
        uint8_t* d2; cudaMalloc(&d2, mb << 20);
        snprintf(nm, sizeof nm, "cudaMemcpyAsync contiguous %lld MiB", (long long)mb);
        cudaEventRecord(a); for (int r = 0; r < 3; ++r) cudaMemcpyAsync(d2, host, mb << 20, cudaMemcpyHostToDevice); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
        printf("%-48s %8.1f us %6.1f GB/s\n", nm, ms * 1e3, (mb << 20) / (ms * 1e-3) / 1e9);
        cudaFree(d2);
    }
    return 0;
}
