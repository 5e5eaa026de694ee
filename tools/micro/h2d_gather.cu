// Microbenchmark: gather N random 8 KiB records from pinned (mapped) host memory into HBM.
// (a) SM zero-copy 16-B loads, one warp per record, U loads in flight per lane
// (b) TMA bulk copy host->smem, then bulk copy smem->global (one warp per record)
// (c) cudaMemcpyAsync per record (DMA engines), and one big contiguous cudaMemcpy
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2605_18071_b200/csrc/common.cuh"
using namespace kvd;

template <int U>
__global__ void zc_kernel(const uint8_t* host, uint8_t* dev, const int* ids, int n) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < n; i += nw) {
        const int4* src = reinterpret_cast<const int4*>(host + (int64_t)ids[i] * 8192);
        int4* dst = reinterpret_cast<int4*>(dev + i * 8192);
        for (int c0 = 0; c0 < 512; c0 += 32 * U) {
            int4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = ld_stream16(src + c0 + u * 32 + lane);
#pragma unroll
            for (int u = 0; u < U; ++u) dst[c0 + u * 32 + lane] = v[u];
        }
    }
}

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// one warp per record, 2 records in flight per warp (16 KiB smem per warp)
__global__ void tma_kernel(const uint8_t* host, uint8_t* dev, const int* ids, int n) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[8][2];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint8_t* buf = sm + wl * 16384;
    if (lane == 0) { mbar_init(&bar[wl][0], 1); mbar_init(&bar[wl][1], 1); fence_mbar_init(); }
    __syncwarp();
    int k = 0;
    for (int64_t i = warp; i < n; i += nw, ++k) {
        const int b = k & 1;
        if (lane == 0) {
            bulk_wait_read0();   // smem buffer free again
            mbar_arrive_expect_tx(&bar[wl][b], 8192);
            bulk_g2s(buf + b * 8192, host + (int64_t)ids[i] * 8192, 8192, &bar[wl][b]);
            mbar_wait(&bar[wl][b], (k >> 1) & 1);
            bulk_s2g(dev + i * 8192, buf + b * 8192, 8192);
            bulk_commit();
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const int64_t nrec_host = (8ll << 30) / 8192;      // 8 GiB pinned host store
    const int n = 4096;                                 // 32 MiB per gather
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
        printf("%-44s %8.1f us %6.1f GB/s (%s)\n", name, ms * 1e3, n * 8192.0 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    for (int grid : {74, 148, 296, 592}) {
        char nm[96];
        snprintf(nm, sizeof nm, "zero-copy U=8 grid=%d x256", grid);
        report(nm, [&] { zc_kernel<8><<<grid, 256>>>(host, dev, ids, n); });
        snprintf(nm, sizeof nm, "zero-copy U=16 grid=%d x256", grid);
        report(nm, [&] { zc_kernel<16><<<grid, 256>>>(host, dev, ids, n); });
        snprintf(nm, sizeof nm, "zero-copy U=4 grid=%d x256", grid);
        report(nm, [&] { zc_kernel<4><<<grid, 256>>>(host, dev, ids, n); });
    }
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
    for (int grid : {74, 148, 296}) {
        char nm[96];
        snprintf(nm, sizeof nm, "TMA host->smem->HBM grid=%d x256", grid);
        report(nm, [&] { tma_kernel<<<grid, 256, 8 * 16384>>>(host, dev, ids, n); });
    }
    report("cudaMemcpyAsync per record (4096 calls)", [&] {
        for (int i = 0; i < n; ++i) cudaMemcpyAsync(dev + (int64_t)i * 8192, host + (int64_t)hid[i] * 8192, 8192, cudaMemcpyHostToDevice);
    });
    report("cudaMemcpyAsync contiguous 32 MiB", [&] { cudaMemcpyAsync(dev, host, (int64_t)n * 8192, cudaMemcpyHostToDevice); });
    return 0;
}
