// synth_gpu.cu — device copy of synth.c's K/V generator (inputs only; holds
// none of the method's arithmetic).  The per-token topic run scan and the
// topic centres are computed on the host by synth_segment_plan (synth.c); this
// kernel expands them into the bf16 K/V bytes with the same counter-based hash
// and the same IEEE fp32 operations (explicit _rn intrinsics, no contraction),
// so its output is byte-identical to synth_segment_kv (tests/test_synth_gpu.py).
// Used by bench.py to build 100+ GiB synthetic caches in seconds.
#include <cstdint>
#include <cuda_runtime.h>

namespace {
__device__ __forceinline__ uint64_t sm_mix(uint64_t x) {
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27; x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}
__device__ __forceinline__ uint64_t ctr_u64(uint64_t key, uint64_t ctr) {
    return sm_mix(key ^ sm_mix(ctr + 0x9E3779B97F4A7C15ull));
}
__device__ __forceinline__ float ctr_normal(uint64_t key, uint64_t ctr) {
    uint64_t x = ctr_u64(key, ctr);
    uint32_t s = (uint32_t)(x & 0xFFFF) + (uint32_t)((x >> 16) & 0xFFFF) + (uint32_t)((x >> 32) & 0xFFFF) +
                 (uint32_t)(x >> 48);
    return __fmul_rn(__fsub_rn((float)s, 131070.0f), 1.7320508f / 65536.0f);
}
__device__ __forceinline__ uint16_t to_bf16(float f) {
    uint32_t u = __float_as_uint(f);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

// grid-stride over 8-element groups of [n][d]; writes one 16-byte chunk each of K and V.
__global__ void kv_kernel(int64_t n, int32_t d, const uint8_t* __restrict__ topic, const float* __restrict__ mu,
                          uint64_t kk, uint64_t kv, uint16_t* __restrict__ K, uint16_t* __restrict__ V) {
    const int64_t groups = n * d / 8;
    for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < groups;
         gi += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e0 = gi * 8;
        const int64_t i = e0 / d;
        const int32_t j0 = (int32_t)(e0 % d);
        const float* m = mu + (int64_t)topic[i] * d;
        uint16_t ko[8], vo[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint64_t c = (uint64_t)(e0 + u);
            ko[u] = to_bf16(__fadd_rn(m[j0 + u], __fmul_rn(0.5f, ctr_normal(kk, c))));
            vo[u] = to_bf16(ctr_normal(kv, c));
        }
        if (K) *reinterpret_cast<uint4*>(K + e0) = *reinterpret_cast<uint4*>(ko);
        if (V) *reinterpret_cast<uint4*>(V + e0) = *reinterpret_cast<uint4*>(vo);
    }
}
}  // namespace

extern "C" {
// topic: device u8 [n]; mu: device f32 [32][d]; K, V: device bf16 [n][d] (d % 8 == 0).
int synth_gpu_segment_kv(int64_t n, int32_t d, const uint8_t* topic, const float* mu, uint64_t key_k,
                         uint64_t key_v, uint16_t* K, uint16_t* V, void* stream) {
    if (n <= 0) return 0;
    kv_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(n, d, topic, mu, key_k, key_v, K, V);
    return (int)cudaGetLastError();
}
}
