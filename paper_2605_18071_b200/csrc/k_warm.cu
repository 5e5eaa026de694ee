// k_warm.cu — importance-guided warm-up (DESIGN.md §3 R29; the oracle's O14).
//
// "At the end of the prefill phase, the model has already computed the attention between the
// prompt's final tokens and the entire prefix ... we assign importance scores to prefix tokens
// based on the attention distribution produced by the queries in the prompt's final observation
// window ... the entries with the highest scores are placed in GPU HBM for immediate access"
// (PAPER.md:593-604).  kvd_load_prefix_obs: after the prefix is ingested, warm_kernel (one CTA per
// KV head) computes, for the G x n_obs observation queries of the head, the softmax over all prefix
// tokens (pass 1: per-query max and normaliser, online over token slices; pass 2: per block, the
// attention mass of its tokens summed over the queries), then places the C - pinned most important
// non-pinned blocks (importance desc, block asc; an 8-bit radix select over the importances'
// bits) in the slots after the pinned blocks, ascending by block, as admitted at step 0.  The
// records of those blocks are then copied into their slots with the pinned ones.  fp32 with expf:
// the choice agrees with the oracle's fp64 one except at importance ties within fp32 rounding.
#include "common.cuh"
#include "internal.h"

namespace kvd {

constexpr int kWarmThreads = 1024;
constexpr int kMaxObsQueries = 128;              // G x n_obs (<= 8 x 16)

struct WarmArgs {
    const uint16_t* k;              // [Hkv][n][128] device, token-major
    const uint16_t* q;              // [Hkv * G][n_obs][128] device
    int64_t n;
    int n_obs, G, P;
    SegGeom g;
    float* imp;                     // [Hkv][nb] scratch
    int32_t* table;                 // segment rows of head 0 (stride nb_pad / C)
    int32_t* slot_block;
    uint32_t* last_use;
    uint8_t* phase;
    uint32_t* use_count;
    int32_t* slot_of;               // [Hkv][nb] record destinations (pinned already set)
    const int32_t* cap;             // [Hkv] slots of the layer-head window (2D scaling) or NULL
    int64_t nb_pad, C;
};

__global__ void __launch_bounds__(kWarmThreads) warm_kernel(WarmArgs wa) {
    extern __shared__ float wq[];                 // [Qn][128] observation queries (fp32)
    __shared__ float red_m[kWarmThreads], red_s[kWarmThreads];
    __shared__ float qm[kMaxObsQueries], qz[kMaxObsQueries];
    __shared__ int hist[256];
    __shared__ int scan[33];
    __shared__ int s_digit, s_above;
    const int h = blockIdx.x, tid = threadIdx.x;
    const int Qn = wa.G * wa.n_obs;
    const float scale = 1.0f / sqrtf((float)kHeadDim);
    const uint16_t* Kh = wa.k + (int64_t)h * wa.n * kHeadDim;
    for (int i = tid; i < Qn * kHeadDim; i += kWarmThreads) {
        const int qi = i / kHeadDim, j = i % kHeadDim;
        const int g = qi / wa.n_obs, w = qi % wa.n_obs;
        wq[i] = bf16_bits(wa.q[(((int64_t)h * wa.G + g) * wa.n_obs + w) * kHeadDim + j]);
    }
    __syncthreads();
    // ---- pass 1: per query, max logit and softmax normaliser (thread = (query, token slice))
    const int slices = kWarmThreads / Qn;
    if (tid < Qn * slices) {
        const int qi = tid / slices, sl = tid % slices;
        float m = -INFINITY, s = 0.0f;
        for (int64_t t = sl; t < wa.n; t += slices) {
            float z = 0.0f;
            for (int j = 0; j < kHeadDim; ++j) z = __fmaf_rn(wq[qi * kHeadDim + j], bf16_bits(Kh[t * kHeadDim + j]), z);
            z *= scale;
            if (z > m) {
                s = s * expf(m - z) + 1.0f;
                m = z;
            } else {
                s += expf(z - m);
            }
        }
        red_m[tid] = m;
        red_s[tid] = s;
    }
    __syncthreads();
    if (tid < Qn) {
        float M = -INFINITY;
        for (int i = 0; i < slices; ++i) M = fmaxf(M, red_m[tid * slices + i]);
        float Z = 0.0f;
        for (int i = 0; i < slices; ++i)
            if (red_m[tid * slices + i] > -INFINITY) Z += red_s[tid * slices + i] * expf(red_m[tid * slices + i] - M);
        qm[tid] = M;
        qz[tid] = Z;
    }
    __syncthreads();
    // ---- pass 2: block importance = attention mass of its tokens, summed over the queries
    const int nb = wa.g.nb;
    float* imp = wa.imp + (int64_t)h * nb;
    for (int b = tid; b < nb; b += kWarmThreads) {
        float acc = 0.0f;
        const int64_t t0 = (int64_t)b * wa.P, t1 = t0 + wa.P < wa.n ? t0 + wa.P : wa.n;
        for (int qi = 0; qi < Qn; ++qi)
            for (int64_t t = t0; t < t1; ++t) {
                float z = 0.0f;
                for (int j = 0; j < kHeadDim; ++j) z = __fmaf_rn(wq[qi * kHeadDim + j], bf16_bits(Kh[t * kHeadDim + j]), z);
                acc += expf(z * scale - qm[qi]) / qz[qi];
            }
        imp[b] = acc;
    }
    __syncthreads();
    // ---- the room = C - pinned most important candidates: radix select on the importance bits
    // (non-negative floats order like their bit patterns), ties -> lowest block (block order)
    const int64_t C = wa.cap ? (int64_t)wa.cap[h] : wa.C;
    const int pinned = wa.g.sink_end + (nb - wa.g.local_begin);
    const int ncand = wa.g.local_begin - wa.g.sink_end;
    const int room = (int)(C - pinned < ncand ? C - pinned : ncand);
    if (room <= 0) return;
    auto keyof = [&](int b) { return (b >= wa.g.sink_end && b < wa.g.local_begin) ? __float_as_uint(imp[b]) : 0u; };
    uint32_t prefix = 0u, mask = 0u;
    int kk = room;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += kWarmThreads) hist[i] = 0;
        __syncthreads();
        for (int b = tid; b < nb; b += kWarmThreads) {
            const bool cand = b >= wa.g.sink_end && b < wa.g.local_begin;
            const uint32_t key = keyof(b);
            if (cand && (key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1);
        }
        __syncthreads();
        if (tid == 0) {
            int above = 0;
            for (int d = 255; d >= 0; --d) {
                if (above + hist[d] >= kk) {
                    s_digit = d;
                    s_above = above;
                    break;
                }
                above += hist[d];
            }
        }
        __syncthreads();
        prefix |= (uint32_t)s_digit << shift;
        mask |= 255u << shift;
        kk -= s_above;
        __syncthreads();
    }
    const uint32_t T = prefix;
    int32_t* table = wa.table + (int64_t)h * wa.nb_pad;
    int32_t* sb = wa.slot_block + (int64_t)h * wa.C;
    int taken = 0, eqs = 0;
    for (int b0 = 0; b0 < nb; b0 += kWarmThreads) {
        const int b = b0 + tid;
        const bool cand = b < nb && b >= wa.g.sink_end && b < wa.g.local_begin;
        const uint32_t key = cand ? keyof(b) : 0u;
        const bool eq = cand && key == T;
        int tot_eq;
        const int eq_rank = eqs + block_exclusive_scan(eq ? 1 : 0, scan, &tot_eq);
        const bool take = cand && (key > T || (eq && eq_rank < kk));
        int tot;
        const int pos = taken + block_exclusive_scan(take ? 1 : 0, scan, &tot);
        if (take) {
            const int s = pinned + pos;
            table[b] = s;
            sb[s] = b;
            wa.last_use[(int64_t)h * wa.C + s] = 0u;
            wa.phase[(int64_t)h * wa.C + s] = 1;
            wa.use_count[(int64_t)h * wa.C + s] = 1u;
            wa.slot_of[(int64_t)h * nb + b] = s;
        }
        taken += tot;
        eqs += tot_eq;
    }
}

cudaError_t launch_warm(kvd_cache* c, int layer, int req, const uint16_t* dk, const uint16_t* dq, int n_obs, int64_t n,
                        int32_t* slot_of, cudaStream_t s) {
    const SegGeom g = seg_geom(n, c->P, c->cfg.sink_tokens, c->cfg.local_tokens);
    const int64_t sl = ((int64_t)layer * c->R + req) * c->Hkv;
    if (!c->warm_imp) {
        cudaError_t e = cudaMalloc(&c->warm_imp, (size_t)c->Hkv * c->nb_max * 4);
        if (e != cudaSuccess) return e;
    }
    WarmArgs wa;
    wa.k = dk;
    wa.q = dq;
    wa.n = n;
    wa.n_obs = n_obs;
    wa.G = c->G;
    wa.P = c->P;
    wa.g = g;
    wa.imp = c->warm_imp;
    wa.table = c->table + sl * c->nb_pad;
    wa.slot_block = c->slot_block + sl * c->C;
    wa.last_use = c->last_use + sl * c->C;
    wa.phase = c->phase + sl * c->C;
    wa.use_count = c->use_count + sl * c->C;
    wa.slot_of = slot_of;
    wa.cap = c->cap_dev + (int64_t)layer * c->Hkv;
    wa.nb_pad = c->nb_pad;
    wa.C = c->C;
    const size_t smem = (size_t)c->G * n_obs * kHeadDim * 4;
    static bool attr[64] = {};
    if (!attr[c->cfg.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(warm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(kMaxObsQueries * kHeadDim * 4));
        if (e != cudaSuccess) return e;
        attr[c->cfg.device & 63] = true;
    }
    warm_kernel<<<c->Hkv, kWarmThreads, smem, s>>>(wa);
    return cudaGetLastError();
}

}  // namespace kvd
