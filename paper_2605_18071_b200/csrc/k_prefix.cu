// k_prefix.cu — row (a0): prefix ingest.  Builds the per-block mean-key
// summaries ("the mean key of each page is used as its
// representative"), packs K/V into swizzled block records and resets the
// segment's block table and slot metadata.  Setup only; not in the decode step.
#include "common.cuh"
#include "internal.h"

namespace kvd {

// Summary of block b, dim j: acc = +0; for t < cnt: acc += K[P b + t][j] (fp32,
// token order); S = bf16_rne(acc / cnt) with an IEEE divide (DESIGN.md §3 R2).
// grid (nb_pad / 32, Hkv), block 128 threads = dims; each CTA handles 32
// consecutive blocks and transposes through smem so the dim-major rows are
// written 64 B at a time.
// kind 0: mean key (R2); kind 1: Quest channel-wise minimum -> summ_lr, maximum -> summ2_lr (R30;
// exact: a min / max of bf16 values is one of them; strict comparisons keep the first of equals)
__global__ void __launch_bounds__(128) summary_kernel(const uint16_t* __restrict__ K, int64_t n, int P,
                                                      int64_t nb_pad, uint16_t* __restrict__ summ_lr,
                                                      uint16_t* __restrict__ summ2_lr, int kind) {
    __shared__ uint16_t tile[128][33];
    __shared__ uint16_t tile2[128][33];
    const int j = threadIdx.x;
    const int h = blockIdx.y;
    const int64_t b0 = (int64_t)blockIdx.x * 32;
    const int64_t nb = (n + P - 1) / P;
    const uint16_t* Kh = K + (int64_t)h * n * kHeadDim;
    for (int i = 0; i < 32; ++i) {
        int64_t b = b0 + i;
        uint16_t out = 0;
        if (b < nb) {
            int64_t cnt = n - (int64_t)P * b;
            if (cnt > P) cnt = P;
            if (kind == 0) {
                float acc = 0.0f;
                for (int64_t t = 0; t < cnt; ++t) acc = __fadd_rn(acc, bf16_bits(Kh[((int64_t)P * b + t) * kHeadDim + j]));
                out = f32_to_bf16_rne(__fdiv_rn(acc, (float)cnt));
            } else {
                uint16_t lo = Kh[((int64_t)P * b) * kHeadDim + j], hi = lo;
                for (int64_t t = 1; t < cnt; ++t) {
                    const uint16_t x = Kh[((int64_t)P * b + t) * kHeadDim + j];
                    if (bf16_bits(x) < bf16_bits(lo)) lo = x;
                    if (bf16_bits(x) > bf16_bits(hi)) hi = x;
                }
                out = lo;
                tile2[j][i] = hi;
            }
        }
        tile[j][i] = out;
        if (kind == 0 || b >= nb) tile2[j][i] = 0;
    }
    __syncthreads();
    // write rows: for each dim jj, 32 consecutive blocks (64 B)
    uint16_t* base = summ_lr + (int64_t)h * kHeadDim * nb_pad;
    uint16_t* base2 = summ2_lr ? summ2_lr + (int64_t)h * kHeadDim * nb_pad : nullptr;
    for (int e = threadIdx.x; e < 128 * 32; e += 128) {
        int jj = e >> 5, i = e & 31;
        if (b0 + i < nb_pad) {
            base[(int64_t)jj * nb_pad + b0 + i] = tile[jj][i];
            if (base2) base2[(int64_t)jj * nb_pad + b0 + i] = tile2[jj][i];
        }
    }
}

// Pack block records.  One CTA per (block, head); 128 threads move 16-byte
// chunks.  dst record for block b of head h at dst + (h * dst_head_stride + b) *
// rec_bytes, or (if slot_of != nullptr) at slot slot_of[h * nb + b] (skipped if < 0).
// Rows past the end of the prefix are zero.
__global__ void __launch_bounds__(128) record_kernel(const uint16_t* __restrict__ K, const uint16_t* __restrict__ V,
                                                     int64_t n, int P, uint8_t* __restrict__ dst,
                                                     int64_t dst_head_stride, int rec_bytes,
                                                     const int32_t* __restrict__ slot_of, int64_t nb) {
    const int64_t b = blockIdx.x;
    const int h = blockIdx.y;
    int64_t didx = b;
    if (slot_of) {
        didx = slot_of[(int64_t)h * nb + b];
        if (didx < 0) return;
    }
    uint8_t* rec = dst + ((int64_t)h * dst_head_stride + didx) * rec_bytes;
    const int chunks = rec_bytes / 16;           // 2 * P * 16
    for (int c = threadIdx.x; c < chunks; c += blockDim.x) {
        int half = c / (P * 16);                 // 0 = K, 1 = V
        int t = (c / 16) % P;                    // token row inside the block
        int cc = c % 16;                         // logical 16-B chunk (8 dims)
        int64_t tok = (int64_t)P * b + t;
        int4 v = make_int4(0, 0, 0, 0);
        if (tok < n) {
            const uint16_t* src = (half ? V : K) + ((int64_t)h * n + tok) * kHeadDim + cc * 8;
            v = *reinterpret_cast<const int4*>(src);
        }
        int phys = cc ^ (t & 7);
        *reinterpret_cast<int4*>(rec + half * P * kRowBytes + t * kRowBytes + phys * 16) = v;
    }
}

// Reset one (layer, request)'s segment tables.  grid Hkv, block 256.
// resident: block b <-> slot b.  cold: pinned blocks (ascending) in slots 0..p-1.
// Also writes slot_of[h][b] (destination slot for record packing, -1 = none).
__global__ void table_init_kernel(int32_t* __restrict__ table_lr, int32_t* __restrict__ sb_lr,
                                  uint32_t* __restrict__ lu_lr, uint8_t* __restrict__ ph_lr,
                                  uint32_t* __restrict__ uc_lr, int32_t* __restrict__ slot_of, int64_t nb_pad,
                                  int64_t C, SegGeom g, int resident) {
    const int h = blockIdx.x;
    int32_t* table = table_lr + (int64_t)h * nb_pad;
    int32_t* sb = sb_lr + (int64_t)h * C;
    const int32_t p_sink = g.sink_end;
    for (int64_t b = threadIdx.x; b < nb_pad; b += blockDim.x) {
        int32_t s = -1;
        if (b < g.nb) {
            if (resident) s = (int32_t)b;
            else if (b < g.sink_end) s = (int32_t)b;
            else if (b >= g.local_begin) s = p_sink + (int32_t)(b - g.local_begin);
        }
        table[b] = s;
        if (b < g.nb) slot_of[(int64_t)h * g.nb + b] = s;
    }
    for (int64_t s = threadIdx.x; s < C; s += blockDim.x) {
        int32_t blk = -1;
        if (resident) blk = s < g.nb ? (int32_t)s : -1;
        else if (s < p_sink) blk = (int32_t)s;
        else if (s < p_sink + (g.nb - g.local_begin)) blk = g.local_begin + (int32_t)(s - p_sink);
        sb[s] = blk;
        lu_lr[(int64_t)h * C + s] = 0u;
        ph_lr[(int64_t)h * C + s] = 0;
        uc_lr[(int64_t)h * C + s] = 0u;
    }
}

__global__ void set_ntok_kernel(int32_t* ntok, int req, int32_t n) { ntok[req] = n; }

cudaError_t launch_prefix(kvd_cache* c, int layer, int req, const uint16_t* dk, const uint16_t* dv, int64_t n,
                          cudaStream_t s, const uint16_t* dq_obs, int n_obs) {
    const int64_t sl = ((int64_t)layer * c->R + req) * c->Hkv;      // first segment of (layer, req)
    SegGeom g = seg_geom(n, c->P, c->cfg.sink_tokens, c->cfg.local_tokens);
    summary_kernel<<<dim3((unsigned)(c->nb_pad / 32), c->Hkv), 128, 0, s>>>(
        dk, n, c->P, c->nb_pad, c->summ + sl * kHeadDim * c->nb_pad,
        c->summ2 ? c->summ2 + sl * kHeadDim * c->nb_pad : nullptr, c->summary_kind);
    // slot_of scratch: the first kSlotOfBytes of stage_rec
    int32_t* slot_of = reinterpret_cast<int32_t*>(c->stage_rec);
    table_init_kernel<<<c->Hkv, 256, 0, s>>>(c->table + sl * c->nb_pad, c->slot_block + sl * c->C,
                                             c->last_use + sl * c->C, c->phase + sl * c->C,
                                             c->use_count + sl * c->C, slot_of, c->nb_pad, c->C, g,
                                             c->resident ? 1 : 0);
    if (dq_obs && n_obs > 0 && !c->resident) {    // importance-guided warm-up (k_warm.cu, R29)
        cudaError_t e = launch_warm(c, layer, req, dk, dq_obs, n_obs, n, slot_of, s);
        if (e != cudaSuccess) return e;
    }
    dim3 rg((unsigned)g.nb, c->Hkv);
    // resident blocks / pinned blocks -> their slots
    record_kernel<<<rg, 128, 0, s>>>(dk, dv, n, c->P, c->slots + sl * c->C * c->rec_bytes, c->C, (int)c->rec_bytes,
                                     slot_of, g.nb);
    if (!c->resident && layer < c->A) {
        // all blocks -> device staging records, then D2H into the pinned host store
        // (host layer = layer; layers >= A alias host layer layer % A, kvd.h)
        uint8_t* recs = c->stage_rec + kSlotOfBytes;
        record_kernel<<<rg, 128, 0, s>>>(dk, dv, n, c->P, recs, g.nb, (int)c->rec_bytes, nullptr, g.nb);
        {
            for (int h = 0; h < c->Hkv; ++h) {
                uint8_t* dst = c->host_store +
                               ((((int64_t)layer * c->R + req) * c->Hkv + h) * c->nb_max) * c->rec_bytes;
                const cudaError_t e = cudaMemcpyAsync(dst, recs + (int64_t)h * g.nb * c->rec_bytes,
                                                      (size_t)g.nb * c->rec_bytes, cudaMemcpyDeviceToHost, s);
                if (e != cudaSuccess) return e;
            }
        }
    }
    set_ntok_kernel<<<1, 1, 0, s>>>(c->ntok_dev + (int64_t)layer * c->R, req, (int32_t)n);
    return cudaGetLastError();
}

}  // namespace kvd
