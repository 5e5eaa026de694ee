// k_append.cu — decode-time append (DESIGN.md §3 R16; the oracle's O13).
//
// "In the subsequent decoding phase, tokens are generated autoregressively, with each step
// appending new key and value vectors to the cache".  kvd_append_token writes one
// new token per request of a layer at position n_r: the token falls in the always-resident local
// window.  When it opens a new block b (n_r % P == 0) that block is admitted like a miss: a fully
// resident cache keeps block b in slot b; a host-backed cache takes the lowest free slot of the
// layer-head's window, else evicts the resident block with the smallest policy key among those
// not pinned after the append (LRU / LFU / lookahead on the layer's last scores).  The token's
// K / V rows go to the block's slot record (and to the host store record of a host-backed cache),
// and the block's summary is recomputed from its records' keys exactly as kvd_load_prefix computes
// it (mean: fp32 sum in token order, IEEE divide, bf16 RNE; min/max: channel-wise).  One CTA per
// (KV head, request); the layer's token count grows by one.
#include "resolve.cuh"

namespace kvd {

struct AppendArgs {
    const uint16_t* k;              // [B][Hkv][128] bf16 (device)
    const uint16_t* v;
    int32_t* ntok;                  // [R] token counts of the layer
    int32_t n[KVD_MAX_BATCH];       // token count of each request before the append (host copy)
    int64_t nb_max;
    int32_t resident, kind;
    const uint8_t* zero;            // unused
    uint8_t* host_store;            // NULL: resident
    uint16_t* summ;
    uint16_t* summ2;                // NULL unless min/max summaries
};

constexpr int kAppendThreads = 256;

__global__ void __launch_bounds__(kAppendThreads) append_kernel(StepParams p, ResolveBufs rb, AppendArgs aa,
                                                                uint8_t* __restrict__ slots) {
    __shared__ int scan[33];
    __shared__ int s_dest, s_victim;
    __shared__ unsigned long long s_best;
    const int h = blockIdx.x, bi = blockIdx.y, tid = threadIdx.x;
    const int r = p.req[bi];
    const int n = aa.n[bi];
    const int lp = __ffs(p.P) - 1;
    const int b = n >> lp, o = n & (p.P - 1);
    const SegGeom g = seg_geom(n + 1, p.P, p.sink_tokens, p.local_tokens);   // after the append
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    int32_t* table = rb.table + seg * p.nb_pad;
    int32_t* sb = rb.slot_block + seg * p.C;
    uint32_t* lu = rb.last_use + seg * p.C;
    uint8_t* ph = rb.phase + seg * p.C;
    uint32_t* uc = rb.use_count + seg * p.C;
    const float* sc = rb.scores + seg * p.nb_pad;
    const int64_t Ceff = rb.cap ? (int64_t)rb.cap[p.layer * p.Hkv + h] : p.C;
    griddep_wait();
    if (o == 0) {                                 // the token opens block b: admit it
        if (tid == 0) {
            s_dest = -1;
            s_victim = -1;
            s_best = ~0ull;
        }
        __syncthreads();
        if (aa.resident) {
            if (tid == 0) s_dest = b;
        } else {
            for (int base = 0; base < Ceff; base += kAppendThreads) {   // lowest free slot
                const int64_t s = base + tid;
                const int fr = (s < Ceff && sb[s] < 0) ? 1 : 0;
                int tot;
                const int pos = block_exclusive_scan(fr, scan, &tot);
                if (fr && pos == 0 && s_dest < 0) s_dest = (int)s;
                __syncthreads();
                if (s_dest >= 0) break;
            }
            if (s_dest < 0) {                     // victim: smallest policy key, not pinned after the append
                for (int64_t s = tid; s < Ceff; s += kAppendThreads) {
                    const int32_t blk = sb[s];
                    if (blk >= 0 && blk < b && blk >= g.sink_end && blk < g.local_begin) {
                        const uint64_t key = victim_key(p.policy, lu[s], ph[s], uc[s], blk, sc[blk], rb.err);
                        atomicMin(&s_best, (unsigned long long)key);
                    }
                }
                __syncthreads();
                for (int64_t s = tid; s < Ceff; s += kAppendThreads) {
                    const int32_t blk = sb[s];
                    if (blk >= 0 && blk < b && blk >= g.sink_end && blk < g.local_begin &&
                        victim_key(p.policy, lu[s], ph[s], uc[s], blk, sc[blk], rb.err) == s_best) {
                        s_dest = (int)s;          // keys are unique (the block id is part of every key)
                        s_victim = blk;
                    }
                }
            }
        }
        __syncthreads();
        const int dest = s_dest;
        if (dest < 0) {
            if (tid == 0) atomicOr(rb.err, 8);    // nothing evictable (C too small for the pinned set)
            return;
        }
        if (tid == 0) {
            if (s_victim >= 0) table[s_victim] = -1;
            table[b] = dest;
            sb[dest] = b;
            lu[dest] = p.step_dev ? *p.step_dev : p.step;
            ph[dest] = 1;
            uc[dest] = 1;
        }
        // a fresh record: zero rows (the new token's row is written below)
        uint8_t* rec = slots + (seg * p.C + dest) * (int64_t)p.rec_bytes;
        for (int c = tid; c < p.rec_bytes / 16; c += kAppendThreads) reinterpret_cast<int4*>(rec)[c] = make_int4(0, 0, 0, 0);
        if (aa.host_store) {
            uint8_t* hrec = aa.host_store + (((int64_t)p.layer * p.R + r) * p.Hkv + h) * aa.nb_max * p.rec_bytes +
                            (int64_t)b * p.rec_bytes;
            for (int c = tid; c < p.rec_bytes / 16; c += kAppendThreads)
                reinterpret_cast<int4*>(hrec)[c] = make_int4(0, 0, 0, 0);
        }
        __syncthreads();
    }
    const int slot = aa.resident ? b : table[b];  // the local block is resident
    uint8_t* rec = slots + (seg * p.C + slot) * (int64_t)p.rec_bytes;
    uint8_t* hrec = aa.host_store ? aa.host_store + (((int64_t)p.layer * p.R + r) * p.Hkv + h) * aa.nb_max * p.rec_bytes +
                                        (int64_t)b * p.rec_bytes
                                  : nullptr;
    if (tid < 32) {                               // row o of K (chunks 0..15) and V (16..31), swizzled
        const int half = tid >> 4, cc = tid & 15;
        const uint16_t* src = (half ? aa.v : aa.k) + ((int64_t)bi * p.Hkv + h) * kHeadDim + cc * 8;
        const int4 x = *reinterpret_cast<const int4*>(src);
        const int64_t off = (int64_t)half * p.P * kRowBytes + (int64_t)o * kRowBytes + ((cc ^ (o & 7)) * 16);
        *reinterpret_cast<int4*>(rec + off) = x;
        if (hrec) *reinterpret_cast<int4*>(hrec + off) = x;
    }
    __syncthreads();
    if (tid < kHeadDim) {                         // the block's summary over its o + 1 tokens (R2 / R30)
        const int j = tid;
        auto key_at = [&](int t) {                // K[t][j] of the block, from the record
            const uint16_t* row = reinterpret_cast<const uint16_t*>(rec + (int64_t)t * kRowBytes);
            return row[(((j >> 3) ^ (t & 7)) << 3) + (j & 7)];
        };
        const int64_t col = seg * kHeadDim * p.nb_pad + (int64_t)j * p.nb_pad + b;
        if (aa.kind == 0) {
            float acc = 0.0f;
            for (int t = 0; t <= o; ++t) acc = __fadd_rn(acc, bf16_bits(key_at(t)));
            aa.summ[col] = f32_to_bf16_rne(__fdiv_rn(acc, (float)(o + 1)));
        } else {
            uint16_t lo = key_at(0), hi = lo;
            for (int t = 1; t <= o; ++t) {
                const uint16_t x = key_at(t);
                if (bf16_bits(x) < bf16_bits(lo)) lo = x;
                if (bf16_bits(x) > bf16_bits(hi)) hi = x;
            }
            aa.summ[col] = lo;
            aa.summ2[col] = hi;
        }
    }
    if (h == 0 && tid == 0) aa.ntok[r] = n + 1;
}

cudaError_t launch_append(kvd_cache* c, const StepParams& p, const uint16_t* k, const uint16_t* v, const int32_t* n,
                          cudaStream_t s) {
    AppendArgs aa{};
    aa.k = k;
    aa.v = v;
    aa.ntok = c->ntok_dev + (int64_t)p.layer * c->R;
    for (int b = 0; b < p.B; ++b) aa.n[b] = n[b];
    aa.nb_max = c->nb_max;
    aa.resident = c->resident ? 1 : 0;
    aa.kind = c->summary_kind;
    aa.host_store = c->resident ? nullptr : c->host_store;
    aa.summ = c->summ;
    aa.summ2 = c->summ2;
    const ResolveBufs rb = resolve_bufs(c, p.layer);
    count_launch();
    append_kernel<<<dim3(p.Hkv, p.B), kAppendThreads, 0, s>>>(p, rb, aa, c->slots);
    return cudaGetLastError();
}

}  // namespace kvd
