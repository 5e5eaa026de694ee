// k_index.cu — the hierarchical centroid index (DESIGN.md §3 R27).
//
// "the mean key of each page is used as its representative, forming higher-level
// centroids for similarity grouping ... this hierarchical structure preserves local
// semantic continuity among contiguous tokens"; "KVDrive achieves
// comparable accuracy to spatial-chunking methods using only half as many centroids,
// significantly reducing selection latency".
//
// Build (row a0, kvd_load_prefix; the oracle's O9): the block summaries of a segment are
// clustered by Lloyd k-means inside windows of kIdxWindow = 64 consecutive blocks into
// ceil(len / ratio) centroids per window -- deterministic init (block floor(i*len/nw)),
// kIdxIters (assign, update) rounds then a final assignment, fp32 in the oracle's order,
// centroids without members dropped -- index_kmeans_kernel, one CTA per window; then
// index_finish_kernel numbers the centroids window by window, stores them bf16 dim-major
// (the layout of the block summaries, so stage 1 is the same streaming scan), and builds the
// member lists (blocks ordered by (centroid, block): a centroid's members are one range).
//
// Select (rows a1 + a2, the oracle's O10): stage 1 runs select_kernel over the segment's
// centroid matrix (k-means centroids scored exactly like blocks, fp32 FMA chain) and keeps the
// m = min(nc, max(ceil(4k/ratio), k + pinned)) best centroids.  Stage 2, cand_kernel, one CTA
// per segment: marks the non-pinned members of those centroids in a bitmap, compacts them in
// ascending block order, scores them exactly (the flat path's arithmetic), and takes the top k
// (score desc, block asc) by an 8-bit radix select over their keys -- emitted ascending by a
// scan, since candidates are already in block order.  Fused (kvd_select_resolve_fetch), the same
// CTA then resolves the segment and copies its misses (resolve.cuh), as the flat select does.
// Bytes per segment: 256 B per centroid + ~256 B x 4k candidate blocks, against 256 B x nb flat
// (c4: 4.3 MB against 16.8 MB).
#include <algorithm>

#include "resolve.cuh"

namespace kvd {

// ---------------------------------------------------------------- build (O9)
struct IndexStage {                 // setup scratch, per head of one (layer, request)
    uint16_t* cent;                 // [Hkv][nwin][64][128] bf16, window-local centroids
    int32_t* as;                    // [Hkv][nb_pad] window-local centroid of each block
    int32_t* cnt;                   // [Hkv][nwin][64] members per window-local centroid
    int32_t* nonempty;              // [Hkv][nwin]
};

// grid (nwin, Hkv), 128 threads: thread j owns dim j in the update; thread b < len owns block b
// in the assignment.
__global__ void __launch_bounds__(128) index_kmeans_kernel(const uint16_t* __restrict__ summ, int64_t nb_pad, int nb,
                                                           int ratio, IndexStage st) {
    extern __shared__ float kmem[];               // x [64][129] | cc [64][129] (+1: conflict-free by block)
    float (*x)[kHeadDim + 1] = reinterpret_cast<float (*)[kHeadDim + 1]>(kmem);
    float (*cc)[kHeadDim + 1] = reinterpret_cast<float (*)[kHeadDim + 1]>(kmem + kIdxWindow * (kHeadDim + 1));
    __shared__ int as[kIdxWindow];
    __shared__ int cnt[kIdxWindow];
    const int w = blockIdx.x, h = blockIdx.y, tid = threadIdx.x;
    const int64_t w0 = (int64_t)w * kIdxWindow;
    const int len = (int)(nb - w0 < kIdxWindow ? nb - w0 : kIdxWindow);
    const int nw = (len + ratio - 1) / ratio;
    const uint16_t* sh = summ + (int64_t)h * kHeadDim * nb_pad;
    for (int b = 0; b < len; ++b) x[b][tid] = bf16_bits(sh[(int64_t)tid * nb_pad + w0 + b]);
    __syncthreads();
    for (int i = 0; i < nw; ++i) cc[i][tid] = x[(int)(((int64_t)i * len) / nw)][tid];
    __syncthreads();
    for (int it = 0; it <= kIdxIters; ++it) {
        if (tid < len) {                          // assign: argmin fp32 distance, ties -> lowest
            int best = 0;
            float bd = 0.0f;
            for (int i = 0; i < nw; ++i) {
                float acc = 0.0f;
                for (int j = 0; j < kHeadDim; ++j) {
                    const float diff = __fsub_rn(x[tid][j], cc[i][j]);
                    acc = __fmaf_rn(diff, diff, acc);
                }
                if (i == 0 || acc < bd) {
                    bd = acc;
                    best = i;
                }
            }
            as[tid] = best;
        }
        __syncthreads();
        if (it == kIdxIters) break;               // final assignment only
        for (int i = 0; i < nw; ++i) {            // update: member mean, block order, IEEE divide
            int n = 0;
            float acc = 0.0f;
            for (int b = 0; b < len; ++b)
                if (as[b] == i) {
                    ++n;
                    acc = __fadd_rn(acc, x[b][tid]);
                }
            if (n > 0) cc[i][tid] = __fdiv_rn(acc, (float)n);
        }
        __syncthreads();
    }
    if (tid < nw) {
        int n = 0;
        for (int b = 0; b < len; ++b) n += as[b] == tid;
        cnt[tid] = n;
    }
    __syncthreads();
    const int64_t wi = (int64_t)h * (nb_pad / kIdxWindow) + w;
    for (int i = 0; i < nw; ++i) st.cent[(wi * kIdxWindow + i) * kHeadDim + tid] = f32_to_bf16_rne(cc[i][tid]);
    if (tid < len) st.as[(int64_t)h * nb_pad + w0 + tid] = as[tid];
    if (tid < nw) st.cnt[wi * kIdxWindow + tid] = cnt[tid];
    if (tid == 0) {
        int ne = 0;
        for (int i = 0; i < nw; ++i) ne += cnt[i] > 0;
        st.nonempty[wi] = ne;
    }
}

struct IndexOut {                   // the segment buffers of head 0 of (layer, request)
    uint16_t* cent;                 // [Hkv][128][nc_pad]
    int32_t* ncent;                 // [Hkv]
    int32_t* cent_of;               // [Hkv][nb_pad]
    int32_t* memb;                  // [Hkv][nb_pad]
    int32_t* moff;                  // [Hkv][nc_pad + 1]
};

// grid (Hkv), 1024 threads: number the non-empty centroids window by window, store them
// dim-major, block -> centroid map, member lists ordered by (centroid, block).
__global__ void __launch_bounds__(1024) index_finish_kernel(int64_t nb_pad, int64_t nc_pad, int nb, int ratio,
                                                            IndexStage st, IndexOut io) {
    __shared__ int scan[33];
    extern __shared__ int wbase[];                // [nwin]
    const int h = blockIdx.x, tid = threadIdx.x;
    const int nwin = (nb + kIdxWindow - 1) / kIdxWindow;
    const int64_t wpad = nb_pad / kIdxWindow;
    int carry = 0;
    for (int w0 = 0; w0 < nwin; w0 += blockDim.x) {
        const int w = w0 + tid;
        const int v = w < nwin ? st.nonempty[h * wpad + w] : 0;
        int tot;
        const int pos = block_exclusive_scan(v, scan, &tot);
        if (w < nwin) wbase[w] = carry + pos;
        carry += tot;
    }
    __syncthreads();
    const int nc = carry;
    uint16_t* cent = io.cent + (int64_t)h * kHeadDim * nc_pad;
    int32_t* cent_of = io.cent_of + (int64_t)h * nb_pad;
    int32_t* memb = io.memb + (int64_t)h * nb_pad;
    int32_t* moff = io.moff + (int64_t)h * (nc_pad + 1);
    for (int w = tid; w < nwin; w += blockDim.x) {
        const int64_t w0 = (int64_t)w * kIdxWindow;
        const int len = (int)(nb - w0 < kIdxWindow ? nb - w0 : kIdxWindow);
        const int nw = (len + ratio - 1) / ratio;
        const int64_t wi = h * wpad + w;
        int newid[kIdxWindow];
        int id = wbase[w], off = 0;
        for (int i = 0; i < nw; ++i) {
            const int n = st.cnt[wi * kIdxWindow + i];
            newid[i] = n > 0 ? id : -1;
            if (n == 0) continue;
            moff[id] = (int32_t)(w0 + off);
            for (int j = 0; j < kHeadDim; ++j) cent[(int64_t)j * nc_pad + id] = st.cent[(wi * kIdxWindow + i) * kHeadDim + j];
            for (int b = 0; b < len; ++b)
                if (st.as[h * nb_pad + w0 + b] == i) memb[w0 + off++] = (int32_t)(w0 + b);
            ++id;
        }
        for (int b = 0; b < len; ++b) cent_of[w0 + b] = newid[st.as[h * nb_pad + w0 + b]];
    }
    if (tid == 0) {
        moff[nc] = nb;
        io.ncent[h] = nc;
    }
}

cudaError_t launch_index_build(kvd_cache* c, int layer, int req, int64_t n, cudaStream_t s) {
    const SegGeom g = seg_geom(n, c->P, c->cfg.sink_tokens, c->cfg.local_tokens);
    const int64_t sl = ((int64_t)layer * c->R + req) * c->Hkv;      // first segment of (layer, req)
    const int nwin = (g.nb + kIdxWindow - 1) / kIdxWindow;
    const int64_t wpad = c->nb_pad / kIdxWindow;
    uint8_t* p = c->idx_stage;
    IndexStage st;
    st.cent = reinterpret_cast<uint16_t*>(p);
    p += (size_t)c->Hkv * wpad * kIdxWindow * kHeadDim * 2;
    st.as = reinterpret_cast<int32_t*>(p);
    p += (size_t)c->Hkv * c->nb_pad * 4;
    st.cnt = reinterpret_cast<int32_t*>(p);
    p += (size_t)c->Hkv * wpad * kIdxWindow * 4;
    st.nonempty = reinterpret_cast<int32_t*>(p);
    constexpr size_t ksmem = 2 * sizeof(float) * kIdxWindow * (kHeadDim + 1);
    static bool attr[64] = {};
    if (!attr[c->cfg.device & 63]) {
        cudaError_t e = cudaFuncSetAttribute(index_kmeans_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ksmem);
        if (e != cudaSuccess) return e;
        attr[c->cfg.device & 63] = true;
    }
    index_kmeans_kernel<<<dim3((unsigned)nwin, c->Hkv), 128, ksmem, s>>>(c->summ + sl * kHeadDim * c->nb_pad, c->nb_pad,
                                                                        g.nb, c->index_ratio, st);
    IndexOut io{c->cent + sl * kHeadDim * c->nc_pad, c->ncent + sl, c->cent_of + sl * c->nb_pad,
                c->memb + sl * c->nb_pad, c->moff + sl * (c->nc_pad + 1)};
    index_finish_kernel<<<c->Hkv, 1024, (size_t)nwin * 4, s>>>(c->nb_pad, c->nc_pad, g.nb, c->index_ratio, st, io);
    return cudaGetLastError();
}

size_t index_stage_bytes(int Hkv, int64_t nb_pad) {
    const int64_t wpad = nb_pad / kIdxWindow;
    return (size_t)Hkv * (wpad * kIdxWindow * kHeadDim * 2 + nb_pad * 4 + wpad * kIdxWindow * 4 + wpad * 4);
}

// ---------------------------------------------------------------- select stage 2 (O10)
constexpr int kCandThreads = 1024;

struct CandArgs {
    FuseArgs fa;                    // fused resolve + fetch (fa.out_attn == NULL: select only)
    const uint16_t* summ;
    float* scores;                  // [seg][nb_pad]: exact scores of this step's candidates
    uint32_t* cand_bits;            // [seg][nb_pad / 32]: this step's candidates (lookahead victims)
    const float* cscores;           // [seg][nc_pad]
    const int32_t* csel;            // [R][Hkv][m_max] stage-1 centroids
    const int32_t* ncent;
    const int32_t* cent_of;
    const int32_t* memb;
    const int32_t* moff;
    int64_t nc_pad;
    int32_t m_max, ratio;
};

// dynamic smem: [nb_pad/32] candidate bitmap | [kCandCap] candidate ids | [kCandCap] keys;
// the fused resolve reuses it from offset 0 afterwards.
size_t cand_smem_bytes(int64_t nb_pad) { return (size_t)nb_pad / 8 + (size_t)kCandCap * 8; }

template <bool RESOLVE>
__global__ void __launch_bounds__(kCandThreads, 1) cand_kernel(CandArgs ca, StepParams p, const uint16_t* __restrict__ q,
                                                               const int32_t* __restrict__ ntok,
                                                               int32_t* __restrict__ out_ids,
                                                               float* __restrict__ out_scores) {
    extern __shared__ __align__(16) uint32_t bits[];
    __shared__ float qbar[kHeadDim];
    __shared__ int scan[33];
    __shared__ int hist[256];
    __shared__ int s_digit, s_above;
    __shared__ ResolveShared rsm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int h = p.h0 + blockIdx.x, bi = blockIdx.y;
    const int r = p.req[bi];
    const int64_t seg = ((int64_t)p.layer * p.R + r) * p.Hkv + h;
    const SegGeom g = seg_geom(ntok[r], p.P, p.sink_tokens, p.local_tokens);
    const int nb = g.nb;
    const int nwords = (nb + 31) >> 5;
    int32_t* cand = reinterpret_cast<int32_t*>(bits + p.nb_pad / 32);
    uint32_t* keys = reinterpret_cast<uint32_t*>(cand + kCandCap);
    if (RESOLVE) resolve_pre(p, ca.fa.rb, bi, h, rsm);
    for (int w = tid; w < nwords; w += kCandThreads) bits[w] = 0u;
    if (tid == 0) EXP_STAMP(p.exp_trace, 8192 + bi * p.Hkv + h, 0);
    griddep_wait();                               // stage-1 selection and scores; q
    if (tid == 0) kt_begin(p.kt_slots, p.kt_base + kKtSelect);
    if (tid == 0) EXP_STAMP(p.exp_trace, 8192 + bi * p.Hkv + h, 1);
    if (tid < kHeadDim) {
        const uint16_t* qh = q + ((int64_t)bi * p.Hq + (int64_t)h * p.G) * kHeadDim;
        float a = 0.0f;
        for (int gq = 0; gq < p.G; ++gq) a = __fadd_rn(a, bf16_bits(qh[gq * kHeadDim + tid]));
        qbar[tid] = a;                            // R3
    }
    const int nc = ca.ncent[seg];
    const int pin = g.sink_end + (g.nb - g.local_begin);
    const int m = min(nc, max((kIdxFanout * p.k + ca.ratio - 1) / ca.ratio, p.k + pin));
    __syncthreads();
    // ---- candidates: non-pinned members of the m chosen centroids.  Thread i < m owns chosen
    // centroid i: one round trip for the ids, one for the member ranges, then its members
    // (contiguous in memb, independent loads) are marked in the bitmap.
    const int32_t* sel = ca.csel + ((int64_t)r * p.Hkv + h) * ca.m_max;   // per request id (see select.cuh)
    const int32_t* moff = ca.moff + seg * (ca.nc_pad + 1);
    const int32_t* memb = ca.memb + seg * p.nb_pad;
    if (tid < m) {
        const int cidx = __ldcg(&sel[tid]);
        const int a = moff[cidx], e = moff[cidx + 1];
        for (int x = a; x < e; ++x) {
            const int b = memb[x];
            if (b >= g.sink_end && b < g.local_begin) atomicOr(&bits[b >> 5], 1u << (b & 31));
        }
    }
    __syncthreads();
    // ---- compact them in ascending block order
    int ncand = 0;
    for (int w0 = 0; w0 < nwords; w0 += kCandThreads) {
        const int w = w0 + tid;
        uint32_t word = w < nwords ? bits[w] : 0u;
        int tot;
        const int pos = ncand + block_exclusive_scan(__popc(word), scan, &tot);
        int o = pos;
        while (word) {
            const int bit = __ffs(word) - 1;
            if (o < kCandCap) cand[o] = (w << 5) + bit;
            ++o;
            word &= word - 1u;
        }
        ncand += tot;
    }
    if (ncand > kCandCap || ncand < p.k) {        // impossible by the fan-out rule (R27)
        if (tid == 0) atomicOr(ca.fa.rb.err, 4);
        ncand = min(ncand, kCandCap);
    }
    if (tid == 0) EXP_STAMP(p.exp_trace, 8192 + bi * p.Hkv + h, 2);
    // ---- this step's candidate set, for the lookahead victim keys (resolve.cuh)
    uint32_t* gbits = ca.cand_bits + seg * (p.nb_pad >> 5);
    for (int w = tid; w < nwords; w += kCandThreads) gbits[w] = bits[w];
    float* sc = ca.scores + seg * p.nb_pad;
    __syncthreads();
    if (tid == 0) EXP_STAMP(p.exp_trace, 8192 + bi * p.Hkv + h, 3);
    // ---- exact scores of the candidates (fp32 FMA chain over j = 0..127, R5)
    const uint16_t* sseg = ca.summ + seg * kHeadDim * p.nb_pad;
    for (int c0 = 0; c0 < ncand; c0 += kCandThreads) {
        const int ci = c0 + tid;
        const bool v = ci < ncand;
        const int b = v ? cand[ci] : 0;
        float acc = 0.0f;
#pragma unroll 1
        for (int j0 = 0; j0 < kHeadDim; j0 += 32) {
            uint16_t row[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) row[u] = v ? __ldcs(sseg + (int64_t)(j0 + u) * p.nb_pad + b) : (uint16_t)0;
#pragma unroll
            for (int u = 0; u < 32; ++u) acc = __fmaf_rn(qbar[j0 + u], bf16_bits(row[u]), acc);
        }
        if (v) {
            keys[ci] = score_key32(acc);
            sc[b] = acc;
        }
    }
    __syncthreads();
    if (tid == 0) EXP_STAMP(p.exp_trace, 8192 + bi * p.Hkv + h, 4);
    // ---- top k of the candidates: 8-bit radix select of the k-th largest key T, then every key
    // above T and the first (k - #above) keys equal to T in candidate (= block) order
    uint32_t prefix = 0u, mask = 0u;
    int kk = p.k;
    for (int shift = 24; shift >= 0 && kk > 0; shift -= 8) {
        for (int i = tid; i < 256; i += kCandThreads) hist[i] = 0;
        __syncthreads();
        for (int c0 = 0; c0 < ncand; c0 += kCandThreads) {
            const int ci = c0 + tid;
            const uint32_t key = ci < ncand ? keys[ci] : 0u;
            warp_hist_add(hist, (key >> shift) & 255u, ci < ncand && (key & mask) == prefix);
        }
        __syncthreads();
        if (warp == 0) {                          // descending bins: lane l owns bins 255-8l-j
            int c8[8], t = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                c8[j] = hist[255 - (8 * lane + j)];
                t += c8[j];
            }
            int incl = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int above = incl - t;
            if (above < kk && kk <= incl) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (above + c8[j] >= kk) {
                        s_digit = 255 - (8 * lane + j);
                        s_above = above;
                        break;
                    }
                    above += c8[j];
                }
            }
        }
        __syncthreads();
        prefix |= (uint32_t)s_digit << shift;
        mask |= 255u << shift;
        kk -= s_above;
        __syncthreads();
    }
    const uint32_t T = prefix;                    // the k-th largest key; kk of the keys == T taken
    if (tid == 0) EXP_STAMP(p.exp_trace, 8192 + bi * p.Hkv + h, 5);
    int32_t* ids_out = out_ids + ((int64_t)bi * p.Hkv + h) * p.k;
    float* sc_out = out_scores ? out_scores + ((int64_t)bi * p.Hkv + h) * p.k : nullptr;
    int taken = 0, eqs = 0;
    for (int c0 = 0; c0 < ncand; c0 += kCandThreads) {
        const int ci = c0 + tid;
        const uint32_t key = ci < ncand ? keys[ci] : 0u;
        const bool eq = ci < ncand && key == T;
        int tot_eq;
        const int eq_rank = eqs + block_exclusive_scan(eq ? 1 : 0, scan, &tot_eq);
        const bool take = ci < ncand && (key > T || (eq && eq_rank < kk));
        int tot;
        const int pos = taken + block_exclusive_scan(take ? 1 : 0, scan, &tot);
        if (take) {
            ids_out[pos] = cand[ci];
            if (sc_out) sc_out[pos] = sc[cand[ci]];
        }
        taken += tot;
        eqs += tot_eq;
    }
    if (tid == 0) EXP_STAMP(p.exp_trace, 8192 + bi * p.Hkv + h, 6);
    if constexpr (RESOLVE) {
        __syncthreads();                          // ids written (read back by the resolve, L2)
        uint8_t* smraw = reinterpret_cast<uint8_t*>(bits);
        const int nm = resolve_main(p, ca.fa.rb, bi, h, out_ids, ca.fa.out_attn, smraw, rsm, true, false);
        if (nm > 0 && ca.fa.host_store) {
            const int32_t* S = reinterpret_cast<const int32_t*>(reinterpret_cast<uint64_t*>(smraw) + ca.fa.rb.nkeys);
            gather_segment(p, bi, h, S + 2 * ca.fa.rb.kmax, S + 3 * ca.fa.rb.kmax, nm, ca.fa.host_store, ca.fa.slots, 0, 1);
        }
    } else {
        griddep_launch();
    }
#ifdef KVD_EXPERIMENTS
    __syncthreads();
    if (tid == 0) EXP_STAMP(p.exp_trace, 8192 + bi * p.Hkv + h, 7);
#endif
    if (p.kt_slots) {
        __syncthreads();
        if (tid == 0) kt_end(p.kt_slots, p.kt_acc, p.kt_base + kKtSelect, kKtSelect, (unsigned long long)gridDim.x * gridDim.y);
    }
}

// stage 1 (select_kernel over the centroids) then stage 2 (cand_kernel, fused resolve + fetch
// when out_attn != NULL).  The kernel timer counts the two as one select launch... stage 1's
// timing slot is separate (kind select of the centroid launch) -- both are reported.
cudaError_t launch_index_select(kvd_cache* c, const StepParams& p, const uint16_t* q, int32_t* out_ids,
                                float* out_scores, int32_t* out_attn, cudaStream_t s) {
    StepParams p1 = p;
    p1.sel_mode = 1;
    p1.sel_ratio = c->index_ratio;
    p1.sel_stride = c->m_max;
    p1.sel_count = c->ncent;
    p1.nb_pad = c->nc_pad;                        // row stride of the centroid matrix
    cudaError_t e = launch_select_centroids(c, p1, q, s);
    if (e != cudaSuccess) return e;
    CandArgs ca;
    ca.fa.rb = resolve_bufs(c, p.layer);
    ca.fa.out_attn = out_attn;
    ca.fa.host_store = c->resident ? nullptr : c->host_store;
    ca.fa.slots = c->slots;
    ca.summ = c->summ;
    ca.scores = c->scores;
    ca.cand_bits = c->cand_bits;
    ca.cscores = c->cscores;
    ca.csel = c->csel;
    ca.ncent = c->ncent;
    ca.cent_of = c->cent_of;
    ca.memb = c->memb;
    ca.moff = c->moff;
    ca.nc_pad = c->nc_pad;
    ca.m_max = c->m_max;
    ca.ratio = c->index_ratio;
    const bool fused = out_attn != nullptr;
    size_t smem = cand_smem_bytes(c->nb_pad);
    if (fused) smem = std::max(smem, resolve_smem_bytes(ca.fa.rb.nkeys, c->kmax, c->nb_pad));
    static size_t smem_set[2][64] = {};
    const int dev = c->cfg.device & 63;
    if (smem > smem_set[fused][dev]) {
        e = fused ? cudaFuncSetAttribute(cand_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                  : cudaFuncSetAttribute(cand_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        smem_set[fused][dev] = smem;
    }
    const int prio = (fused && ca.fa.host_store) ? c->prio_hi : 0;
    e = fused ? launch_pdl_prio(prio, cand_kernel<true>, dim3(p.nh, p.B), dim3(kCandThreads), smem, s, ca, p, q,
                                (const int32_t*)c->ntok_dev + (int64_t)p.layer * c->R, out_ids, out_scores)
              : launch_pdl(cand_kernel<false>, dim3(p.nh, p.B), dim3(kCandThreads), smem, s, ca, p, q,
                           (const int32_t*)c->ntok_dev + (int64_t)p.layer * c->R, out_ids, out_scores);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace kvd
