// k_select.cu — launch geometry and entry points of the select kernel (rows a1 + a2, fused
// with a3 + a4); the kernel itself is in select.cuh, instantiated per CTA size in
// k_select_nt512.cu and k_select_nt1024.cu.
#include "select.cuh"

namespace kvd {

// Launch geometry for `segs` segments of nb_pad blocks: threads per CTA, cluster size, keys per
// thread and vector width.  The cluster starts at the fewest CTAs whose shared memory holds the
// segment (<= kMaxKpt keys per 1024-thread CTA) and doubles (<= 8, portable) while the launch
// has fewer than kSelectCtaTarget CTAs and a CTA keeps >= 1024 blocks: a few long segments (c4:
// 4 per chain) are spread over many SMs -- one SM streams a segment's summaries at only
// ~50-80 GB/s (tools/micro/score_stream.cu) -- while launches of many segments keep one CTA per
// segment (no cluster barriers).  CTAs of up to 2048 blocks run 512 threads (4 keys each), longer
// spans 1024.  The choice never changes a result (scores are per block; the top-k is exact).
// V (blocks per row load) = 2, 4 or 8 keys per thread: 4-, 8- or 16-byte loads.
constexpr int kMaxKpt = kMaxSelectBlocks / (8 * 1024);   // 32 at 1024 threads: 5 B of smem per key
constexpr int kSelectCtaTarget = 64;
static int tune(const char* name, int dflt) {
#ifdef KVD_EXPERIMENTS
    const char* e = getenv(name);             // experiment builds only (tools/; never the product)
    if (e) return atoi(e);
#else
    (void)name;
#endif
    return dflt;
}
void select_geometry(int64_t nb_pad, int segs, bool resident, int* nt, int* cl, int* kpt, int* v) {
    static const int target = tune("KVD_SELECT_CTAS", kSelectCtaTarget),
                     min_span_res = tune("KVD_SELECT_MINSPAN", 1024),
                     min_span_host = tune("KVD_SELECT_MINSPAN_HOST", 8192),
                     nt_small = tune("KVD_SELECT_NT_SMALL", 512), nt_large = tune("KVD_SELECT_NT_LARGE", 1024);
    // host-backed: rank 0 fetches the misses over the host link after the selection, holding its
    // SM; spans of up to 8192 blocks stay on one CTA (c3: 2799 vs 2397 tok/s with 8 CTAs/segment)
    const int min_span = resident ? min_span_res : min_span_host;
    int c = 1;
    while (c < 8 && (int64_t)c * 1024 * kMaxKpt < nb_pad) c <<= 1;
    while (c < 8 && (int64_t)segs * c < target && nb_pad / (2 * c) >= min_span) c <<= 1;
    const int64_t span = (nb_pad + c - 1) / c;
    const int threads = span <= 2048 ? nt_small : nt_large;
    int64_t per = (span + threads - 1) / threads;
    const int vw = per >= 8 ? 8 : per >= 4 ? 4 : 2;
    per = (per + vw - 1) / vw * vw;
    *nt = threads;
    *cl = c;
    *kpt = (int)per;
    *v = vw;
}

// Geometry of rank_kernel (behind score_kernel): it only ranks scores from L2.  Its phases are
// instruction-bound on one SM (a few dozen instructions per key and pass), so a segment is cut
// into CTAs of at most 8192 keys (c4's 65,536 blocks: a cluster of 8; 1632 vs 1475 tok/s with
// 2 CTAs of 32,768) -- up to the portable cluster size of 8 -- and the rank-0 merge takes the
// rest.  512 threads up to 2048 blocks per CTA, else 1024.  (KVD_SELECT_PRE_SPAN: experiments.)
void select_geometry_pre(int64_t nb_pad, int* nt, int* cl, int* kpt, int* v) {
    static const int max_span = tune("KVD_SELECT_PRE_SPAN", 8192),
                     nt_small = tune("KVD_SELECT_NT_SMALL", 512), nt_large = tune("KVD_SELECT_NT_LARGE", 1024);
    int c = 1;
    while (c < 8 && (nb_pad + c - 1) / c > max_span) c <<= 1;
    const int64_t span = (nb_pad + c - 1) / c;
    const int threads = span <= 2048 ? nt_small : nt_large;
    int64_t per = (span + threads - 1) / threads;
    per = (per + 1) / 2 * 2;
    *nt = threads;
    *cl = c;
    *kpt = (int)(per < 2 ? 2 : per);
    *v = 2;
}

// The default selection (select_fast) gathers up to min(K, span) candidates per CTA on rank 0 of
// a cluster: at most kCandMax rank keys (64 KiB).  Larger K x cluster products take the general
// path.
constexpr int64_t kCandMax = 8192;
size_t select_static_smem();
bool select_fast_ok(int cl, int64_t span, int64_t kb) {
    if (cl > 1 && cl * std::min(kb, span) > kCandMax) return false;
    const size_t fast = (size_t)span * 4 + (size_t)kRankList * 8 + (cl > 1 ? 8 * (size_t)cl * std::min(kb, span) : 0);
    return fast + 16 + 4 * (size_t)kb + select_static_smem() <= kMaxSmemBytes;
}

// dynamic shared memory: general path [span] keys | [kListCap] compacted pairs | [span] first-digit
// bins; default path [span] keys | [kRankList] rank keys | [CL * min(K, span)] candidates (CL > 1).
// (The fused kernel adds the selection, 4 B per id, past the larger of this and the resolve's set.)
size_t select_smem_bytes(int nt, int kpt, int cl, int64_t kb) {
    const int64_t span = (int64_t)nt * kpt;
    const size_t general = (size_t)span * 5 + (size_t)kListCap * 8;
    const size_t fast = select_fast_ok(cl, span, kb)
                            ? (size_t)span * 4 + (size_t)kRankList * 8 + (cl > 1 ? 8 * (size_t)cl * std::min(kb, span) : 0)
                            : 0;
    return std::max(general, fast);
}

size_t select_static_smem() {
    return sizeof(TopkShared) + sizeof(KthShared) + sizeof(ResolveShared) + sizeof(float) * kHeadDim;
}

// score_kernel over the launch's segments, then rank_kernel ranking those scores from L2 (PDL).
// A cluster whose candidates do not fit rank 0 (K x cluster size > kCandMax) takes the
// self-scoring select_kernel with the general top-k instead.
template <bool RESOLVE>
static cudaError_t launch_select_any(kvd_cache* c, const StepParams& p, const uint16_t* q, int32_t* out_ids,
                                     float* out_scores, const FuseArgs& fa, cudaStream_t s) {
    int nt, cl, kpt, v;
    select_geometry_pre(c->nb_pad, &nt, &cl, &kpt, &v);
    if (!select_fast_ok(cl, (int64_t)nt * kpt, p.k)) {
        select_geometry(c->nb_pad, p.B * p.nh, c->resident, &nt, &cl, &kpt, &v);
        return nt == 512 ? launch_select_nt<512, RESOLVE>(c, p, q, c->summ, c->scores, cl, kpt, v, out_ids, out_scores, fa, s)
                         : launch_select_nt<1024, RESOLVE>(c, p, q, c->summ, c->scores, cl, kpt, v, out_ids, out_scores, fa, s);
    }
    cudaError_t e = launch_score(c, p, q, c->summ, c->summ2, c->scores, s);
    if (e != cudaSuccess) return e;
    return nt == 512 ? launch_rank_nt<512, RESOLVE>(c, p, c->scores, cl, kpt, out_ids, out_scores, fa, s)
                     : launch_rank_nt<1024, RESOLVE>(c, p, c->scores, cl, kpt, out_ids, out_scores, fa, s);
}

// Stage 1 of the hierarchical index (R27): the same kernel over the segment's centroid matrix
// (p.nb_pad = nc_pad, p.sel_mode = 1), selected centroid ids -> c->csel.  No fetch inside, so the
// resident geometry (spread over SMs) applies.
cudaError_t launch_select_centroids(kvd_cache* c, const StepParams& p, const uint16_t* q, cudaStream_t s) {
    int nt, cl, kpt, v;
    select_geometry_pre(c->nc_pad, &nt, &cl, &kpt, &v);
    const FuseArgs fa{};
    cudaError_t e;
    if (!select_fast_ok(cl, (int64_t)nt * kpt, c->m_max)) {
        select_geometry(c->nc_pad, p.B * p.nh, true, &nt, &cl, &kpt, &v);
        e = nt == 512 ? launch_select_nt<512, false>(c, p, q, c->cent, c->cscores, cl, kpt, v, c->csel, nullptr, fa, s)
                      : launch_select_nt<1024, false>(c, p, q, c->cent, c->cscores, cl, kpt, v, c->csel, nullptr, fa, s);
    } else {
        e = launch_score(c, p, q, c->cent, nullptr, c->cscores, s);
        if (e == cudaSuccess)
            e = nt == 512 ? launch_rank_nt<512, false>(c, p, c->cscores, cl, kpt, c->csel, nullptr, fa, s)
                          : launch_rank_nt<1024, false>(c, p, c->cscores, cl, kpt, c->csel, nullptr, fa, s);
    }
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_select(kvd_cache* c, const StepParams& p, const uint16_t* q, int32_t* out_ids, float* out_scores,
                          cudaStream_t s) {
    if (c->index_ratio > 0) return launch_index_select(c, p, q, out_ids, out_scores, nullptr, s);
    const FuseArgs fa{};
    cudaError_t e = launch_select_any<false>(c, p, q, out_ids, out_scores, fa, s);
    return e != cudaSuccess ? e : cudaGetLastError();
}

// kvd_select_resolve_fetch: one kernel scores, selects, resolves and copies the misses.
cudaError_t launch_select_resolve(kvd_cache* c, const StepParams& p, const uint16_t* q, int32_t* out_ids,
                                  float* out_scores, int32_t* out_attn, cudaStream_t s) {
    if (c->index_ratio > 0) return launch_index_select(c, p, q, out_ids, out_scores, out_attn, s);
    FuseArgs fa;
    fa.rb = resolve_bufs(c, p.layer);
    fa.out_attn = out_attn;
    fa.host_store = c->resident ? nullptr : c->host_store;
    fa.slots = c->slots;
    cudaError_t e = launch_select_any<true>(c, p, q, out_ids, out_scores, fa, s);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace kvd
