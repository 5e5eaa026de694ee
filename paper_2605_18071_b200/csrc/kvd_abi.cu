// kvd_abi.cu — the C ABI of libkvd.so (include/kvd.h): configuration and
// allocation, synchronous argument validation, step-call dispatch to the
// kernels, introspection.  No exception crosses this boundary.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

using namespace kvd;

namespace {

thread_local std::string g_err;
#ifdef KVD_EXPERIMENTS
unsigned long long* g_exp_trace = nullptr;   // [kExpUnits][kExpPhases] phase stamps (tuning builds)
#endif

kvd_status fail(kvd_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define KVD_CUDA(call)                                                                            \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(e_ == cudaErrorMemoryAllocation ? KVD_ENOMEM : KVD_ECUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                       \
    } while (0)

struct Geometry {
    int L, Hq, Hkv, G, P, R, kmax, pmax, A, E, max_splits;
    int64_t nmax, nb_max, nb_pad, C, rec_bytes;
    bool resident;
    int ratio, m_max;                 // hierarchical index (0 = flat)
    int64_t nc_pad;
};

kvd_status check_config(const kvd_config* cfg, Geometry* g) {
    if (!cfg) return fail(KVD_EINVAL, "config is NULL");
    if (cfg->head_dim != KVD_HEAD_DIM) return fail(KVD_EINVAL, "head_dim must be %d", KVD_HEAD_DIM);
    if (cfg->num_layers < 1 || cfg->num_kv_heads < 1 || cfg->num_q_heads < 1 || cfg->max_requests < 1)
        return fail(KVD_EINVAL, "layers, heads and max_requests must be >= 1");
    if (cfg->num_q_heads % cfg->num_kv_heads) return fail(KVD_EINVAL, "num_q_heads %% num_kv_heads != 0");
    if (cfg->num_q_heads / cfg->num_kv_heads > KVD_MAX_GROUP)
        return fail(KVD_EINVAL, "group size > %d unsupported", KVD_MAX_GROUP);
    const int P = cfg->block_tokens;
    if (P != 1 && P != 2 && P != 4 && P != 8 && P != 16) return fail(KVD_EINVAL, "block_tokens must be 1,2,4,8,16");
    if (cfg->max_context < 1) return fail(KVD_EINVAL, "max_context must be >= 1");
    if (cfg->slots_per_segment < 1) return fail(KVD_EINVAL, "slots_per_segment must be >= 1");
    if (cfg->max_select < 0) return fail(KVD_EINVAL, "max_select must be >= 0");
    if (cfg->sink_tokens < 0 || cfg->local_tokens < 0) return fail(KVD_EINVAL, "sink/local tokens must be >= 0");
    if (cfg->policy < 0 || cfg->policy > 2) return fail(KVD_EINVAL, "unknown policy %d", cfg->policy);
    g->L = cfg->num_layers;
    g->Hq = cfg->num_q_heads;
    g->Hkv = cfg->num_kv_heads;
    g->G = g->Hq / g->Hkv;
    g->P = P;
    g->E = 16 / P;
    g->R = cfg->max_requests;
    g->nmax = cfg->max_context;
    g->nb_max = (g->nmax + P - 1) / P;
    if (g->nb_max >= (1ll << 23)) return fail(KVD_EINVAL, "too many blocks per request");
    g->nb_pad = (g->nb_max + kScoreCols - 1) / kScoreCols * kScoreCols;
    g->C = cfg->slots_per_segment;
    g->resident = g->C >= g->nb_max;
    g->kmax = cfg->max_select;
    if (g->kmax > g->nb_max) return fail(KVD_EINVAL, "max_select > blocks per request");
    if (g->nb_pad > kMaxSelectBlocks) return fail(KVD_EINVAL, "context too long: > %d blocks", kMaxSelectBlocks);
    {
        // on-chip working sets (dynamic + static shared memory of the step kernels, kvd.h)
        int nt, cl, kpt, v;
        select_geometry(g->nb_pad, 1 << 30, g->resident, &nt, &cl, &kpt, &v);   // fewest CTAs: most keys each
        const size_t sel = select_smem_bytes(nt, kpt, cl, g->kmax);
        const size_t res = resolve_smem_bytes(g->resident ? 0 : g->C, g->kmax, g->nb_pad);
        // the fused kernel keeps the selection (4 B per id) past the larger of the two
        if ((std::max(sel, res) + 15) / 16 * 16 + 4 * (size_t)g->kmax + select_static_smem() > kMaxSmemBytes ||
            res + resolve_static_smem() > kMaxSmemBytes)
            return fail(KVD_EINVAL, "slots_per_segment=%lld too large for on-chip victim selection (host-backed cache)",
                        (long long)g->C);
    }
    g->pmax = (cfg->sink_tokens + P - 1) / P + (cfg->local_tokens > 0 ? (cfg->local_tokens + P - 1) / P + 1 : 0);
    g->A = (cfg->host_layer_alias <= 0 || cfg->host_layer_alias > g->L) ? g->L : cfg->host_layer_alias;
    g->rec_bytes = 2ll * P * kRowBytes;
    if (g->pmax > 256) return fail(KVD_EINVAL, "sink/local tokens pin %d blocks (> 256)", g->pmax);
    // a host-backed cache keeps every pinned block of a request in its own slot (R14): slots
    // 0 .. pinned-1 must exist for the longest request (kvd_load_prefix places them there)
    if (!g->resident && g->C < g->pmax)
        return fail(KVD_EINVAL, "slots_per_segment=%lld < %d pinned blocks (sink/local tokens)", (long long)g->C,
                    g->pmax);
    g->max_splits = kMaxPieces;
    g->ratio = cfg->index_ratio;
    if (cfg->summary_kind < 0 || cfg->summary_kind > 1) return fail(KVD_EINVAL, "summary_kind must be 0 (mean) or 1 (min/max)");
    if (cfg->summary_kind == 1 && cfg->index_ratio > 0)
        return fail(KVD_EINVAL, "the hierarchical index clusters mean-key summaries (summary_kind 0)");
    g->nc_pad = 0;
    g->m_max = 0;
    if (g->ratio < 0 || g->ratio > kIdxWindow) return fail(KVD_EINVAL, "index_ratio must be 0 (flat) or 1..%d", kIdxWindow);
    if (g->ratio > 0) {
        const int64_t nwin = (g->nb_max + kIdxWindow - 1) / kIdxWindow;
        const int64_t nc_max = nwin * ((kIdxWindow + g->ratio - 1) / g->ratio);
        g->nc_pad = (nc_max + kScoreCols - 1) / kScoreCols * kScoreCols;
        const int64_t f = (kIdxFanout * (int64_t)g->kmax + g->ratio - 1) / g->ratio;
        g->m_max = (int)std::min<int64_t>(nc_max, std::max<int64_t>(f, g->kmax + g->pmax));
        if (std::min<int64_t>(g->nb_max, (int64_t)kIdxWindow * g->m_max) > kCandCap)
            return fail(KVD_EINVAL, "hierarchical index: max_select=%d with index_ratio=%d may give %lld candidates "
                        "(> %d)", g->kmax, g->ratio, (long long)std::min<int64_t>(g->nb_max, (int64_t)kIdxWindow * g->m_max),
                        kCandCap);
        if (g->m_max > 1024) return fail(KVD_EINVAL, "hierarchical index: %d stage-1 centroids > 1024", g->m_max);
        if (cand_smem_bytes(g->nb_pad) + 4096 > kMaxSmemBytes)
            return fail(KVD_EINVAL, "hierarchical index: context too long for the candidate kernel");
    }
    if ((int64_t)g->Hkv * g->nb_max * 4 > kSlotOfBytes) return fail(KVD_EINVAL, "context too long for setup scratch");
    return KVD_OK;
}

struct Sizes {
    size_t slots, summ, scores, table, meta4, meta1, miss, small, host, index, summ2;
    size_t dev_total() const { return slots + summ + scores + table + 3 * meta4 + meta1 + miss + small + index + summ2; }
};

Sizes sizes_of(const Geometry& g, int summary_kind = 0) {
    Sizes s;
    const size_t segs = (size_t)g.L * g.R * g.Hkv;
    const size_t rsegs = (size_t)g.R * g.Hkv;
    s.slots = segs * g.C * g.rec_bytes;
    s.summ = segs * kHeadDim * g.nb_pad * 2;
    s.scores = segs * g.nb_pad * 4;
    s.table = segs * g.nb_pad * 4;
    s.meta4 = segs * g.C * 4;
    s.meta1 = segs * g.C;
    s.miss = rsegs * (size_t)(g.kmax > 0 ? g.kmax : 1) * 2 * 4 + rsegs * 4;
    s.small = rsegs * 12 + 64 + 4 + (size_t)g.R * 4 + g.rec_bytes;
    s.host = g.resident ? 0 : (size_t)g.A * g.R * g.Hkv * g.nb_max * g.rec_bytes;
    s.index = 0;
    s.summ2 = summary_kind == 1 ? s.summ : 0;
    if (g.ratio > 0)   // centroids + centroid scores + counts + cent_of + members + offsets + stage-1 ids
        s.index = segs * (kHeadDim * g.nc_pad * 2 + g.nc_pad * 4 + 4 + 2 * g.nb_pad * 4 + (g.nc_pad + 1) * 4) +
                  rsegs * g.m_max * 4 + segs * g.nb_pad / 8;
    return s;
}

template <class T>
cudaError_t dalloc(T** p, size_t bytes) {
    void* v = nullptr;
    cudaError_t e = cudaMalloc(&v, bytes ? bytes : 16);
    *p = static_cast<T*>(v);
    return e;
}

kvd_status check_step(kvd_cache* c, int32_t layer, const int32_t* req_ids, int32_t B, int32_t k, StepParams* p) {
    if (!c) return fail(KVD_EINVAL, "cache is NULL");
    if (!req_ids) return fail(KVD_EINVAL, "req_ids is NULL");
    if (B < 1 || B > KVD_MAX_BATCH) return fail(KVD_EINVAL, "B=%d outside [1, %d]", B, KVD_MAX_BATCH);
    if (layer < 0 || layer >= c->L) return fail(KVD_EINVAL, "layer %d out of range", layer);
    if (k < 0 || k > c->kmax) return fail(KVD_EINVAL, "k_blocks=%d outside [0, max_select=%d]", k, c->kmax);
    std::vector<char> seen((size_t)c->R, 0);
    for (int b = 0; b < B; ++b) {
        const int r = req_ids[b];
        if (r < 0 || r >= c->R) return fail(KVD_EINVAL, "req_ids[%d]=%d out of range", b, r);
        if (seen[(size_t)r]) return fail(KVD_EINVAL, "req_ids[%d]=%d repeated", b, r);
        seen[(size_t)r] = 1;
        const int64_t nr = c->ntok[(size_t)layer * c->R + r];
        if (nr <= 0) return fail(KVD_ESTATE, "request %d has no prefix loaded in layer %d", r, layer);
        const SegGeom sg = seg_geom(nr, c->P, c->cfg.sink_tokens, c->cfg.local_tokens);
        const int pr = sg.sink_end + (sg.nb - sg.local_begin);
        if (k > sg.nb - pr)
            return fail(KVD_ERANGE, "request %d: k_blocks=%d > %d candidate blocks", r, k, sg.nb - pr);
        int64_t cap = c->C;                       // 2D window scaling: the layer's smallest head capacity
        for (int hh = 0; hh < c->Hkv; ++hh) cap = std::min(cap, c->cap_host[(size_t)layer * c->Hkv + hh]);
        if ((int64_t)k + pr > cap)
            return fail(KVD_ECAPACITY, "request %d: k_blocks + pinned = %d > slots %lld of layer %d", r, k + pr,
                        (long long)cap, layer);
        p->req[b] = r;
    }
    p->B = B;
    p->layer = layer;
    p->k = k;
    p->W = k + c->pmax;
    p->R = c->R;
    p->Hkv = c->Hkv;
    p->Hq = c->Hq;
    p->G = c->G;
    p->P = c->P;
    p->E = c->E;
    p->nb_pad = c->nb_pad;
    p->C = c->C;
    p->nb_max = c->nb_max;
    p->sink_tokens = c->cfg.sink_tokens;
    p->local_tokens = c->cfg.local_tokens;
    p->policy = c->cfg.policy;
    p->step = 0;
    p->step_dev = c->step_dev;
    p->host_layer = layer % c->A;
    p->rec_bytes = (int32_t)c->rec_bytes;
    p->scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)KVD_HEAD_DIM));
    p->kt_slots = c->kt_on ? c->kt_slots : nullptr;
    p->kt_acc = c->kt_acc;
    p->h0 = 0;
    p->nh = c->Hkv;
    p->early_trigger = 1;
#ifdef KVD_EXPERIMENTS
    if (const char* e = getenv("KVD_EARLY_TRIGGER")) p->early_trigger = atoi(e);
#endif
    p->kt_base = ((layer * c->R + p->req[0]) * c->Hkv) * kKtKinds;
    p->exp_trace = nullptr;
    p->sel_mode = c->summary_kind == 1 ? 2 : 0;   // Quest min/max scoring (R30) or mean summaries
    p->sel_ratio = 0;
    p->sel_stride = 0;
    p->sel_count = nullptr;
    p->summ2 = c->summ2;
#ifdef KVD_EXPERIMENTS
    if (getenv("KVD_EXP_TRACE")) {
        if (!g_exp_trace) {
            cudaMalloc(&g_exp_trace, (size_t)kExpUnits * kExpPhases * 8);
            cudaMemset(g_exp_trace, 0, (size_t)kExpUnits * kExpPhases * 8);
        }
        p->exp_trace = g_exp_trace;
    }
#endif
    return KVD_OK;
}

std::atomic<uint64_t> g_launches{0};

kvd_status launched(cudaError_t e) {
    if (e != cudaSuccess) return fail(KVD_ECUDA, "kernel launch: %s", cudaGetErrorString(e));
    return KVD_OK;
}

}  // namespace

void kvd::count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" {

const char* kvd_last_error(void) { return g_err.c_str(); }

#ifdef KVD_EXPERIMENTS
const char* kvd_version(void) { return "kvd 0.3 sm_100a (experiments build)"; }
#else
const char* kvd_version(void) { return "kvd 0.3 sm_100a"; }
#endif

uint64_t kvd_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

kvd_status kvd_required_bytes(const kvd_config* cfg, size_t* dev_bytes, size_t* host_pinned_bytes) {
    Geometry g;
    kvd_status st = check_config(cfg, &g);
    if (st) return st;
    Sizes s = sizes_of(g, cfg->summary_kind);
    if (dev_bytes) *dev_bytes = s.dev_total();
    if (host_pinned_bytes) *host_pinned_bytes = s.host;
    return KVD_OK;
}

kvd_status kvd_create_cache(const kvd_config* cfg, kvd_cache** out) {
    if (!out) return fail(KVD_EINVAL, "out is NULL");
    *out = nullptr;
    Geometry g;
    kvd_status st = check_config(cfg, &g);
    if (st) return st;
    KVD_CUDA(cudaSetDevice(cfg->device));
    kvd_cache* c = new (std::nothrow) kvd_cache();
    if (!c) return fail(KVD_ENOMEM, "host allocation failed");
    c->cfg = *cfg;
    c->L = g.L; c->Hq = g.Hq; c->Hkv = g.Hkv; c->G = g.G; c->P = g.P; c->R = g.R; c->kmax = g.kmax;
    c->pmax = g.pmax; c->A = g.A; c->E = g.E; c->nmax = g.nmax; c->nb_max = g.nb_max; c->nb_pad = g.nb_pad;
    c->C = g.C; c->resident = g.resident; c->rec_bytes = g.rec_bytes; c->max_splits = g.max_splits;
    c->index_ratio = g.ratio; c->nc_pad = g.nc_pad; c->m_max = g.m_max;
    c->cap_host.assign((size_t)g.L * g.Hkv, g.C);
    c->summary_kind = cfg->summary_kind;
    c->ntok.assign((size_t)g.L * g.R, 0);
    {
        int lo = 0, hi = 0;
        if (cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess) c->prio_hi = hi;
    }
    const Sizes s = sizes_of(g);
    const size_t rsegs = (size_t)g.R * g.Hkv;
    cudaError_t e = cudaSuccess;
#define ALLOC(ptr, bytes)                                       \
    if (e == cudaSuccess) e = dalloc(&c->ptr, (bytes));
    ALLOC(slots, s.slots);
    ALLOC(summ, s.summ);
    ALLOC(scores, s.scores);
    ALLOC(table, s.table);
    ALLOC(slot_block, s.meta4);
    ALLOC(last_use, s.meta4);
    ALLOC(use_count, s.meta4);
    ALLOC(phase, s.meta1);
    ALLOC(miss, rsegs * (size_t)(g.kmax > 0 ? g.kmax : 1) * 2 * 4);
    ALLOC(miss_count, rsegs * 4);
    ALLOC(stats, 64);
    ALLOC(err, 4);
    ALLOC(ntok_dev, (size_t)g.L * g.R * 4);
    ALLOC(zero_rec, (size_t)g.rec_bytes);
    ALLOC(cap_dev, (size_t)g.L * g.Hkv * 4);
    if (cfg->summary_kind == 1) ALLOC(summ2, s.summ);
    ALLOC(seg_stats, (size_t)g.L * g.Hkv * 16);
    if (g.ratio > 0) {
        const size_t segs = (size_t)g.L * g.R * g.Hkv;
        ALLOC(cent, segs * kHeadDim * g.nc_pad * 2);
        ALLOC(cscores, segs * g.nc_pad * 4);
        ALLOC(ncent, segs * 4);
        ALLOC(cent_of, segs * g.nb_pad * 4);
        ALLOC(memb, segs * g.nb_pad * 4);
        ALLOC(moff, segs * (g.nc_pad + 1) * 4);
        ALLOC(csel, rsegs * (size_t)g.m_max * 4);
        ALLOC(cand_bits, segs * g.nb_pad / 8);
    }
#undef ALLOC
    if (e == cudaSuccess) e = cudaMemset(c->scores, 0, s.scores);
    if (e == cudaSuccess) e = cudaMemset(c->table, 0xFF, s.table);
    if (e == cudaSuccess) e = cudaMemset(c->slot_block, 0xFF, s.meta4);
    if (e == cudaSuccess) e = cudaMemset(c->miss_count, 0, rsegs * 4);
    if (e == cudaSuccess) e = cudaMemset(c->stats, 0, 64);
    if (e == cudaSuccess && c->cand_bits) e = cudaMemset(c->cand_bits, 0, (size_t)g.L * g.R * g.Hkv * g.nb_pad / 8);
    if (e == cudaSuccess) e = cudaMemset(c->seg_stats, 0, (size_t)g.L * g.Hkv * 16);
    if (e == cudaSuccess) {
        std::vector<int32_t> caps((size_t)g.L * g.Hkv, (int32_t)std::min<int64_t>(g.C, INT32_MAX));
        e = cudaMemcpy(c->cap_dev, caps.data(), caps.size() * 4, cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = cudaMemset(c->err, 0, 4);
    if (e == cudaSuccess) e = cudaMemset(c->ntok_dev, 0, (size_t)g.L * g.R * 4);
    if (e == cudaSuccess) e = cudaMemset(c->zero_rec, 0, (size_t)g.rec_bytes);
    if (e == cudaSuccess && !g.resident) {
        void* h = nullptr;
        e = cudaHostAlloc(&h, s.host, cudaHostAllocMapped | cudaHostAllocPortable);
        c->host_store = static_cast<uint8_t*>(h);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        kvd_destroy_cache(c);
        return fail(e == cudaErrorMemoryAllocation ? KVD_ENOMEM : KVD_ECUDA, "create: %s", cudaGetErrorString(e));
    }
    *out = c;
    return KVD_OK;
}

void kvd_destroy_cache(kvd_cache* c) {
    if (!c) return;
    cudaSetDevice(c->cfg.device);
    cudaDeviceSynchronize();
    void* dev[] = {c->slots, c->summ, c->scores, c->table, c->slot_block, c->last_use, c->phase,
                   c->use_count, c->miss, c->miss_count, c->kt_slots, c->kt_acc, c->summ2, c->cap_dev, c->seg_stats, c->cent, c->cscores, c->ncent, c->cent_of, c->memb, c->moff, c->csel, c->cand_bits, c->idx_stage, c->stats,
                   c->err, c->ntok_dev, c->zero_rec, c->stage_kv, c->stage_rec, c->stage_q, c->warm_imp};
    for (void* p : dev)
        if (p) cudaFree(p);
    if (c->host_store) cudaFreeHost(c->host_store);
    delete c;
}

kvd_status kvd_set_device_step(kvd_cache* c, const uint32_t* dev_step) {
    if (!c) return fail(KVD_EINVAL, "cache is NULL");
    c->step_dev = dev_step;
    return KVD_OK;
}

kvd_status kvd_get_info(const kvd_cache* c, kvd_cache_info* out) {
    if (!c || !out) return fail(KVD_EINVAL, "NULL argument");
    out->nb_max = c->nb_max;
    out->nb_pad = c->nb_pad;
    out->slots_per_segment = c->C;
    out->max_pinned = c->pmax;
    out->record_bytes = (int32_t)c->rec_bytes;
    out->resident = c->resident ? 1 : 0;
    out->host_layers = c->A;
    return KVD_OK;
}

int32_t kvd_attn_width(const kvd_cache* c, int32_t k_blocks) { return c ? k_blocks + c->pmax : -1; }

static kvd_status load_prefix_impl(kvd_cache* c, int32_t layer, int32_t req, const uint16_t* k, const uint16_t* v,
                                   int64_t n_tokens, const uint16_t* q_obs, int32_t n_obs, kvd_stream stream) {
    if (!c || !k || !v) return fail(KVD_EINVAL, "NULL argument");
    if (layer < 0 || layer >= c->L) return fail(KVD_EINVAL, "layer %d out of range", layer);
    if (req < 0 || req >= c->R) return fail(KVD_EINVAL, "req %d out of range", req);
    if (n_tokens < 1 || n_tokens > c->nmax)
        return fail(KVD_EINVAL, "n_tokens=%lld outside [1, %lld]", (long long)n_tokens, (long long)c->nmax);
    KVD_CUDA(cudaSetDevice(c->cfg.device));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t kv_elems = (size_t)c->Hkv * n_tokens * kHeadDim;
    if (!c->stage_kv) KVD_CUDA(dalloc(&c->stage_kv, 2 * (size_t)c->Hkv * c->nmax * kHeadDim * 2));
    if (!c->stage_rec)
        KVD_CUDA(dalloc(&c->stage_rec, (size_t)kSlotOfBytes +
                                           (c->resident ? 0 : (size_t)c->Hkv * c->nb_max * c->rec_bytes)));
    const uint16_t* dk = k;
    const uint16_t* dv = v;
    cudaPointerAttributes ak{}, av{};
    KVD_CUDA(cudaPointerGetAttributes(&ak, k));
    KVD_CUDA(cudaPointerGetAttributes(&av, v));
    if (ak.type != cudaMemoryTypeDevice && ak.type != cudaMemoryTypeManaged) {
        KVD_CUDA(cudaMemcpyAsync(c->stage_kv, k, kv_elems * 2, cudaMemcpyHostToDevice, s));
        dk = c->stage_kv;
    }
    if (av.type != cudaMemoryTypeDevice && av.type != cudaMemoryTypeManaged) {
        KVD_CUDA(cudaMemcpyAsync(c->stage_kv + kv_elems, v, kv_elems * 2, cudaMemcpyHostToDevice, s));
        dv = c->stage_kv + kv_elems;
    }
    const uint16_t* dq = nullptr;
    if (q_obs && n_obs > 0 && !c->resident) {
        if (n_obs > 16 || c->G * n_obs > 128) return fail(KVD_EINVAL, "n_obs=%d: at most 16 (and G x n_obs <= 128)", n_obs);
        const size_t qbytes = (size_t)c->Hq * n_obs * kHeadDim * 2;
        if (!c->stage_q) KVD_CUDA(dalloc(&c->stage_q, (size_t)c->Hq * 16 * kHeadDim * 2));
        cudaPointerAttributes aq{};
        KVD_CUDA(cudaPointerGetAttributes(&aq, q_obs));
        if (aq.type != cudaMemoryTypeDevice && aq.type != cudaMemoryTypeManaged) {
            KVD_CUDA(cudaMemcpyAsync(c->stage_q, q_obs, qbytes, cudaMemcpyHostToDevice, s));
            dq = c->stage_q;
        } else {
            dq = q_obs;
        }
    }
    KVD_CUDA(launch_prefix(c, layer, req, dk, dv, n_tokens, s, dq, dq ? n_obs : 0));
    if (c->index_ratio > 0) {                     // hierarchical index over the new summaries (R27)
        if (!c->idx_stage) KVD_CUDA(dalloc(&c->idx_stage, index_stage_bytes(c->Hkv, c->nb_pad)));
        KVD_CUDA(launch_index_build(c, layer, req, n_tokens, s));
    }
    KVD_CUDA(cudaStreamSynchronize(s));
    c->ntok[(size_t)layer * c->R + req] = n_tokens;
    return KVD_OK;
}

kvd_status kvd_load_prefix(kvd_cache* c, int32_t layer, int32_t req, const uint16_t* k, const uint16_t* v,
                           int64_t n_tokens, kvd_stream stream) {
    return load_prefix_impl(c, layer, req, k, v, n_tokens, nullptr, 0, stream);
}

kvd_status kvd_load_prefix_obs(kvd_cache* c, int32_t layer, int32_t req, const uint16_t* k, const uint16_t* v,
                               int64_t n_tokens, const uint16_t* q_obs, int32_t n_obs, kvd_stream stream) {
    if (!q_obs || n_obs < 1) return fail(KVD_EINVAL, "q_obs / n_obs");
    return load_prefix_impl(c, layer, req, k, v, n_tokens, q_obs, n_obs, stream);
}

kvd_status kvd_select_topk(kvd_cache* c, int32_t layer, const uint16_t* q, const int32_t* req_ids, int32_t B,
                           int32_t k_blocks, int32_t* out_ids, float* out_scores, kvd_stream stream) {
    StepParams p;
    kvd_status st = check_step(c, layer, req_ids, B, k_blocks, &p);
    if (st) return st;
    if (!q || (!out_ids && k_blocks > 0)) return fail(KVD_EINVAL, "q / out_ids is NULL");
    return launched(launch_select(c, p, q, out_ids, out_scores, reinterpret_cast<cudaStream_t>(stream)));
}

kvd_status kvd_resolve_and_fetch(kvd_cache* c, int32_t layer, const int32_t* req_ids, int32_t B, const int32_t* ids,
                                 int32_t k_blocks, uint32_t step, int32_t* out_attn, kvd_stream stream) {
    StepParams p;
    kvd_status st = check_step(c, layer, req_ids, B, k_blocks, &p);
    if (st) return st;
    if ((!ids && k_blocks > 0) || !out_attn) return fail(KVD_EINVAL, "ids / out_attn is NULL");
    p.step = step;
    return launched(launch_resolve(c, p, ids, out_attn, reinterpret_cast<cudaStream_t>(stream)));
}

kvd_status kvd_select_resolve_fetch(kvd_cache* c, int32_t layer, const uint16_t* q, const int32_t* req_ids,
                                    int32_t B, int32_t k_blocks, uint32_t step, int32_t* out_ids, float* out_scores,
                                    int32_t* out_attn, kvd_stream stream) {
    StepParams p;
    kvd_status st = check_step(c, layer, req_ids, B, k_blocks, &p);
    if (st) return st;
    if (!q || (!out_ids && k_blocks > 0) || !out_attn) return fail(KVD_EINVAL, "q / out_ids / out_attn is NULL");
    p.step = step;
    return launched(launch_select_resolve(c, p, q, out_ids, out_scores, out_attn, reinterpret_cast<cudaStream_t>(stream)));
}

// KV-head range of a step call (the arrays keep their [B][Hkv] layouts; only heads [h0, h0+nh) run)
static kvd_status set_heads(kvd_cache* c, StepParams* p, int32_t h0, int32_t nh) {
    if (h0 < 0 || nh < 1 || h0 + nh > c->Hkv) return fail(KVD_EINVAL, "KV heads [%d, %d) outside [0, %d)", h0, h0 + nh, c->Hkv);
    p->h0 = h0;
    p->nh = nh;
    p->kt_base = ((p->layer * c->R + p->req[0]) * c->Hkv + h0) * kKtKinds;   // one timer slot per launch
    return KVD_OK;
}

kvd_status kvd_select_resolve_fetch_heads(kvd_cache* c, int32_t layer, const uint16_t* q, const int32_t* req_ids,
                                          int32_t B, int32_t h0, int32_t nh, int32_t k_blocks, uint32_t step,
                                          int32_t* out_ids, float* out_scores, int32_t* out_attn, kvd_stream stream) {
    StepParams p;
    kvd_status st = check_step(c, layer, req_ids, B, k_blocks, &p);
    if (st) return st;
    if ((st = set_heads(c, &p, h0, nh))) return st;
    if (!q || (!out_ids && k_blocks > 0) || !out_attn) return fail(KVD_EINVAL, "q / out_ids / out_attn is NULL");
    p.step = step;
    return launched(launch_select_resolve(c, p, q, out_ids, out_scores, out_attn, reinterpret_cast<cudaStream_t>(stream)));
}

kvd_status kvd_sparse_decode_heads(kvd_cache* c, int32_t layer, const uint16_t* q, const int32_t* req_ids, int32_t B,
                                   int32_t h0, int32_t nh, const int32_t* attn, int32_t W, float* out, float* out_lse,
                                   kvd_stream stream) {
    if (!c) return fail(KVD_EINVAL, "cache is NULL");
    const int32_t k = W - c->pmax;
    if (k < 0) return fail(KVD_EINVAL, "W=%d smaller than max pinned %d", W, c->pmax);
    StepParams p;
    kvd_status st = check_step(c, layer, req_ids, B, k, &p);
    if (st) return st;
    if ((st = set_heads(c, &p, h0, nh))) return st;
    if (!q || !attn || !out) return fail(KVD_EINVAL, "q / attn / out is NULL");
    return launched(launch_attention(c, p, q, attn, out, out_lse, reinterpret_cast<cudaStream_t>(stream)));
}

kvd_status kvd_append_token(kvd_cache* c, int32_t layer, const int32_t* req_ids, int32_t B, const uint16_t* k,
                            const uint16_t* v, uint32_t step, kvd_stream stream) {
    StepParams p;
    kvd_status st = check_step(c, layer, req_ids, B, 0, &p);
    if (st) return st;
    if (!k || !v) return fail(KVD_EINVAL, "k / v is NULL");
    if (c->index_ratio > 0) return fail(KVD_ESTATE, "append with the hierarchical index needs an index rebuild");
    if (!c->resident && c->A != c->L) return fail(KVD_ESTATE, "append needs one host layer per layer (host_layer_alias 0)");
    int32_t n[KVD_MAX_BATCH];
    for (int b = 0; b < B; ++b) {
        const int64_t nr = c->ntok[(size_t)layer * c->R + req_ids[b]];
        if (nr + 1 > c->nmax) return fail(KVD_ERANGE, "request %d: context full (%lld tokens)", req_ids[b], (long long)nr);
        n[b] = (int32_t)nr;
    }
    p.step = step;
    const cudaError_t e = launch_append(c, p, k, v, n, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(KVD_ECUDA, "append: %s", cudaGetErrorString(e));
    for (int b = 0; b < B; ++b) c->ntok[(size_t)layer * c->R + req_ids[b]] += 1;
    return KVD_OK;
}

kvd_status kvd_sparse_decode(kvd_cache* c, int32_t layer, const uint16_t* q, const int32_t* req_ids, int32_t B,
                             const int32_t* attn, int32_t W, float* out, float* out_lse, kvd_stream stream) {
    if (!c) return fail(KVD_EINVAL, "cache is NULL");
    const int32_t k = W - c->pmax;
    if (k < 0) return fail(KVD_EINVAL, "W=%d smaller than max pinned %d", W, c->pmax);
    StepParams p;
    kvd_status st = check_step(c, layer, req_ids, B, k, &p);
    if (st) return st;
    if (!q || !attn || !out) return fail(KVD_EINVAL, "q / attn / out is NULL");
    return launched(launch_attention(c, p, q, attn, out, out_lse, reinterpret_cast<cudaStream_t>(stream)));
}

static kvd_status check_seg(kvd_cache* c, int32_t layer, int32_t req, int32_t head) {
    if (!c) return fail(KVD_EINVAL, "cache is NULL");
    if (layer < 0 || layer >= c->L || req < 0 || req >= c->R || head < 0 || head >= c->Hkv)
        return fail(KVD_EINVAL, "segment (%d,%d,%d) out of range", layer, req, head);
    return KVD_OK;
}

kvd_status kvd_read_segment(kvd_cache* c, int32_t layer, int32_t req, int32_t head, int32_t* table,
                            int32_t* slot_block, uint32_t* last_use, uint8_t* phase, uint32_t* use_count) {
    kvd_status st = check_seg(c, layer, req, head);
    if (st) return st;
    KVD_CUDA(cudaDeviceSynchronize());
    const int64_t seg = ((int64_t)layer * c->R + req) * c->Hkv + head;
    if (table) KVD_CUDA(cudaMemcpy(table, c->table + seg * c->nb_pad, c->nb_pad * 4, cudaMemcpyDeviceToHost));
    if (slot_block) KVD_CUDA(cudaMemcpy(slot_block, c->slot_block + seg * c->C, c->C * 4, cudaMemcpyDeviceToHost));
    if (last_use) KVD_CUDA(cudaMemcpy(last_use, c->last_use + seg * c->C, c->C * 4, cudaMemcpyDeviceToHost));
    if (phase) KVD_CUDA(cudaMemcpy(phase, c->phase + seg * c->C, c->C, cudaMemcpyDeviceToHost));
    if (use_count) KVD_CUDA(cudaMemcpy(use_count, c->use_count + seg * c->C, c->C * 4, cudaMemcpyDeviceToHost));
    return KVD_OK;
}

kvd_status kvd_read_slot(kvd_cache* c, int32_t layer, int32_t req, int32_t head, int64_t slot, void* out_record) {
    kvd_status st = check_seg(c, layer, req, head);
    if (st) return st;
    if (slot < 0 || slot >= c->C || !out_record) return fail(KVD_EINVAL, "bad slot / NULL");
    KVD_CUDA(cudaDeviceSynchronize());
    const int64_t seg = ((int64_t)layer * c->R + req) * c->Hkv + head;
    KVD_CUDA(cudaMemcpy(out_record, c->slots + (seg * c->C + slot) * c->rec_bytes, (size_t)c->rec_bytes,
                        cudaMemcpyDeviceToHost));
    return KVD_OK;
}

kvd_status kvd_read_host_record(kvd_cache* c, int32_t layer, int32_t req, int32_t head, int64_t block,
                                void* out_record) {
    kvd_status st = check_seg(c, layer, req, head);
    if (st) return st;
    if (c->resident || !c->host_store) return fail(KVD_ESTATE, "fully resident cache has no host store");
    if (block < 0 || block >= c->nb_max || !out_record) return fail(KVD_EINVAL, "bad block / NULL");
    KVD_CUDA(cudaDeviceSynchronize());
    const int64_t hl = layer % c->A;
    memcpy(out_record, c->host_store + (((hl * c->R + req) * c->Hkv + head) * c->nb_max + block) * c->rec_bytes,
           (size_t)c->rec_bytes);
    return KVD_OK;
}

kvd_status kvd_read_summaries(kvd_cache* c, int32_t layer, int32_t req, int32_t head, uint16_t* out) {
    kvd_status st = check_seg(c, layer, req, head);
    if (st) return st;
    if (!out) return fail(KVD_EINVAL, "out is NULL");
    if (c->ntok[(size_t)layer * c->R + req] <= 0) return fail(KVD_ESTATE, "request %d not loaded", req);
    KVD_CUDA(cudaDeviceSynchronize());
    const int64_t seg = ((int64_t)layer * c->R + req) * c->Hkv + head;
    const int64_t nb = (c->ntok[(size_t)layer * c->R + req] + c->P - 1) / c->P;
    std::vector<uint16_t> tmp((size_t)(kHeadDim * c->nb_pad));
    KVD_CUDA(cudaMemcpy(tmp.data(), c->summ + seg * kHeadDim * c->nb_pad, tmp.size() * 2, cudaMemcpyDeviceToHost));
    for (int64_t b = 0; b < nb; ++b)
        for (int j = 0; j < kHeadDim; ++j) out[b * kHeadDim + j] = tmp[(size_t)(j * c->nb_pad + b)];
    return KVD_OK;
}

kvd_status kvd_read_index(kvd_cache* c, int32_t layer, int32_t req, int32_t head, int64_t* nc, uint16_t* centroids,
                          int32_t* cent_of) {
    kvd_status st = check_seg(c, layer, req, head);
    if (st) return st;
    if (c->index_ratio <= 0) return fail(KVD_ESTATE, "cache has no hierarchical index");
    if (!nc) return fail(KVD_EINVAL, "nc is NULL");
    if (c->ntok[(size_t)layer * c->R + req] <= 0) return fail(KVD_ESTATE, "request %d not loaded", req);
    KVD_CUDA(cudaDeviceSynchronize());
    const int64_t seg = ((int64_t)layer * c->R + req) * c->Hkv + head;
    int32_t n = 0;
    KVD_CUDA(cudaMemcpy(&n, c->ncent + seg, 4, cudaMemcpyDeviceToHost));
    *nc = n;
    if (centroids) {
        std::vector<uint16_t> tmp((size_t)(kHeadDim * c->nc_pad));
        KVD_CUDA(cudaMemcpy(tmp.data(), c->cent + seg * kHeadDim * c->nc_pad, tmp.size() * 2, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < n; ++i)
            for (int j = 0; j < kHeadDim; ++j) centroids[i * kHeadDim + j] = tmp[(size_t)(j * c->nc_pad + i)];
    }
    if (cent_of) {
        const int64_t nb = (c->ntok[(size_t)layer * c->R + req] + c->P - 1) / c->P;
        KVD_CUDA(cudaMemcpy(cent_of, c->cent_of + seg * c->nb_pad, (size_t)nb * 4, cudaMemcpyDeviceToHost));
    }
    return KVD_OK;
}

kvd_status kvd_read_warm_importance(kvd_cache* c, int32_t head, int64_t nb, float* out) {
    if (!c || !out || head < 0 || head >= c->Hkv || nb < 1 || nb > c->nb_max) return fail(KVD_EINVAL, "bad arguments");
    if (!c->warm_imp) return fail(KVD_ESTATE, "no warm-up has run");
    KVD_CUDA(cudaDeviceSynchronize());
    KVD_CUDA(cudaMemcpy(out, c->warm_imp + (int64_t)head * nb, (size_t)nb * 4, cudaMemcpyDeviceToHost));
    return KVD_OK;
}

kvd_status kvd_read_minmax(kvd_cache* c, int32_t layer, int32_t req, int32_t head, uint16_t* mn, uint16_t* mx) {
    kvd_status st = check_seg(c, layer, req, head);
    if (st) return st;
    if (c->summary_kind != 1) return fail(KVD_ESTATE, "cache keeps mean-key summaries");
    if (!mn || !mx) return fail(KVD_EINVAL, "NULL argument");
    if (c->ntok[(size_t)layer * c->R + req] <= 0) return fail(KVD_ESTATE, "request %d not loaded", req);
    KVD_CUDA(cudaDeviceSynchronize());
    const int64_t seg = ((int64_t)layer * c->R + req) * c->Hkv + head;
    const int64_t nb = (c->ntok[(size_t)layer * c->R + req] + c->P - 1) / c->P;
    std::vector<uint16_t> tmp((size_t)(kHeadDim * c->nb_pad));
    for (int which = 0; which < 2; ++which) {
        const uint16_t* src = (which ? c->summ2 : c->summ) + seg * kHeadDim * c->nb_pad;
        KVD_CUDA(cudaMemcpy(tmp.data(), src, tmp.size() * 2, cudaMemcpyDeviceToHost));
        uint16_t* out = which ? mx : mn;
        for (int64_t b = 0; b < nb; ++b)
            for (int j = 0; j < kHeadDim; ++j) out[b * kHeadDim + j] = tmp[(size_t)(j * c->nb_pad + b)];
    }
    return KVD_OK;
}

kvd_status kvd_read_scores(kvd_cache* c, int32_t layer, int32_t req, int32_t head, float* out) {
    kvd_status st = check_seg(c, layer, req, head);
    if (st) return st;
    if (!out) return fail(KVD_EINVAL, "out is NULL");
    if (c->ntok[(size_t)layer * c->R + req] <= 0) return fail(KVD_ESTATE, "request %d not loaded", req);
    KVD_CUDA(cudaDeviceSynchronize());
    const int64_t seg = ((int64_t)layer * c->R + req) * c->Hkv + head;
    const int64_t nb = (c->ntok[(size_t)layer * c->R + req] + c->P - 1) / c->P;
    KVD_CUDA(cudaMemcpy(out, c->scores + seg * c->nb_pad, (size_t)nb * 4, cudaMemcpyDeviceToHost));
    if (c->index_ratio > 0) {                     // lookahead scores: exact if scored, else the centroid's
        std::vector<uint32_t> bits((size_t)c->nb_pad / 32);
        std::vector<int32_t> cof((size_t)nb);
        std::vector<float> cs((size_t)c->nc_pad);
        KVD_CUDA(cudaMemcpy(bits.data(), c->cand_bits + seg * (c->nb_pad / 32), bits.size() * 4, cudaMemcpyDeviceToHost));
        KVD_CUDA(cudaMemcpy(cof.data(), c->cent_of + seg * c->nb_pad, cof.size() * 4, cudaMemcpyDeviceToHost));
        KVD_CUDA(cudaMemcpy(cs.data(), c->cscores + seg * c->nc_pad, cs.size() * 4, cudaMemcpyDeviceToHost));
        for (int64_t b = 0; b < nb; ++b)
            if (!((bits[(size_t)(b >> 5)] >> (b & 31)) & 1u)) out[b] = cs[(size_t)cof[(size_t)b]];
    }
    return KVD_OK;
}

#ifdef KVD_EXPERIMENTS
// experiment builds only: copy (and clear) the phase stamps [units][8]
kvd_status kvd_exp_read_trace(uint64_t* out, int32_t units) {
    if (!out || units < 1 || units > kExpUnits) return fail(KVD_EINVAL, "bad trace arguments");
    if (!g_exp_trace) return fail(KVD_ESTATE, "no trace");
    KVD_CUDA(cudaDeviceSynchronize());
    KVD_CUDA(cudaMemcpy(out, g_exp_trace, (size_t)units * kExpPhases * 8, cudaMemcpyDeviceToHost));
    KVD_CUDA(cudaMemset(g_exp_trace, 0, (size_t)kExpUnits * kExpPhases * 8));
    return KVD_OK;
}
#endif

kvd_status kvd_probe_zero_copy(const void* host, void* dev, size_t bytes, int32_t ctas, kvd_stream stream) {
    if (!host || !dev || bytes % 16 || ctas < 1) return fail(KVD_EINVAL, "bad probe arguments");
    cudaPointerAttributes a{};
    KVD_CUDA(cudaPointerGetAttributes(&a, host));
    if (a.type != cudaMemoryTypeHost) return fail(KVD_EINVAL, "probe source is not pinned host memory");
    KVD_CUDA(launch_zero_copy(a.devicePointer ? a.devicePointer : host, dev, bytes, ctas,
                              reinterpret_cast<cudaStream_t>(stream)));
    return KVD_OK;
}

kvd_status kvd_enable_kernel_timer(kvd_cache* c, int32_t enable) {
    if (!c) return fail(KVD_EINVAL, "cache is NULL");
    KVD_CUDA(cudaSetDevice(c->cfg.device));
    KVD_CUDA(cudaDeviceSynchronize());
    const size_t nslots = (size_t)c->L * c->R * c->Hkv * kKtKinds;
    if (enable && !c->kt_slots) {
        KVD_CUDA(dalloc(&c->kt_slots, nslots * 16));
        KVD_CUDA(dalloc(&c->kt_acc, (size_t)kKtKinds * 16));
    }
    if (c->kt_slots) {
        std::vector<unsigned long long> init(nslots * 2);
        for (size_t i = 0; i < nslots; ++i) {
            init[2 * i] = ~0ull;
            init[2 * i + 1] = 0;
        }
        KVD_CUDA(cudaMemcpy(c->kt_slots, init.data(), nslots * 16, cudaMemcpyHostToDevice));
        KVD_CUDA(cudaMemset(c->kt_acc, 0, (size_t)kKtKinds * 16));
    }
    c->kt_on = enable != 0;
    return KVD_OK;
}

kvd_status kvd_read_kernel_timer(kvd_cache* c, uint64_t* ns, uint64_t* launches) {
    if (!c || !ns || !launches) return fail(KVD_EINVAL, "NULL argument");
    if (!c->kt_acc) return fail(KVD_ESTATE, "kernel timer was never enabled");
    KVD_CUDA(cudaDeviceSynchronize());
    unsigned long long v[2 * kKtKinds];
    KVD_CUDA(cudaMemcpy(v, c->kt_acc, sizeof v, cudaMemcpyDeviceToHost));
    for (int i = 0; i < kKtKinds; ++i) {
        ns[i] = v[2 * i];
        launches[i] = v[2 * i + 1];
    }
    return KVD_OK;
}

kvd_status kvd_set_segment_capacity(kvd_cache* c, int32_t layer, int32_t head, int64_t slots) {
    if (!c) return fail(KVD_EINVAL, "cache is NULL");
    if (layer < 0 || layer >= c->L || head < 0 || head >= c->Hkv) return fail(KVD_EINVAL, "bad layer / head");
    if (c->resident) return fail(KVD_ESTATE, "a fully resident cache has no window to scale");
    if (slots < c->pmax || slots > c->C)
        return fail(KVD_EINVAL, "slots=%lld outside [%d pinned, %lld allocated]", (long long)slots, c->pmax,
                    (long long)c->C);
    KVD_CUDA(cudaSetDevice(c->cfg.device));
    KVD_CUDA(cudaDeviceSynchronize());
    int64_t& cur = c->cap_host[(size_t)layer * c->Hkv + head];
    if (slots < cur) {
        KVD_CUDA(launch_shrink_capacity(c, layer, head, slots, nullptr));
        KVD_CUDA(cudaDeviceSynchronize());
    }
    cur = slots;
    const int32_t v = (int32_t)slots;
    KVD_CUDA(cudaMemcpy(c->cap_dev + (size_t)layer * c->Hkv + head, &v, 4, cudaMemcpyHostToDevice));
    return KVD_OK;
}

kvd_status kvd_get_segment_stats(kvd_cache* c, uint64_t* selected, uint64_t* misses) {
    if (!c || !selected || !misses) return fail(KVD_EINVAL, "NULL argument");
    KVD_CUDA(cudaDeviceSynchronize());
    std::vector<unsigned long long> v((size_t)c->L * c->Hkv * 2);
    KVD_CUDA(cudaMemcpy(v.data(), c->seg_stats, v.size() * 8, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < (size_t)c->L * c->Hkv; ++i) {
        selected[i] = v[2 * i];
        misses[i] = v[2 * i + 1];
    }
    return KVD_OK;
}

// Offline planner of 2D window scaling: greedy multiple-choice knapsack.
// Every pair starts at its smallest size; the single upgrade (pair, larger size) with the highest
// benefit gain per cost gain that fits the budget is applied until none fits (ties: lower pair,
// then smaller size).
kvd_status kvd_plan_window_scaling(const double* benefit, const double* cost, int32_t pairs, int32_t sizes,
                                   double budget, int32_t* choice) {
    if (!benefit || !cost || !choice || pairs < 1 || sizes < 1) return fail(KVD_EINVAL, "bad planner arguments");
    double used = 0.0;
    for (int32_t p = 0; p < pairs; ++p) {
        choice[p] = 0;
        used += cost[(size_t)p * sizes];
    }
    if (used > budget) return fail(KVD_EINVAL, "the smallest windows already exceed the budget");
    while (true) {
        int32_t bp = -1, bs = -1;
        double best = 0.0;
        for (int32_t p = 0; p < pairs; ++p) {
            const double* bpair = benefit + (size_t)p * sizes;
            const double* cpair = cost + (size_t)p * sizes;
            for (int32_t s = choice[p] + 1; s < sizes; ++s) {
                const double dc = cpair[s] - cpair[choice[p]], db = bpair[s] - bpair[choice[p]];
                if (used + dc > budget || (db <= 0.0 && dc >= 0.0)) continue;
                const double ratio = dc > 0.0 ? db / dc : (db > 0.0 ? INFINITY : 0.0);
                if (bp < 0 || ratio > best) {
                    bp = p;
                    bs = s;
                    best = ratio;
                }
            }
        }
        if (bp < 0) break;
        used += cost[(size_t)bp * sizes + bs] - cost[(size_t)bp * sizes + choice[bp]];
        choice[bp] = bs;
    }
    return KVD_OK;
}

kvd_status kvd_get_stats(kvd_cache* c, kvd_stats* out) {
    if (!c || !out) return fail(KVD_EINVAL, "NULL argument");
    KVD_CUDA(cudaDeviceSynchronize());
    unsigned long long v[5];
    KVD_CUDA(cudaMemcpy(v, c->stats, sizeof v, cudaMemcpyDeviceToHost));
    out->selected = v[0];
    out->hits = v[1];
    out->misses = v[2];
    out->pinned = v[3];
    out->fetched_bytes = v[4];
    return KVD_OK;
}

kvd_status kvd_reset_stats(kvd_cache* c) {
    if (!c) return fail(KVD_EINVAL, "cache is NULL");
    KVD_CUDA(cudaDeviceSynchronize());
    KVD_CUDA(cudaMemset(c->stats, 0, 64));
    KVD_CUDA(cudaMemset(c->seg_stats, 0, (size_t)c->L * c->Hkv * 16));
    KVD_CUDA(cudaDeviceSynchronize());
    return KVD_OK;
}

kvd_status kvd_check(kvd_cache* c) {
    if (!c) return fail(KVD_EINVAL, "cache is NULL");
    KVD_CUDA(cudaDeviceSynchronize());
    int32_t e = 0;
    KVD_CUDA(cudaMemcpy(&e, c->err, 4, cudaMemcpyDeviceToHost));
    if (e) {
        KVD_CUDA(cudaMemset(c->err, 0, 4));
        return fail(KVD_EDEVICE, "device flagged bad input (code %d: %s)", e,
                    (e & 1) ? "selection not ascending / out of range / pinned"
                    : (e & 2) ? "LFU key bounds exceeded"
                    : (e & 4) ? "hierarchical index candidate bound violated" : "append found no slot");
    }
    return KVD_OK;
}

}  // extern "C"
