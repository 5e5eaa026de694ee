// internal.h — libkvd's cache object and the launch interface of its kernels.
// Layouts:
//   slots      [L][R][Hkv][C] records; record = K[P][128] || V[P][128] bf16,
//              each 256-B token row stored as 16 chunks of 16 B, chunk c of row
//              t at position c ^ (t & 7)  (bank-conflict-free ldmatrix)
//   host store [A][R][Hkv][nb_max] records (same layout), pinned + mapped
//   summ       [L][R][Hkv][128][nb_pad] bf16, dim-major (row = one dim j)
//   scores     [L][R][Hkv][nb_pad] fp32 (last select of that layer)
//   table      [L][R][Hkv][nb_pad] int32 block -> slot | -1
//   slot_block/last_use/phase/use_count [L][R][Hkv][C]
//   miss       [R][Hkv][kmax] int2 (block, slot) + miss_count [R][Hkv]
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#include "../../include/kvd.h"

namespace kvd {

constexpr int kScoreCols = 128;       // nb_pad is a multiple of this (summary / table rows)

constexpr int kAttnWarps = 4;         // warps per attention CTA
constexpr int kAttnStages = 3;        // smem stages per warp
constexpr int kTileBytes = 8192;      // one 16-token K||V tile
constexpr int kMaxSelectBlocks = 8 * 1024 * 32;   // select cluster capacity: 8 CTAs x 1024 threads x 32 keys
constexpr int kMaxPieces = 32;        // attention pieces (partials) per (request, KV head) (k_attn.cu)
constexpr int kPieceTiles = 8;        // 16-token tiles per attention piece (at least)
constexpr int64_t kSlotOfBytes = 64ll << 20;   // setup scratch for per-block slot targets

struct SegGeom {                      // per-request pinned geometry (device copy in params)
    int32_t n, nb, sink_end, local_begin;   // pinned = [0, sink_end) U [local_begin, nb)
};

struct StepParams {
    int32_t B, layer, k, W;
    int32_t R, Hkv, Hq, G, P, E;      // E = 16 / P list entries per 16-token tile
    int64_t nb_pad, C, nb_max;
    int32_t sink_tokens, local_tokens;
    int32_t policy;
    uint32_t step;
    const uint32_t* step_dev;         // non-null: read the step on the device (graph replay)
    int32_t host_layer;
    int32_t rec_bytes;
    float scale_log2;
    unsigned long long* kt_slots;     // kvd_enable_kernel_timer: [L*R*kKtKinds][2], or NULL
    unsigned long long* kt_acc;       // [kKtKinds][2] (ns, launches)
    int32_t kt_base;                  // slot of (layer, first request): (layer*R + req[0]) * kKtKinds
    unsigned long long* exp_trace;    // experiment builds: phase stamps (NULL otherwise)
    // hierarchical index (kvd_config.index_ratio > 0): select_kernel's view for stage 1
    int32_t sel_mode;                 // 0 = block summaries; 1 = centroids of the segment (stage 1)
    int32_t sel_ratio;                // blocks per centroid (stage-1 fan-out, reading R27)
    int32_t sel_stride;               // stage 1: output stride per segment (m_max)
    const int32_t* sel_count;         // stage 1: centroids per segment [L][R][Hkv]
    const uint16_t* summ2;            // Quest min/max summaries (sel_mode 2): the maximum matrix
    int32_t h0, nh;                   // the launch's KV heads [h0, h0 + nh) (arrays keep all Hkv heads)
    // 1: every step kernel triggers its dependent launch right after its own griddepcontrol.wait
    // (the dependent's CTAs become resident and run their prologue while this kernel works; they
    // still wait for its completion).  c2 +3 %, c4 +7 %, c3 unchanged.  2: score / attention only.
    int32_t early_trigger;
    int32_t req[KVD_MAX_BATCH];
};

}  // namespace kvd

struct kvd_cache {
    kvd_config cfg;
    int L, Hq, Hkv, G, P, R, kmax, pmax, A, E;
    int64_t nmax, nb_max, nb_pad, C;
    bool resident;
    int64_t rec_bytes;
    int max_splits;
    int prio_hi = 0;                      // greatest stream priority of the device (host-link kernels)
    // device
    uint8_t* slots = nullptr;
    uint16_t* summ = nullptr;
    float* scores = nullptr;
    int32_t* table = nullptr;
    int32_t* slot_block = nullptr;
    uint32_t* last_use = nullptr;
    uint8_t* phase = nullptr;
    uint32_t* use_count = nullptr;
    int32_t* miss = nullptr;
    int32_t* miss_count = nullptr;
    int summary_kind = 0;                  // 0 mean key (R2); 1 Quest min (summ) / max (summ2) (R30)
    uint16_t* summ2 = nullptr;             // [L][R][Hkv][128][nb_pad] bf16 channel-wise maxima
    // hierarchical index (index_ratio > 0; k_index.cu, DESIGN.md §3 R27)
    int index_ratio = 0;
    int64_t nc_pad = 0;                    // centroid rows per segment (multiple of 128)
    int m_max = 0;                         // stage-1 centroids per segment at most
    uint16_t* cent = nullptr;              // [L][R][Hkv][128][nc_pad] bf16, dim-major
    float* cscores = nullptr;              // [L][R][Hkv][nc_pad] fp32 (stage-1 scores)
    int32_t* ncent = nullptr;              // [L][R][Hkv] centroids per segment
    int32_t* cent_of = nullptr;            // [L][R][Hkv][nb_pad] block -> centroid
    int32_t* memb = nullptr;               // [L][R][Hkv][nb_pad] blocks ordered by (centroid, block)
    int32_t* moff = nullptr;               // [L][R][Hkv][nc_pad + 1] member offsets
    int32_t* csel = nullptr;               // [R][Hkv][m_max] stage-1 selection (scratch)
    uint32_t* cand_bits = nullptr;         // [L][R][Hkv][nb_pad / 32] last step's stage-2 candidates
    uint8_t* idx_stage = nullptr;          // setup scratch of the index build
    float* warm_imp = nullptr;             // setup scratch of the importance warm-up [Hkv][nb_max]
    // 2D window scaling (R28): per layer-head capacity; per layer-head selection / miss counters
    std::vector<int64_t> cap_host;         // [L][Hkv]
    int32_t* cap_dev = nullptr;            // [L][Hkv]
    unsigned long long* seg_stats = nullptr;   // [L][Hkv][2]
    unsigned long long* kt_slots = nullptr;  // kernel timer (bench instrumentation)
    unsigned long long* kt_acc = nullptr;
    bool kt_on = false;
    unsigned long long* stats = nullptr;   // [5] kvd_stats fields
    int32_t* err = nullptr;
    int32_t* ntok_dev = nullptr;           // [L][R] token counts (kernels get the launch layer's row)
    uint8_t* zero_rec = nullptr;           // one zero record (padding entries)
    const uint32_t* step_dev = nullptr;    // kvd_set_device_step
    // setup staging (lazily allocated)
    uint16_t* stage_kv = nullptr;
    uint8_t* stage_rec = nullptr;
    uint16_t* stage_q = nullptr;                 // observation-window queries (warm-up)
    // host
    uint8_t* host_store = nullptr;          // pinned, mapped (UVA: same pointer on device)
    std::vector<int64_t> ntok;              // host copy of the token counts [L][R] (kvd_append_token grows them)
};

namespace kvd {
// launchers (return cudaGetLastError())
cudaError_t launch_prefix(kvd_cache* c, int layer, int req, const uint16_t* dk, const uint16_t* dv, int64_t n,
                          cudaStream_t s, const uint16_t* dq_obs = nullptr, int n_obs = 0);
cudaError_t launch_warm(kvd_cache* c, int layer, int req, const uint16_t* dk, const uint16_t* dq, int n_obs, int64_t n,
                        int32_t* slot_of, cudaStream_t s);                                  // k_warm.cu
cudaError_t launch_select(kvd_cache* c, const StepParams& p, const uint16_t* q, int32_t* out_ids, float* out_scores,
                          cudaStream_t s);
size_t resolve_smem_bytes(int64_t nkeys, int64_t kmax, int64_t nb_pad);   // k_resolve.cu
size_t resolve_static_smem();                                               // k_resolve.cu
void select_geometry(int64_t nb_pad, int segs, bool resident, int* nt, int* cl, int* kpt, int* v);   // k_select.cu
size_t select_smem_bytes(int nt, int kpt, int cl, int64_t kb);              // k_select.cu (dynamic)
bool select_fast_ok(int cl, int64_t span, int64_t kb);                      // k_select.cu
size_t select_static_smem();                                                // k_select.cu
constexpr size_t kMaxSmemBytes = 227 * 1024;
cudaError_t launch_resolve(kvd_cache* c, const StepParams& p, const int32_t* ids, int32_t* out_attn, cudaStream_t s);
cudaError_t launch_gather(kvd_cache* c, const StepParams& p, cudaStream_t s);
cudaError_t launch_index_build(kvd_cache* c, int layer, int req, int64_t n, cudaStream_t s);   // k_index.cu
cudaError_t launch_index_select(kvd_cache* c, const StepParams& p, const uint16_t* q, int32_t* out_ids,
                                float* out_scores, int32_t* out_attn, cudaStream_t s);   // k_index.cu
size_t cand_smem_bytes(int64_t nb_pad);                                                     // k_index.cu
size_t index_stage_bytes(int Hkv, int64_t nb_pad);                                          // k_index.cu
cudaError_t launch_select_centroids(kvd_cache* c, const StepParams& p, const uint16_t* q, cudaStream_t s);  // k_select.cu
constexpr int kIdxWindow = 64;        // blocks per k-means window (oracle OR_IDX_WIN)
constexpr int kIdxIters = 4;          // Lloyd rounds before the final assignment (OR_IDX_ITERS)
constexpr int kIdxFanout = 4;         // stage-1 centroids: ceil(kIdxFanout * k / ratio), >= k + pinned
constexpr int kCandCap = 16384;       // stage-2 candidates per segment at most (64 * m_max)
cudaError_t launch_shrink_capacity(kvd_cache* c, int layer, int head, int64_t cap, cudaStream_t s);   // k_resolve.cu
cudaError_t launch_append(kvd_cache* c, const StepParams& p, const uint16_t* k, const uint16_t* v, const int32_t* n,
                          cudaStream_t s);                                                  // k_append.cu
cudaError_t launch_zero_copy(const void* host, void* dev, size_t bytes, int ctas, cudaStream_t s);
cudaError_t launch_score(kvd_cache* c, const StepParams& p, const uint16_t* q, const uint16_t* mat,
                         const uint16_t* mat2, float* scores, cudaStream_t s);                // k_score.cu
cudaError_t launch_select_resolve(kvd_cache* c, const StepParams& p, const uint16_t* q, int32_t* out_ids,
                                  float* out_scores, int32_t* out_attn, cudaStream_t s);
cudaError_t launch_attention(kvd_cache* c, const StepParams& p, const uint16_t* q, const int32_t* attn, float* out,
                             float* out_lse, cudaStream_t s);

// Split-K plan of one segment's attention: its TS tiles are cut into NP pieces, a multiple of
// 4 (one thread-block cluster of NP/4 CTAs x 4 warps per segment, k_attn.cu) of about
// kPieceTiles tiles, 4 <= NP <= kMaxPieces; piece j = tiles [j*TS/NP, (j+1)*TS/NP).  A function
// of TS (i.e. of k) only -- not of how many segments share a launch or a GPU -- so every output
// is bit-identical however the requests are batched, chained or sharded.
__host__ __device__ inline int attn_pieces(int TS) {
    int c = (TS + 4 * kPieceTiles - 1) / (4 * kPieceTiles);
    c = c < 1 ? 1 : c > kMaxPieces / 4 ? kMaxPieces / 4 : c;
    return 4 * c;
}

__host__ __device__ inline SegGeom seg_geom(int64_t n64, int P, int sink, int local) {
    // 32-bit, shift-only (P in {1, 2, 4, 8, 16}; n < 2^27): every thread of the step kernels
    // evaluates this, so no 64-bit integer divisions
    const int lp = P >= 16 ? 4 : P >= 8 ? 3 : P >= 4 ? 2 : P >= 2 ? 1 : 0;
    const int32_t n = (int32_t)n64;
    SegGeom g;
    g.n = n;
    g.nb = (n + P - 1) >> lp;
    int32_t se = (sink + P - 1) >> lp;
    int32_t ft = n - local;
    if (ft < 0) ft = 0;
    int32_t lb = local > 0 ? (ft >> lp) : g.nb;
    if (lb > g.nb) lb = g.nb;
    if (se > lb) se = lb;                  // overlapping sink/local: all blocks pinned
    g.sink_end = se;
    g.local_begin = lb;
    return g;
}
}  // namespace kvd
