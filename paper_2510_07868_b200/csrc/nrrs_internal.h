// nrrs_internal.h -- kernel parameter blocks shared by nrrs_kernels.cu and the
// C ABI layer (nrrs_capi.cu).  Not part of the public ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/nrrs_gpu.h"

namespace nrrs {

// Device-side launch bookkeeping of the look-back kernels (nrrs_device.cuh):
// claim = [63:32] epoch | [31:0] tiles claimed; done = CTAs finished.
struct LaunchSync {
    unsigned long long claim;
    unsigned int done;
    unsigned int pad;
};

// infer_kernel template kinds
enum : int {
    kKindHeuristic = 0,  // Fixed / Throughput / depth-1 pin (no MMA)
    kKindAdrrs = 1,      // ADRRS-NN: StatNet -> adrrs_factor
    kKindNrrs = 2,       // NRRS: StatNet -> build_nrrs_input -> RRSNet
    kKindAid = 3,        // AID-NRRS: own grid + tail -> RRSNet
    kKindStats = 4       // predict_stats batch (StatNet outputs only)
};

// One MLP layer inside the smem weight blob (byte offsets from the blob start).
// W_hi / W_lo are the fp16 split of [W | bias] in the UMMA K-major canonical
// layout (N rows x K cols, 8x16B core matrices, LBO = 128 B, SBO = K*16 B).
// The bias is a weight column multiplied by a constant-ones input column:
// either a dedicated K16 slice (`ones_slice`, 2 MMA terms) or, for the 11-input
// NRRS RRSNet layer, input column 11 of the single K16 slice.
constexpr uint32_t kNoBias = 0xFFFFFFFFu;

// One MLP layer in the smem weight blob: W_hi (N x K) immediately followed by
// W_lo (N x K), both fp16 in the UMMA K-major SWIZZLE_NONE canonical layout, so
// [W_hi ; W_lo] is one 2N x K operand; fp32 bias[N] at `bias` (kNoBias: the
// bias is a weight column of an input that is constant 1).
struct LayerDesc {
    uint32_t w_hi, w_lo;
    uint16_t K, N;        // K in {16, 32}, N in {16, 32}
    uint32_t bias;        // blob byte offset of the fp32 bias, or kNoBias
};

struct NetDesc {
    LayerDesc layer[4];
};

struct KernelNets {
    NetDesc stat, rrs;
};

// Hash-grid tables on the device: kPairCopies copies of the reference layout
// [level][entry][feature], `copy_stride` entries apart:
//   copy 0: the reference table (pairs (e, e^1) share an aligned pair)
//   copy 1: hashed levels: permuted so (e, e^3) share a pair; dense levels: shifted by one entry
//   copy t: hashed levels: permuted so (e, e^(2^(t+1)-1)) share a pair
// A hashed x-edge (cx, cx+1) has entries e and e ^ (2^(t+1)-1), t = trailing ones of cx,
// so copy t serves it with one gather when t < kPairCopies (all but 2^-kPairCopies of edges).
#ifndef NRRS_PAIR_COPIES
#define NRRS_PAIR_COPIES 8
#endif
#ifndef NRRS_PAIR_COPIES_F32
#define NRRS_PAIR_COPIES_F32 8
#endif
constexpr uint32_t kPairCopies = NRRS_PAIR_COPIES;         // fp16 AID grid (1 MiB per copy; sweep DESIGN.md 3a)
constexpr uint32_t kPairCopiesF32 = NRRS_PAIR_COPIES_F32;  // fp32 StatNet grid (2 MiB per copy)

struct GridDev {
    int32_t levels;
    int32_t base_resolution;
    uint32_t table_size;
    uint32_t dense_mask;  // bit l: level l is dense ((res+1)^3 <= T, hashgrid.hpp / hashgrid.cpp:16-22)
    uint64_t copy_stride; // entries between table copies (= levels * table_size)
    uint32_t pair_copies; // usable copies: t < pair_copies needs 2^(t+1) <= table_size
};

// Peer mailbox of the in-kernel rank exchange (replaces the two 8-byte
// all-gathers per depth of wavefront.cpp:141-154 / rrs.cpp:8-24 across ranks).  Each rank's
// mailbox holds, per kind (0: the rank's sum of q as f64 bits, 1: its realized total) and per
// SOURCE rank, one 64-byte line {generation, value}.  A rank writes its value into its line of
// EVERY rank's mailbox (peer mappings over NVLink / NVSwitch, CUDA IPC), value first, then the
// generation with release semantics at system scope; a waiter polls only its own mailbox.
// Generations are device counters advanced by the publishing kernel itself, so the protocol
// needs no host round trip and stays valid under CUDA graph replay.
constexpr int kMboxMaxRanks = 8;
constexpr int kMboxLineWords = 8;  // u64 words per line
constexpr int kMboxKinds = 2;
constexpr size_t kMboxBytes = (size_t)kMboxKinds * kMboxMaxRanks * kMboxLineWords * 8;
struct MboxDev {
    unsigned long long *peer[kMboxMaxRanks];  // every rank's mailbox (own included), mapped here
    uint32_t *gen;                            // this rank's generation per kind [kMboxKinds]
    uint32_t *err;                            // set to 1 when a wait times out
    double *sums_seen;                        // [nranks] rank sums the last decide used (rank order)
    unsigned long long *totals_seen;          // [nranks] rank totals the last clip used
    int32_t nranks, rank;
};

// Device-side scalar results of one stage call (mirrors nrrs_stage_result).
struct DevResult {
    double f_norm;
    double sum_q;
    unsigned long long sum_fx[2];  // the exact fixed-point sum (lo, hi) sum_q is converted from
    unsigned long long total;
    unsigned long long dropped;
    unsigned long long nonfinite;
    unsigned long long box_cox_clamps;
    uint32_t spawned;
    uint32_t overflow;
};

struct InferParams {
    const float *p01, *wo01, *roughness, *weight, *i_pixel;
    const uint64_t *path_key;
    const uint32_t *pixel;
    const float *i_acc;
    uint64_t n;
    uint32_t depth;
    int32_t gate;       // 1: stage semantics (depth pin, lum gate, sanitize); 0: raw factor
    int32_t heur_kind;  // 0 fixed, 1 throughput
    float fixed_value;
    float eps;          // max(eps_div, 1e-8)
    uint64_t mixed_seed;  // mix_bits(seed)
    const float2 *stat_grid;
    const void *rrs_grid;   // fp32 (float2 entries) or fp16 (half2 entries) when rrs_half
    uint32_t rrs_half;
    GridDev grid;        // StatNet grid (fp32)
    GridDev grid_rrs;    // AID RRSNet grid (same spec; its own number of pair copies)
    float2 *feat;          // K-A0 planes: AID [levels][feat_stride] float2; StatNet kinds [levels*2][feat_stride] float
    uint64_t feat_stride;
    const float *stat_fm;  // feature-major copy of the fp32 StatNet grid (K-A0 for ADRRS-NN / stats / NRRS)
    const uint8_t *blob;
    uint32_t blob_bytes;
    KernelNets nets;
    float *q_out, *u_out;
    uint8_t *decided_out;
    float *stats_out;
    double *parts;     // [grid] per-CTA partial sums
    uint32_t *part_counts; // [2*grid] per-CTA nonfinite / box_cox clamp counts
    uint32_t *counter; // last-CTA-done counter (self-resetting)
    double *sum_out;   // local sum of q
    DevResult *res;
    uint32_t accumulate;  // chunked launches: add to res counters / sum_q instead of overwriting
    uint32_t in_bulk;  // set by launch_aid_fused: K-A stages row inputs by TMA (aligned inputs)
    uint32_t ablate;   // debug only (env NRRS_DEBUG_ABLATE): bit0 skip grid gathers, bit1 skip MLP
    unsigned long long *dbg;  // debug only (env NRRS_DEBUG_TIMING): per-CTA clock64 phase counters [grid][16]
    const MboxDev *mbox;      // sharded mailbox mode: the last CTA publishes the rank's sum of q
};

// The fused AID-NRRS stage (nrrs_fused.cu): factor inputs + decision outputs.
struct AidStageParams {
    InferParams f;         // inputs, nets, grid, gate, seed; f.q_out / f.u_out: q_orig / u (optional when
                           // park_tmem), f.decided_out optional; f.parts / part_counts / sum_out / res used
    float2 *ring;          // level-plane ring [3][levels][ctas][4 * 128]
    uint32_t *sync;        // grid barrier + ring counters (aid_stage_sync_words, zeroed once)
    uint64_t *state;       // per-CTA prefix words [ctas * kStatePad]
    uint64_t n_pixels;
    float gain;
    uint32_t capacity;
    uint32_t parent_base;
    float *q_norm, *q_real;
    int32_t *k_out;
    uint32_t *offset;
    uint32_t *slots;
    unsigned long long *total_out;
    uint32_t tpc, rounds, park_tmem;
    unsigned long long *dbg;  // NRRS_KERNEL_TIMING builds only: per-CTA %globaltimer role stamps [cta][8]
};

struct DecideParams {
    const float *q, *u;
    const int32_t *counts_in;
    uint64_t n;
    const double *rank_sums;
    const unsigned long long *rank_sums_fx;  // optional: the ranks' exact sums (lo, hi) x nranks, added exactly
    int32_t nranks;
    uint64_t n_pixels;
    float gain;
    uint32_t capacity;
    uint32_t parent_base;
    float *q_norm, *q_real;
    int32_t *k_out;
    uint32_t *offset;
    uint32_t *slots;
    uint64_t *tile_state;
    uint32_t state_cap;     // entries of tile_state (cleared on epoch wrap)
    LaunchSync *sync;       // device-side claim counter + epoch (graph-replay safe)
    uint32_t num_tiles;
    uint32_t *err_flag;
    unsigned long long *total_out;
    DevResult *res;
    uint32_t tile_items;      // items per tile (multiple of 512; set by launch_decide / launch_compact)
    uint32_t single_wave;     // every tile resident at once: prefix = sum of predecessor aggregates
    unsigned long long *dbg;  // NRRS_KERNEL_TIMING builds only: per-tile %globaltimer phase stamps [tile][8]
    const MboxDev *mbox;      // sharded mailbox mode: rank sums from the mailbox, total published to peers
};

struct CompactParams {
    const void *in;
    const uint8_t *used;
    uint64_t count;                        // launch bound
    const unsigned long long *count_in;    // optional device count (clamped to `count`)
    void *out;
    uint32_t *count_out;
    uint64_t *tile_state;
    uint32_t state_cap;
    LaunchSync *sync;
    uint32_t num_tiles;
    uint32_t tile_items;      // items per tile (multiple of 512; set by launch_decide / launch_compact)
    uint32_t single_wave;     // every tile resident at once: prefix = sum of predecessor aggregates
    unsigned long long *dbg;  // NRRS_KERNEL_TIMING builds only: per-tile %globaltimer phase stamps [tile][8]
};

// TrainSample emission for one depth (nrrs_film.cu).
struct TrainParams {
    const float *p01, *wo01, *roughness, *weight;
    const uint32_t *pixel;
    const float *q_norm, *q_real;
    const uint8_t *decided;
    const double *s;
    const float *i_acc;
    uint64_t n;
    uint32_t depth;
    nrrs_train_sample *out;
    uint64_t capacity;
    const unsigned long long *base_in;  // samples already in `out` (device)
    unsigned long long *base_out;       // base_in + this depth's samples (device)
    unsigned long long *nonfinite;
    uint32_t *err;
    uint64_t *tile_state;
    uint32_t state_cap;
    LaunchSync *sync;
    uint32_t num_tiles;
};

uint32_t emit_tiles(uint64_t n);
cudaError_t launch_fold_ordered(double *dst, uint64_t n_dst, const int32_t *keys, const double *terms, uint64_t n,
                                uint32_t *err, cudaStream_t stream);
cudaError_t launch_film_add_frame(double *sum, uint32_t *samples, float *i_cur, const double *frame, uint64_t n,
                                  int num_sms, cudaStream_t stream);
cudaError_t launch_film_roll_acc(float *i_acc, const float *i_cur, uint64_t n, int num_sms, cudaStream_t stream);
cudaError_t launch_emit_train(const TrainParams &p, cudaStream_t stream);
cudaError_t launch_k_i(nrrs_train_sample *s, uint64_t start, const unsigned long long *end, uint64_t capacity,
                       uint32_t *hist, uint32_t n_pixels, int num_sms, cudaStream_t stream);

// StatNet training step (nrrs_train.cu)
struct TrainGrid {
    int32_t levels, base_resolution;
    uint32_t table_size, dense_mask;
};
// HashGrid::encode_backward without float atomics: every (sample, level, corner) contribution
// w * d_out goes to slot (s * levels + l) * 8 + c with its entry as key; a stable radix sort by
// entry then sums each entry's run sequentially in slot order -- the reference's own loop order
// (hashgrid.cpp:84-103), so the gradient is bit-identical from run to run.
// Grid-gradient contributions, level-major: slot (level * n + sample) * 8 + corner, so each level's
// contributions are one segment in (sample, corner) order and the per-entry order is the reference's
// loop order (sample, level, corner).  Each segment is sorted by its own entry bits on its own
// stream (levels run concurrently), the fold then walks the concatenation.
constexpr int kScatterMaxLevels = 8;
struct GridScatter {
    uint32_t *keys, *keys_sorted;  // [n * levels * 8]; keys (level << key_shift) | 2 * entry; pre-set to 0xFFFFFFFF
    float2 *vals, *vals_sorted;    // [n * levels * 8]; sorted along with the keys (stable)
    void *sort_tmp;                // levels x seg_tmp_bytes
    size_t seg_tmp_bytes;
    uint64_t seg;                  // contributions per level (n * 8)
    int levels;
    int key_end_bit;               // sorted key bits [1, key_end_bit) of one level's segment: the entry, plus
                                   // one bit only the sentinel sets, so it sorts after the level's last entry
    uint32_t key_shift;            // 2 + log2 T: the level field of a key
    uint32_t level_stride;         // gradient floats per level (2 * table size)
    uint64_t ngrid;                // floats of the gradient grid (bounds-checked builds)
    cudaStream_t side[kScatterMaxLevels];
    cudaEvent_t fork, join[kScatterMaxLevels];
};
size_t grid_scatter_sort_bytes(uint64_t contributions, int end_bit);

struct TrainStepParams {
    const nrrs_train_sample *batch;
    uint64_t n;
    const float *theta_grid;  // live StatNet grid, reference layout [level][entry][feature]
    const float *mlp;         // live StatNet MLP theta (mlp.cpp:7-32 layout)
    int32_t in;               // StatNet input width (levels * 2 + 16)
    TrainGrid grid;
    float eps, d_scale, inv_n;
    float *ws;                // per-sample workspace
    float *g_grid;            // zeroed by the caller
    double *loss_parts;       // [blocks]
    GridScatter scatter;      // deterministic grid-gradient scatter (launch_*_train fills it)
};
struct RrsStepParams {
    const nrrs_train_sample *batch;
    uint64_t n;
    int32_t variant;                     // 0 NRRS, 1 AID
    int32_t in;                          // RRSNet input width (11 or levels * 2 + 16)
    TrainGrid grid;
    const float *snap_grid, *snap_mlp;   // published StatNet snapshot
    const float *rrs_grid, *rrs_mlp;     // live RRSNet (rrs_grid: AID only)
    const float *errors;                 // PixelError {e, inv_denom} per pixel
    uint64_t n_errors;
    float e_avg;
    int32_t phase;                       // 0 Warmup, 1 Full
    float gamma_min, gamma_avg, gamma_rrs, eps, d_scale, inv_n;
    float *ws;
    float *g_grid;                       // zeroed by the caller (AID)
    double *parts;                       // [blocks][3] min, avg, rrs
    uint32_t *skipped;
    GridScatter scatter;                 // deterministic grid-gradient scatter (launch_*_train fills it)
};
struct AdamParams {
    float lr, beta1, beta2, eps, c1, c2, inv_scale, decay;
};
size_t train_ws_floats(uint64_t n);
int train_param_count(int in);
int train_rrs_param_count(int in);
cudaError_t launch_rrs_train(const RrsStepParams &p, float *partials, uint32_t dw_ctas, float *g_mlp,
                             double *parts_out, uint32_t *nonfinite, uint64_t ngrid, cudaStream_t stream);
uint32_t train_dw_ctas(uint64_t n);
cudaError_t launch_stat_train(const TrainStepParams &p, float *partials, uint32_t dw_ctas, float *g_mlp,
                              double *loss_out, uint32_t *nonfinite, uint64_t ngrid, cudaStream_t stream);
cudaError_t launch_adam_ema(float *theta, const float *grad, float *m, float *v, float *shadow, uint64_t n,
                            const AdamParams &a, int num_sms, cudaStream_t stream);

// Render front-end (nrrs_render.cu): Bvh::Node (geometry.hpp) flattened for the device
struct alignas(16) BvhNodeDev {
    float lo[3], hi[3];
    uint32_t offset;  // leaf: first prim; inner: right child (left child = this + 1)
    uint16_t count;   // > 0: leaf
    uint8_t axis, pad;
};
struct RenderScene {
    const float *pos;            // [3 * n_vert]
    const uint32_t *idx;         // [3 * n_tri]
    const uint32_t *mat_of_tri;  // [n_tri]
    const BvhNodeDev *nodes;
    const uint32_t *prims;
    // per BVH prim slot: {p0.xyz, e1.x}, {e1.yz, e2.xy}, {e2.z, triangle id bits, 0, 0} (host-computed
    // v1 - v0 / v2 - v0, the same IEEE subtractions as intersect_triangle, geometry.cpp:45-47)
    const float4 *tri4;
    uint32_t n_nodes, n_tri;
    const int32_t *mat_kind;     // 0 diffuse, 1 conductor
    const float *mat_albedo, *mat_roughness, *mat_emission;
    float norm_offset[3], norm_scale;
    float cam_pos[3], cam_fwd[3], cam_right[3], cam_up[3], tan_half, aspect;
    // Scene::finalize's light list (scene.cpp:38-47) and env_emission
    const uint32_t *light_tris;
    const float *light_areas;
    const int32_t *light_index;  // [n_tri], -1 = not a light
    uint32_t n_lights;
    float env[3];
};
// PathState (wavefront.hpp:17-26), 72 bytes = 18 words (compact_kernel<18>)
struct PathStateDev {
    float o[3], d[3], t_max, w[3];
    uint64_t key;
    float prev_pdf, rrs;
    uint32_t pixel;
    int32_t parent;
    uint16_t depth, pad16;
    uint32_t pad;
};
static_assert(sizeof(PathStateDev) == 72, "PathState is 72 bytes");
// VertexRec (wavefront.cpp:46-65) of one depth, SoA; s starts as the emission term
struct VertexRecDev {
    float *p, *n_s, *wo, *weight, *p01, *wo01, *rough;
    uint32_t *material, *pixel;
    int32_t *parent;
    uint64_t *key;
    float *rrs, *q_norm, *q_real;
    uint8_t *decided;
    int32_t *k;
    uint32_t *offset;
    double *s;
};
struct TraceCounters {
    unsigned long long shadow_rays, nonfinite;
};
cudaError_t launch_trace_camera(const RenderScene &s, uint32_t width, uint32_t height, uint64_t mixed_seed,
                                uint32_t frame, PathStateDev *q, int num_sms, cudaStream_t stream);
cudaError_t launch_trace_shade(const RenderScene &s, const PathStateDev *q, uint32_t n, uint32_t depth,
                               uint8_t *cls, uint8_t *is_surf, float *hit_t, uint32_t *pair, double *term,
                               float *normals, uint32_t *err, int num_sms, cudaStream_t stream);
cudaError_t launch_trace_records(const RenderScene &s, const PathStateDev *q, const uint32_t *surf, const uint32_t *ns,
                                 uint32_t n_max, const float *hit_t, uint32_t *rank, VertexRecDev v, uint32_t depth,
                                 float *normals, int num_sms, cudaStream_t stream);
cudaError_t launch_trace_scatter(const RenderScene &s, VertexRecDev v, const uint32_t *slots, uint32_t spawned,
                                 uint32_t depth, uint64_t mixed_seed, PathStateDev *next, uint8_t *used,
                                 double *slot_term, TraceCounters *cnt, int num_sms, cudaStream_t stream);
cudaError_t launch_trace_fold_frame(const PathStateDev *q, uint32_t n, const uint8_t *cls, const double *term,
                                    const uint32_t *rank, VertexRecDev v, uint32_t spawned, const double *slot_term,
                                    double *frame, cudaStream_t stream);
cudaError_t launch_trace_fold_parent(const PathStateDev *q, uint32_t n, const uint8_t *cls, const double *term,
                                     double *up_s, cudaStream_t stream);
cudaError_t launch_camera(const RenderScene &s, uint32_t width, uint32_t height, uint64_t mixed_seed, uint32_t frame,
                          float *o, float *d, uint64_t *keys, int num_sms, cudaStream_t stream);
cudaError_t launch_intersect(const RenderScene &s, const float *o, const float *d, const float *tmax, uint64_t n,
                             float *t, uint32_t *tri, float *u, float *v, uint32_t *err, int num_sms,
                             cudaStream_t stream);
cudaError_t launch_surface(const RenderScene &s, const float *o, const float *d, const float *t, const uint32_t *tri,
                           uint64_t n, uint8_t *cls, float *p01, float *wo01, float *rough, uint32_t *material,
                           int num_sms, cudaStream_t stream);

size_t infer_smem_bytes(int kind, const InferParams &p);
// K-A0: one hash-grid level per CTA from shared memory (fp16 tables, T * 4 B <= kLevelSmemMax).
struct GridLevelParams {
    const float *p01;
    uint64_t n;
    const void *table;  // fp16 reference layout [level][T] half2 (copy 0 of the AID grid), or with f32:
                        // the fp32 StatNet grid feature-major [level][feature][T]
    GridDev g;
    float2 *feat;       // planes: [level][stride] float2, or with f32 [level * 2 + feature][stride] float
    uint64_t feat_stride;
    uint32_t f32;
};
constexpr uint32_t kLevelSmemMax = 150u * 1024u;  // table bytes; + 72 KB of staged p01 blocks <= 227 KB
cudaError_t launch_grid_levels(const GridLevelParams &p, int num_sms, cudaStream_t stream);
cudaError_t launch_sharded_clip(const unsigned long long *totals, int nranks, int rank, uint32_t capacity,
                                unsigned long long *out, cudaStream_t stream);
cudaError_t launch_infer(int kind, const InferParams &p, int num_sms, cudaStream_t stream, uint32_t *grid_out);
uint32_t infer_max_grid(int num_sms);
// Upper bounds of the look-back tile count (state array sizes); the launchers pick the tile shape
// (one wave of <= num_sms tiles when the batch fits) and fill num_tiles / tile_items / single_wave.
uint32_t decide_tiles(uint64_t n);
cudaError_t launch_decide(int src, DecideParams p, int num_sms, cudaStream_t stream);
uint32_t compact_tiles(uint64_t count, uint32_t words);
cudaError_t launch_compact(uint32_t words, CompactParams p, int num_sms, cudaStream_t stream);
cudaError_t launch_grid_copies(const float *src, void *dst, uint32_t levels, uint32_t T, uint32_t copies,
                               uint32_t dense_mask, bool half, cudaStream_t stream);
cudaError_t launch_max_abs(const float *x, uint64_t n, unsigned int *out_bits, cudaStream_t stream);
cudaError_t launch_feature_major(const float *src, float *dst, uint32_t levels, uint32_t T, cudaStream_t stream);
void set_pdl(bool on);  // programmatic dependent launches for K-A / K-B / K-C (NRRS_PDL)
// fused AID stage (nrrs_fused.cu)
size_t aid_stage_smem_bytes(uint32_t blob_bytes, uint32_t table_size);
uint32_t aid_stage_ring_floats2(uint32_t levels, uint32_t ctas);
uint32_t aid_stage_sync_words();
bool aid_stage_shape(uint64_t n, int num_sms, uint32_t levels, uint32_t *ctas, uint32_t *tpc, uint32_t *rounds,
                     uint32_t *park);
cudaError_t launch_aid_stage(const AidStageParams &p, uint32_t ctas, cudaStream_t stream);
cudaError_t launch_lum_sum(const float *i_acc, uint64_t n, double *parts, uint32_t *counter, double *sum_out,
                           uint32_t grid, cudaStream_t stream);
cudaError_t launch_sum_check(const float *q, uint64_t n, double *parts, uint32_t *counter, uint32_t *err,
                             double *sum_out, uint32_t grid, cudaStream_t stream);
cudaError_t launch_scale(float *q, uint64_t n, const double *sum, uint64_t n_pixels, const uint32_t *err,
                         double *f_out, int num_sms, cudaStream_t stream);
cudaError_t launch_realize(const float *q, const float *u, int32_t *counts, uint64_t n, uint32_t *err,
                           unsigned long long *total, int num_sms, cudaStream_t stream);

// Mailbox mode: waits for every rank's realized total of this depth and applies the global clip
// (base, kept, spawned, dropped -> out[0..3], as sharded_clip_kernel); one thread.
cudaError_t launch_mbox_clip(const MboxDev *m, uint32_t capacity, unsigned long long *out, double *sums_out,
                             unsigned long long *totals_out, cudaStream_t stream);
// Mailbox mode, empty rank: publishes `value` for `kind` (one thread).
cudaError_t launch_mbox_publish(const MboxDev *m, int kind, unsigned long long value, cudaStream_t stream);

}  // namespace nrrs
