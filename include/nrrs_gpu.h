/*
 * nrrs_gpu.h -- C ABI of the B200 (sm_100a) NRRS per-bounce RRS stage.
 *
 * One batched call per depth replaces the per-vertex and serial calls the
 * reference makes inside trace_frame's RRS decision block
 * (/root/reference/proj/src/wavefront.cpp:363-411, slot layout :413-425,
 * compaction :488-497).  Every entry point names the reference interface it
 * replaces.  Plain pointers and sizes only; no torch or CUDA types appear in the
 * signatures (streams are passed as void*).
 *
 * Conventions:
 *  - every function returns an nrrs_status; 0 = ok.  EINVAL / ESIZE mirror the
 *    reference's fail() / std::invalid_argument cases (rrs.cpp:11-12, :37-38,
 *    wavefront.cpp:146-147, :198-211, encodings.hpp:22-23); ECUDA wraps a CUDA
 *    error.  nrrs_gpu_last_error() returns the message.
 *  - "d_" pointers are device pointers, "h_" pointers host pointers.
 *  - stream-ordered on the context's stream; one context per device per host
 *    thread; not re-entrant.  There is no CPU fallback: without a CUDA device
 *    nrrs_gpu_create fails with ECUDA.
 */
#ifndef NRRS_GPU_H
#define NRRS_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NRRS_GPU_ABI_VERSION 1

#if defined(__GNUC__)
#define NRRS_API __attribute__((visibility("default")))
#else
#define NRRS_API
#endif

typedef enum {
    NRRS_OK = 0,
    NRRS_EINVAL = 1, /* invalid argument / value the reference rejects with fail() */
    NRRS_ESIZE = 2,  /* size mismatch (realize_counts, set_weights block sizes) */
    NRRS_ECUDA = 3,  /* CUDA runtime error or no device */
    NRRS_ENCCL = 4,  /* reserved: collective failure (multi-rank driver) */
    NRRS_ESTATE = 5  /* call order: e.g. neural strategy before set_weights */
} nrrs_status;

/* StrategyKind, rrs.hpp:72-79 (same numbering). */
typedef enum {
    NRRS_FIXED = 0,
    NRRS_THROUGHPUT = 1,
    NRRS_ADRRS_TREE = 2, /* out of scope (octree cache): EINVAL */
    NRRS_ADRRS_NN = 3,
    NRRS_NRRS = 4,
    NRRS_AID_NRRS = 5
} nrrs_strategy_kind;

/* RrsVariant, networks.hpp:75 */
typedef enum { NRRS_VARIANT_NRRS = 0, NRRS_VARIANT_AID = 1 } nrrs_variant;

/* HashGridSpec, hashgrid.hpp:13-22.  features must be 2 and levels*2+16 <= 32. */
typedef struct {
    int32_t levels, features, base_resolution, log2_table_size;
} nrrs_grid_spec;

/* Snapshot parameter blocks as published by NeuralRrs::publish()
 * (networks.cpp:199-204) or read from an NRRSCK01 checkpoint
 * (networks.cpp:610-705): flat fp32 theta vectors in the reference's layout
 * (hash grid [level][entry][feature]; MLP per layer column-major W then bias,
 * mlp.cpp:7-32).  Host pointers; lengths are checked (ESIZE). */
typedef struct {
    int32_t variant;
    nrrs_grid_spec grid;
    const float *stat_grid; uint64_t stat_grid_len;
    const float *stat_mlp;  uint64_t stat_mlp_len;
    const float *rrs_grid;  uint64_t rrs_grid_len; /* empty for NRRS (networks.cpp:26-35) */
    const float *rrs_mlp;   uint64_t rrs_mlp_len;
} nrrs_net_weights;

/* Strategy, rrs.hpp:81-92 */
typedef struct {
    int32_t kind;      /* nrrs_strategy_kind */
    float fixed_value; /* Fixed only */
} nrrs_strategy;

/* Surface vertices entering the decision at one depth, SoA (the VertexRec
 * fields the stage reads, wavefront.cpp:46-65).  Vectors are packed xyz / xy
 * (Eigen Vec3f / Vec2f arrays).  i_pixel is film.i_acc[v.pixel]; pass NULL and
 * set pixel + i_acc to have the stage gather it (wavefront.cpp:378). */
typedef struct {
    const float *p01;       /* [3n] scene-normalized position */
    const float *wo01;      /* [2n] spherical omega_o in [0,1]^2 */
    const float *roughness; /* [n] */
    const float *weight;    /* [3n] path weight w (= t_x) */
    const float *i_pixel;   /* [3n] or NULL */
    const uint64_t *path_key; /* [n] */
    const uint32_t *pixel;  /* [n] (only if i_pixel == NULL) */
    const float *i_acc;     /* [3 * n_pixels] (only if i_pixel == NULL) */
} nrrs_vertex_soa;

typedef struct {
    uint32_t depth;    /* d >= 1; depth 1 pins q = 1 (wavefront.cpp:373-375) */
    uint32_t n_pixels; /* Npx of the normalization budget (rrs.cpp:8-24) */
    uint32_t capacity; /* queue capacity; 0 = queue_capacity_for(n_pixels) */
    nrrs_strategy strategy; /* Mix-Depth gate: assignment[depth-1] (wavefront.cpp:366) */
    float gain;        /* RateControl::gain() (rrs.hpp:30); applied iff depth >= 2 && adaptive */
    float eps_div;     /* ADRRS divisor guard (wavefront.cpp:238-243) */
    uint64_t seed;     /* TraceConfig::seed */
} nrrs_stage_params;

/* Per-vertex and per-slot outputs (device pointers).  q_norm, q_real and slots
 * are required; the rest may be NULL. */
typedef struct {
    float *q_norm;    /* [n] VertexRec::q_norm (wavefront.cpp:400) */
    float *q_real;    /* [n] VertexRec::q_real (wavefront.cpp:401) */
    uint32_t *slots;  /* [2 * capacity] (parent vertex j, child c) per queue slot, slot order */
    int32_t *k;       /* [n] realized counts (rrs.cpp:35-45) */
    uint32_t *offset; /* [n] SpawnPlan::offset (wavefront.cpp:141-154) */
    uint8_t *decided; /* [n] VertexRec::decided */
    float *q_orig;    /* [n] sanitized raw factor before normalization */
    float *u;         /* [n] RrsRound uniform */
} nrrs_stage_out;

/* Scalars of one stage call (FrameReport / SpawnPlan / RateControl inputs). */
typedef struct {
    double f_norm;           /* normalize_factors' return value */
    double sum_q;            /* sum of sanitized raw factors (this rank) */
    uint64_t total;          /* realized child count S */
    uint64_t dropped;        /* SpawnPlan::dropped (bias_drop_events) */
    uint64_t nonfinite;      /* FrameReport::nonfinite_drops increment */
    uint64_t box_cox_clamps; /* diag::box_cox_clamps increment (encodings.hpp:14-17) */
    uint32_t spawned;        /* SpawnPlan::spawned = next queue size before compaction */
    uint32_t overflow;       /* 1 iff dropped > 0: caller does rc.note_overflow() (wavefront.cpp:407-411) */
} nrrs_stage_result;

/* TrainSample (networks.hpp:20-32): 80 bytes, the reference's field order and layout. */
typedef struct {
    float position[3];  /* scene-normalized p01 */
    float omega_o[2];   /* wo01 */
    float roughness;
    float t_x[3];       /* path weight into the vertex */
    float i_pixel[3];   /* film.i_acc[pixel] */
    float lo_sample[3]; /* s / weight per channel (0 where weight <= 0) */
    float q_norm;
    float q_real;
    uint32_t pixel;
    float k_i;          /* this frame's samples in the pixel */
    uint16_t depth;
    uint16_t pad;
} nrrs_train_sample;

/* The VertexRec fields the suffix side reads, SoA for one depth (wavefront.cpp:46-65). */
typedef struct {
    const float *p01;       /* [3n] */
    const float *wo01;      /* [2n] */
    const float *roughness; /* [n] */
    const float *weight;    /* [3n] */
    const uint32_t *pixel;  /* [n] */
    const float *q_norm;    /* [n] */
    const float *q_real;    /* [n] */
    const uint8_t *decided; /* [n] */
    const double *s;        /* [3n] suffix contribution after the reverse pass */
} nrrs_vertex_rec_soa;

/* Material (bsdf.hpp:10-20) and Camera (scene.hpp:12-20) of a scene. */
typedef struct {
    int32_t kind;        /* 0 diffuse, 1 conductor */
    float albedo[3];
    float roughness;     /* GGX alpha, conductor only */
    float emission[3];
} nrrs_material;
typedef struct {
    float position[3], look_at[3], up[3];
    float vfov_deg;
} nrrs_camera;

typedef struct nrrs_scene nrrs_scene;
typedef struct nrrs_tracer nrrs_tracer;

/* TraceConfig (wavefront.hpp:128-140): the fields trace_frame reads. */
typedef struct {
    uint32_t width, height;
    int32_t max_depth;        /* B */
    uint32_t queue_capacity;  /* 0 = queue_capacity_for(W*H) */
    uint64_t seed;
    uint32_t frame_index;
    float adrrs_eps_scale;    /* 1e-4 in the reference */
    int32_t collect_training;
} nrrs_trace_config;

/* RateControl (rrs.hpp:23-36), updated in place on overflow. */
typedef struct {
    float f_rate, alpha, eps;
    int32_t enabled;
    uint64_t overflow_events;
} nrrs_rate_control;

/* FrameReport (wavefront.hpp:175-186). */
typedef struct {
    uint64_t camera_rays, scatter_rays, shadow_rays, nonfinite_drops, overflow_events, bias_drop_events,
        train_samples;
    uint32_t depth_counts[32];
} nrrs_frame_report;

/* Film (wavefront.hpp:78-123) on the device: sum [3n] f64, samples [n], i_cur / i_acc / normal [3n] f32. */
typedef struct {
    double *sum;
    uint32_t *samples;
    float *i_cur, *i_acc, *normal;
} nrrs_film_dev;
typedef struct nrrs_gpu_ctx nrrs_gpu_ctx;

/* ---- context ------------------------------------------------------------ */
NRRS_API int nrrs_gpu_abi_version(void);
NRRS_API int nrrs_gpu_create(int device, nrrs_gpu_ctx **out);
NRRS_API int nrrs_gpu_destroy(nrrs_gpu_ctx *ctx);
NRRS_API const char *nrrs_gpu_last_error(const nrrs_gpu_ctx *ctx);
NRRS_API int nrrs_gpu_set_stream(nrrs_gpu_ctx *ctx, void *cuda_stream);
/* Preallocate per-call scratch for up to max_vertices (no allocation in the hot path after). */
NRRS_API int nrrs_gpu_reserve(nrrs_gpu_ctx *ctx, uint64_t max_vertices, uint32_t max_capacity);
/* Count of kernel launches issued by this context since creation (bench evidence). */
NRRS_API uint64_t nrrs_gpu_launch_count(const nrrs_gpu_ctx *ctx);

/* ---- weights: replaces reading NeuralRrs' snapshot (networks.hpp:147, networks.cpp:276-279) */
NRRS_API int nrrs_gpu_set_weights(nrrs_gpu_ctx *ctx, const nrrs_net_weights *w);

/* The same with DEVICE pointers in w (e.g. the snapshot blocks just broadcast
 * over NCCL by the tile-sharded mode): the hash-grid table copies
 * are built on the device; only the two small MLP blocks are read back for
 * packing.  Same validation, error-budget gate and errors as nrrs_gpu_set_weights. */
NRRS_API int nrrs_gpu_set_weights_dev(nrrs_gpu_ctx *ctx, const nrrs_net_weights *w);

/* ---- fused stage (1 rank): replaces wavefront.cpp:363-425 for one depth:
 *   strategy_factor over ns vertices (:368-389), normalize_factors (:390),
 *   gain (:391), RrsRound uniforms (:393-402), realize_counts (:403-404),
 *   plan_spawns (:406) and the child slot layout (:421-425). Device buffers.
 *   h_result may be NULL (fully asynchronous); otherwise the call syncs the stream. */
NRRS_API int nrrs_gpu_rrs_stage(nrrs_gpu_ctx *ctx, const nrrs_vertex_soa *d_v, uint64_t n,
                       const nrrs_stage_params *p, const nrrs_stage_out *d_out,
                       nrrs_stage_result *h_result);

/* Synchronizes the context's stream and returns the scalars of the most recent
 * stage call (e.g. after replaying a CUDA graph that captured nrrs_gpu_rrs_stage
 * with h_result = NULL; the stage launches are graph-replay safe). */
NRRS_API int nrrs_gpu_fetch_result(nrrs_gpu_ctx *ctx, nrrs_stage_result *h_result);

/* Device address of the u64 realized child total (the reference's plan_spawns
 * `total` before the capacity clip, wavefront.cpp:141-154) that every
 * nrrs_gpu_rrs_stage call writes, so a stream-ordered consumer such as
 * nrrs_gpu_compact_dev (bounded by the capacity) can follow the stage without a
 * host round trip.  Stable for the context's lifetime. */
NRRS_API int nrrs_gpu_stage_total_dev(nrrs_gpu_ctx *ctx, const uint64_t **d_total);

/* Table precision chosen at nrrs_gpu_set_weights for the AID RRSNet grid: fp16
 * only when the error-budget probe (16,384 fixed vertices through the fp16 and
 * the fp32 tables of the same snapshot) keeps max |dq| / q <= 2.5e-4, a quarter
 * of the 1e-3 tolerance; *probe_rel_err < 0 when no probe ran (NRRS variant,
 * NRRS_FP32_TABLES, or |theta| beyond fp16 range). */
NRRS_API int nrrs_gpu_weights_info(nrrs_gpu_ctx *ctx, int32_t *aid_fp16_tables, double *probe_rel_err);

/* Per-frame ADRRS divisor input, replaces the film loop of trace_frame
 * (wavefront.cpp:238-243): *d_sum_out = sum over n_pixels of luminance(i_acc[p])
 * (f32 luminance, f64 sum, fixed order).  eps_div = eps_scale *
 * (float)(sum / n_pixels); in the tile-sharded mode sum the per-rank values in
 * rank order first.  Asynchronous on the context stream. */
NRRS_API int nrrs_gpu_film_luminance_sum(nrrs_gpu_ctx *ctx, const float *d_i_acc, uint64_t n_pixels,
                                         double *d_sum_out);

/* Same call over HOST buffers (the reference-facing plugin path): copies the
 * SoA to the device, runs the stage, copies every non-NULL output back.
 * h_out->slots receives result.spawned records. */
NRRS_API int nrrs_gpu_rrs_stage_host(nrrs_gpu_ctx *ctx, const nrrs_vertex_soa *h_v, uint64_t n,
                            const nrrs_stage_params *p, const nrrs_stage_out *h_out,
                            nrrs_stage_result *h_result);

/* Asynchronous form of nrrs_gpu_rrs_stage_host for a stream of independent
 * batches: enqueues the copies and the stage and returns a ticket.  Two calls
 * may be in flight per context (double-buffered device staging): the inputs of
 * call i+1 stream in while the outputs of call i stream out (PCIe is full
 * duplex).  Host buffers must stay valid until nrrs_gpu_stage_host_wait returns
 * for the ticket, and should be pinned for the copies to overlap.  h_out->slots
 * receives the whole [2 * capacity] array; records [0, result.spawned) are valid.
 * p->gain is taken as given: a caller running RateControl across calls applies
 * the overflow of call i to the first call it issues after waiting for i.
 * ESTATE when a third call is issued before the oldest one was waited for. */
NRRS_API int nrrs_gpu_rrs_stage_host_async(nrrs_gpu_ctx *ctx, const nrrs_vertex_soa *h_v, uint64_t n,
                                           const nrrs_stage_params *p, const nrrs_stage_out *h_out,
                                           uint64_t *ticket);
/* Blocks until the call `ticket` has finished and its outputs are in host memory. */
NRRS_API int nrrs_gpu_stage_host_wait(nrrs_gpu_ctx *ctx, uint64_t ticket, nrrs_stage_result *h_result);

/* ---- suffix side of trace_frame: film folds, reverse pass,
 * TrainSample emission, Film updates.  Bit-identical to the reference's sequential
 * f64 folds.  Device buffers; stream-ordered. */

/* d_dst[key[i]] += d_terms[i] (f64 x3) for i = 0..n-1 in item order.  Keys must be
 * non-decreasing (queue order is pixel and parent order); negative keys (no parent)
 * are skipped.  Replaces frame[pixel] += term (wavefront.cpp:299, :317, :355, :485),
 * parent.s += term (:301, :319) and, one call per depth d = B..2 with the depth-d
 * parent indices and s, the reverse pass (:505-507).  Syncs; EINVAL if the keys are
 * out of order or out of range. */
NRRS_API int nrrs_gpu_fold_ordered(nrrs_gpu_ctx *ctx, double *d_dst, uint64_t n_dst, const int32_t *d_keys,
                                   const double *d_terms, uint64_t n);

/* TrainSample emission for one depth (wavefront.cpp:510-537): one record per decided
 * vertex whose lo = s / weight is finite, in vertex order, written at
 * d_out[*d_count_in ...]; *d_count_out = *d_count_in + records (pass distinct counters;
 * call for depths 1..B-1 in order).  Non-finite lo adds to *d_nonfinite.  k_i is set by
 * nrrs_gpu_train_k_i.  Asynchronous. */
NRRS_API int nrrs_gpu_emit_train(nrrs_gpu_ctx *ctx, uint32_t depth, const nrrs_vertex_rec_soa *d_v, uint64_t n,
                                 const float *d_i_acc, nrrs_train_sample *d_out, uint64_t capacity,
                                 const uint64_t *d_count_in, uint64_t *d_count_out, uint64_t *d_nonfinite);

/* k_i of the frame's samples [start, *d_end) = number of those samples with the same
 * pixel (wavefront.cpp:539-543).  Syncs; ESIZE if an emission ran past capacity. */
NRRS_API int nrrs_gpu_train_k_i(nrrs_gpu_ctx *ctx, nrrs_train_sample *d_samples, uint64_t start,
                                const uint64_t *d_end, uint64_t capacity, uint32_t n_pixels);

/* Film::add_frame (wavefront.cpp:104-111): sum += frame, samples += 1, i_cur = float(frame). */
NRRS_API int nrrs_gpu_film_add_frame(nrrs_gpu_ctx *ctx, double *d_sum, uint32_t *d_samples, float *d_i_cur,
                                     const double *d_frame, uint32_t n_pixels);
/* Film::roll_acc (wavefront.cpp:113-116): i_acc = 0.5f * i_acc + 0.5f * i_cur. */
NRRS_API int nrrs_gpu_film_roll_acc(nrrs_gpu_ctx *ctx, float *d_i_acc, const float *d_i_cur, uint32_t n_pixels);

/* ---- online training, StatNet step ---- */

/* NeuralRrs::stat_loss_impl (networks.cpp:349-391) for one batch of TrainSamples on the
 * live StatNet parameters (reference layouts): batch-mean relative L2 of the 6 stats against
 * (lo, lo^2), and its gradient scaled by d_scale through Mlp::backward (mlp.cpp:74-111) and
 * HashGrid::encode_backward (hashgrid.cpp:84-103).  d_g_mlp / d_g_grid are overwritten;
 * *h_loss = the loss, *h_finite = 1 iff the loss and every gradient entry are finite (the
 * apply_step test, networks.cpp:462-470).  Syncs. */
NRRS_API int nrrs_gpu_stat_loss_grad(nrrs_gpu_ctx *ctx, const nrrs_grid_spec *spec, const float *d_stat_grid,
                                     const float *d_stat_mlp, const nrrs_train_sample *d_batch, uint64_t n,
                                     float eps, float d_scale, float *d_g_mlp, float *d_g_grid, double *h_loss,
                                     int32_t *h_finite);

/* NeuralRrs::rrs_loss_impl (networks.cpp:418-460) for one batch: stats from the published
 * StatNet snapshot (d_snap_*), the RRSNet (variant 0 NRRS / 1 AID; d_rrs_grid AID only) on
 * its live parameters.  phase 0 = Warmup (relative L2 of q to 1), 1 = Full (variance-
 * transfer gradients through d_errors = {e, inv_denom} per pixel, plus the recorded-factor
 * regression; gamma weights as NeuralRrsConfig).  Gradients scaled by d_scale overwrite
 * d_g_mlp / d_g_grid; h_parts = {min, avg, rrs, total} (networks.hpp:219-224); *h_skipped
 * counts samples without a pixel error; *h_finite as in nrrs_gpu_stat_loss_grad.  Syncs. */
NRRS_API int nrrs_gpu_rrs_loss_grad(nrrs_gpu_ctx *ctx, int32_t variant, const nrrs_grid_spec *spec,
                                    const float *d_snap_stat_grid, const float *d_snap_stat_mlp,
                                    const float *d_rrs_grid, const float *d_rrs_mlp,
                                    const nrrs_train_sample *d_batch, uint64_t n, const float *d_errors,
                                    uint64_t n_errors, float e_avg, int32_t phase, float gamma_min,
                                    float gamma_avg, float gamma_rrs, float eps, float d_scale, float *d_g_mlp,
                                    float *d_g_grid, double *h_parts, uint32_t *h_skipped, int32_t *h_finite);

/* apply_step's update (networks.cpp:471-478): grad *= inv_scale, Adam::step with the step
 * counter already advanced to t (optimizer.hpp:21-32), then the EMA shadow (optimizer.hpp:54-61;
 * d_shadow may be NULL).  Asynchronous. */
NRRS_API int nrrs_gpu_adam_ema(nrrs_gpu_ctx *ctx, float *d_theta, const float *d_grad, float *d_m, float *d_v,
                               float *d_shadow, uint64_t n, int64_t t, float lr, float beta1, float beta2,
                               float eps, float inv_scale, float ema_decay);

/* ---- render front-end (first part) ---- */

/* TriMesh + materials + camera on the device; the BVH is built on the host exactly like
 * Bvh::build (geometry.cpp:88-137: median split on the longest axis, nth_element, leaves of
 * <= 4) and Scene::finalize's normalization (scene.cpp:23-37).  Host arrays. */
NRRS_API int nrrs_gpu_scene_create(nrrs_gpu_ctx *ctx, const float *h_positions, uint32_t n_vertices,
                                   const uint32_t *h_indices, uint32_t n_triangles, const uint32_t *h_material_ids,
                                   const nrrs_material *h_materials, uint32_t n_materials,
                                   const nrrs_camera *camera, nrrs_scene **out);
NRRS_API int nrrs_gpu_scene_destroy(nrrs_scene *scene);
NRRS_API uint32_t nrrs_gpu_scene_node_count(const nrrs_scene *scene);
NRRS_API uint32_t nrrs_gpu_scene_light_count(const nrrs_scene *scene);
/* Scene::env_emission (scene.hpp:45), radiance of escaped rays */
NRRS_API int nrrs_gpu_scene_set_env(nrrs_scene *scene, const float env[3]);

/* Depth-1 camera rays of a width x height film (wavefront.cpp:253-268): pixel p's key is
 * root_path_key(p, frame), its jitter path_stream(seed, key, 1, CameraJitter).  d_o / d_d [3n],
 * d_keys [n].  Asynchronous. */
NRRS_API int nrrs_gpu_camera_rays(nrrs_gpu_ctx *ctx, const nrrs_scene *scene, uint32_t width, uint32_t height,
                                  uint64_t seed, uint32_t frame, float *d_o, float *d_d, uint64_t *d_keys);

/* Closest hits (Bvh::intersect, geometry.cpp:139-171); d_t_max may be NULL (inf).  Misses
 * return t = inf, tri = 0xFFFFFFFF.  d_u / d_v may be NULL.  Asynchronous. */
NRRS_API int nrrs_gpu_intersect(nrrs_gpu_ctx *ctx, const nrrs_scene *scene, const float *d_o, const float *d_d,
                                const float *d_t_max, uint64_t n, float *d_t, uint32_t *d_tri, float *d_u,
                                float *d_v);
/* Synchronizes the context stream and reports (then clears) a degenerate ray direction seen by
 * nrrs_gpu_intersect since the last check: NRRS_EINVAL with the reference's message. */
NRRS_API int nrrs_gpu_render_check(nrrs_gpu_ctx *ctx);

/* dispatch (wavefront.cpp:125-138: d_class 0 miss, 1 light, 2 surface) and the surface
 * vertex fields the RRS stage reads (wavefront.cpp:330-345): p01, wo01, roughness, material
 * (d_material may be NULL).  Asynchronous. */
NRRS_API int nrrs_gpu_surface_records(nrrs_gpu_ctx *ctx, const nrrs_scene *scene, const float *d_o,
                                      const float *d_d, const float *d_t, const uint32_t *d_tri, uint64_t n,
                                      uint8_t *d_class, float *d_p01, float *d_wo01, float *d_roughness,
                                      uint32_t *d_material);

/* ---- trace_frame on the GPU ---- */

/* Device queues and per-depth VertexRec storage for films up to max_pixels and depths up to
 * max_depth (capacity 0 = queue_capacity_for(max_pixels)). */
NRRS_API int nrrs_gpu_tracer_create(nrrs_gpu_ctx *ctx, uint32_t max_pixels, int32_t max_depth, uint32_t capacity,
                                    nrrs_tracer **out);
NRRS_API int nrrs_gpu_tracer_destroy(nrrs_tracer *tracer);

/* trace_frame (wavefront.cpp:217-551): camera rays, then per depth closest hits, dispatch, the
 * miss / emitter / emission film terms, the RRS stage with assignment[depth-1] (networks from
 * nrrs_gpu_set_weights), NEE + BSDF sampling per child slot, the ordered film folds and the
 * order-preserving compaction; then the reverse pass, TrainSample emission into d_train (appended
 * at *h_train_count, which is advanced) and Film::add_frame.  Film buffers are device pointers;
 * film->normal receives the depth-1 normals.  Synchronous (a few host reads per depth). */
NRRS_API int nrrs_gpu_trace_frame(nrrs_tracer *tracer, const nrrs_scene *scene, const nrrs_trace_config *cfg,
                                  const nrrs_strategy *assignment, nrrs_rate_control *rc, const nrrs_film_dev *film,
                                  nrrs_train_sample *d_train, uint64_t train_capacity, uint64_t *h_train_count,
                                  nrrs_frame_report *report);
/* The last frame's f64 radiance buffer [3 * W * H] (device) and depth-d vertex records. */
NRRS_API int nrrs_gpu_tracer_frame_buffer(const nrrs_tracer *tracer, const double **d_frame);
NRRS_API int nrrs_gpu_tracer_vertices(const nrrs_tracer *tracer, int32_t depth, nrrs_vertex_rec_soa *out,
                                      uint32_t *count);

/* ---- tile-sharded stage (multi-rank), two phases per depth:
 * phase 1: factors + RrsRound uniforms; writes this rank's sum of sanitized
 *          factors (double) to d_local_sum.  The caller all-gathers it.
 * phase 2: normalization with F = n_pixels_total / sum_r(d_rank_sums[r]) in
 *          rank order, gain, counts, local scan and local slot records
 *          (rank-local parent indices, clipped at p->capacity); writes the
 *          rank's realized total to d_local_total.  The caller all-gathers the
 *          totals; the global tail clip is then a count truncation of the
 *          rank's records (nrrs_gpu_sharded_clip). */
NRRS_API int nrrs_gpu_stage_factors(nrrs_gpu_ctx *ctx, const nrrs_vertex_soa *d_v, uint64_t n,
                           const nrrs_stage_params *p, const nrrs_stage_out *d_out,
                           double *d_local_sum);
NRRS_API int nrrs_gpu_stage_decide(nrrs_gpu_ctx *ctx, uint64_t n, const nrrs_stage_params *p,
                          const double *d_rank_sums, int32_t nranks,
                          const nrrs_stage_out *d_out, uint64_t *d_local_total);
/* Host arithmetic of the global clip: base_r = sum of totals of ranks < rank;
 * rank keeps min(total_r, cap - min(cap, base_r)) records. */
NRRS_API int nrrs_gpu_sharded_clip(const uint64_t *h_rank_totals, int32_t nranks, int32_t rank,
                          uint32_t capacity, uint64_t *h_base, uint32_t *h_kept,
                          uint32_t *h_spawned_global, uint64_t *h_dropped_global);
/* The same clip on the device, asynchronous on the context stream, so a depth of the
 * tile-sharded stage needs no host round trip: d_rank_totals = the all-gathered u64
 * totals (device), d_out[4] = base, kept, spawned (global), dropped (global). */
NRRS_API int nrrs_gpu_sharded_clip_dev(nrrs_gpu_ctx *ctx, const uint64_t *d_rank_totals, int32_t nranks,
                                       int32_t rank, uint32_t capacity, uint64_t *d_out);

/* Exact form of the two phases: the rank's sum of factors as the 128-bit fixed-point integer the
 * stage accumulates (2 x u64 lo, hi, bit-exactness), written to d_out after
 * nrrs_gpu_stage_factors; and phase 2 taking the all-gathered exact sums (2 x nranks words, rank
 * order), added exactly -- so the sharded F equals the one-rank F bit for bit. */
NRRS_API int nrrs_gpu_stage_local_sum_exact(nrrs_gpu_ctx *ctx, uint64_t *d_out);
/* The device address of the same two words inside the context (valid until the next stage call on
 * it), for exchanging them without a copy, e.g. as the send buffer of the all-gather. */
NRRS_API int nrrs_gpu_stage_sum_exact_dev(nrrs_gpu_ctx *ctx, const uint64_t **d_sum);
NRRS_API int nrrs_gpu_stage_decide_exact(nrrs_gpu_ctx *ctx, uint64_t n, const nrrs_stage_params *p,
                                         const uint64_t *d_rank_sums_exact, int32_t nranks,
                                         const nrrs_stage_out *d_out, uint64_t *d_local_total);

/* ---- in-kernel rank exchange over NVLink / NVSwitch peer memory (mailbox mode; DESIGN.md
 * section 7).  Replaces the caller's two all-gathers per depth (wavefront.cpp:141-154 and
 * rrs.cpp:8-24 across ranks): with a connected mailbox, nrrs_gpu_stage_factors' last CTA writes
 * the rank's sum of q into every rank's mailbox, nrrs_gpu_stage_decide_mbox waits for all N
 * sums in its own mailbox (summed in rank order, so F is identical on every rank) and its last
 * tile publishes the realized total, and nrrs_gpu_sharded_clip_mbox waits for the N totals and
 * applies the global clip -- no host round trip and no collective launch per depth.
 * Generations are device counters, so CUDA graph replays stay valid; every rank must run the
 * same sequence of depths.  A wait that sees no peer for 10 s raises the timeout flag
 * (nrrs_gpu_mailbox_status) instead of hanging. */
#define NRRS_IPC_HANDLE_BYTES 64
/* Allocates this rank's mailbox (zeroed): returns its CUDA IPC handle (NRRS_IPC_HANDLE_BYTES)
 * and, optionally, its device address (for ranks that share this process). nranks <= 8. */
NRRS_API int nrrs_gpu_mailbox_init(nrrs_gpu_ctx *ctx, int32_t nranks, int32_t rank, void *ipc_handle_out,
                                   uint64_t *d_addr_out);
/* Maps every rank's mailbox: ipc_handles = nranks x NRRS_IPC_HANDLE_BYTES in rank order (the
 * caller exchanges them, e.g. over the torch.distributed store); same_process_addrs (optional,
 * nranks entries): a nonzero entry is that rank's device address in this process, used directly. */
NRRS_API int nrrs_gpu_mailbox_connect(nrrs_gpu_ctx *ctx, const void *ipc_handles, const uint64_t *same_process_addrs);
/* Phase 2 of the mailbox mode (nrrs_gpu_stage_decide with the rank sums taken from the mailbox). */
NRRS_API int nrrs_gpu_stage_decide_mbox(nrrs_gpu_ctx *ctx, uint64_t n, const nrrs_stage_params *p,
                                        const nrrs_stage_out *d_out, uint64_t *d_local_total);
/* The global clip of the mailbox mode: d_out[4] as nrrs_gpu_sharded_clip_dev; optionally the
 * rank sums (f64) and totals (u64) this depth used, nranks entries each, rank order. */
NRRS_API int nrrs_gpu_sharded_clip_mbox(nrrs_gpu_ctx *ctx, uint32_t capacity, uint64_t *d_out,
                                        double *d_rank_sums_out, uint64_t *d_rank_totals_out);
/* Synchronizes the context stream; *timed_out = 1 if a mailbox wait gave up on a peer. */
NRRS_API int nrrs_gpu_mailbox_status(nrrs_gpu_ctx *ctx, int32_t *timed_out);

/* ---- order-preserving compaction of filled slots (wavefront.cpp:488-497):
 * keeps record s iff d_used[s] != 0, in slot order.  Records are
 * record_words x 32-bit (2 for slot records, 18 for a 72-byte PathState).
 * Writes the kept count to d_count (device) and, if h_count != NULL, to the host. */
NRRS_API int nrrs_gpu_compact(nrrs_gpu_ctx *ctx, const void *d_in, const uint8_t *d_used, uint32_t count,
                     uint32_t record_words, void *d_out, uint32_t *d_count, uint32_t *h_count);

/* Same, with the record count read on the device: count = min(*d_count_in, max_count)
 * (e.g. the stage's realized total, so spawned = min(total, capacity) never
 * round-trips through the host).  Launches max_count/tile CTAs. */
NRRS_API int nrrs_gpu_compact_dev(nrrs_gpu_ctx *ctx, const void *d_in, const uint8_t *d_used,
                                  const uint64_t *d_count_in, uint32_t max_count, uint32_t record_words,
                                  void *d_out, uint32_t *d_count);

/* ---- granular drop-ins for the reference's free functions (device data) ---- */
/* normalize_factors (rrs.hpp:18, rrs.cpp:8-24): in place; EINVAL on negative/non-finite (q untouched) */
NRRS_API int nrrs_gpu_normalize_factors(nrrs_gpu_ctx *ctx, float *d_q, uint64_t n, uint64_t n_pixels,
                               double *h_f_norm);
/* realize_counts (rrs.hpp:45-46, rrs.cpp:35-45): EINVAL where stochastic_round throws */
NRRS_API int nrrs_gpu_realize_counts(nrrs_gpu_ctx *ctx, const float *d_q, const float *d_u, int32_t *d_counts,
                            uint64_t n, uint64_t *h_total);
/* plan_spawns (wavefront.hpp:132, wavefront.cpp:141-154): EINVAL on a negative count */
NRRS_API int nrrs_gpu_plan_spawns(nrrs_gpu_ctx *ctx, const int32_t *d_counts, uint64_t n, uint32_t capacity,
                         uint32_t *d_offset, uint32_t *h_spawned, uint64_t *h_dropped);
/* strategy_factor (wavefront.hpp:161-163) batched, no sanitize/normalize: d_q[j] = raw factor */
NRRS_API int nrrs_gpu_strategy_factor(nrrs_gpu_ctx *ctx, const nrrs_vertex_soa *d_v, uint64_t n,
                             const nrrs_strategy *s, float eps_div, float *d_q);
/* NeuralRrs::predict_stats (networks.hpp:133) batched: d_stats[6j..6j+5] = mean(3), m2(3) */
NRRS_API int nrrs_gpu_predict_stats(nrrs_gpu_ctx *ctx, const nrrs_vertex_soa *d_v, uint64_t n, float *d_stats);
/* HashGrid::encode (hashgrid.cpp:38-82) of the AID RRSNet grid, batched and level-major: the K-A0
 * kernel the AID stage runs first (one level per CTA from shared memory, fp16 tables).
 * d_planes[l * plane_stride + j] = (feature 0, feature 1) of level l for point d_p01[3j..3j+2].
 * ESTATE unless AID weights with fp16 tables that fit in shared memory are installed. */
NRRS_API int nrrs_gpu_encode_levels(nrrs_gpu_ctx *ctx, const float *d_p01, uint64_t n, float *d_planes,
                                    uint64_t plane_stride);

/* ---- host helpers (pure arithmetic, no device) ---- */
NRRS_API uint32_t nrrs_queue_capacity_for(uint32_t n_pixels); /* wavefront.cpp:82-84 */
/* RngStream(seed, seq).next_float() x n, mapped to [lo, hi): used by the host
 * mirror to reproduce NeuralRrs' initializers (rng.hpp:33-62). */
NRRS_API void nrrs_rng_fill(uint64_t seed, uint64_t seq, float *h_out, uint64_t n, float lo, float hi);
/* root_path_key / child_path_key (rng.hpp:70-76) */
NRRS_API uint64_t nrrs_root_path_key(uint32_t pixel, uint32_t frame);
NRRS_API uint64_t nrrs_child_path_key(uint64_t parent_key, uint32_t child_index);

#ifdef __cplusplus
}
#endif
#endif /* NRRS_GPU_H */
