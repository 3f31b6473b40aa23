/*
 * nrrs_oracle.h -- CPU ORACLE for the NRRS per-bounce RRS stage.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference's
 * algorithm (/root/reference/proj, arXiv 2510.07868) used as the parity checker
 * for the CUDA path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  The product library
 * (paper_2510_07868_b200/libnrrs_gpu.so) never links or calls it.
 *
 * Parity pin: every function cites the reference file:line it restates.  The
 * reference itself does not build here (Eigen3 / doctest / CLI11 are absent,
 * SURVEY.md section 8c); rng.hpp is Eigen-free and is compiled verbatim into
 * oracle/_ref/ to pin the RNG, and the integer decision path is pinned by the
 * reference's own known-answer tests (tests/golden/reference_kats.json).
 */
#ifndef NRRS_ORACLE_H
#define NRRS_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:8-82 ------------------------------------------------------- */
typedef struct { uint64_t state, inc; } orc_rng;
uint64_t orc_mix_bits(uint64_t x);
uint64_t orc_mix_bits2(uint64_t a, uint64_t b);
void orc_rng_init(orc_rng *r, uint64_t seed, uint64_t sequence);
uint32_t orc_rng_next_u32(orc_rng *r);
float orc_rng_next_float(orc_rng *r);
uint64_t orc_child_path_key(uint64_t parent_key, uint32_t child_index);
uint64_t orc_root_path_key(uint32_t pixel, uint32_t frame);
void orc_path_stream(orc_rng *r, uint64_t seed, uint64_t path_key, uint32_t depth, uint64_t purpose);
/* u = path_stream(seed, key, depth, Draw::RrsRound).next_float()  (wavefront.cpp:397-399) */
float orc_rrs_uniform(uint64_t seed, uint64_t path_key, uint32_t depth);
void orc_fill_uniform(uint64_t seed, uint64_t sequence, float *out, size_t n, float lo, float hi);

/* ---- encodings.hpp:21-88, core.hpp:24-26 -------------------------------- */
float orc_luminance(const float c[3]);
int orc_stochastic_round(float q, float u); /* returns -1 where the reference throws */
void orc_one_blob(float x, int bins, float *out);
float orc_box_cox(float x); /* lambda = 0.5 */
float orc_roughness_remap(float a);
float orc_softplus_mod(float x);
float orc_softplus_mod_inverse_pos(float y);
uint64_t orc_box_cox_clamps(void);
void orc_reset_box_cox_clamps(void);

/* ---- hashgrid.hpp:13-22, hashgrid.cpp:10-82 ----------------------------- */
typedef struct {
    int levels, features, base_resolution, log2_table_size;
} orc_grid_spec;
size_t orc_grid_param_count(const orc_grid_spec *s);
void orc_grid_init(const orc_grid_spec *s, float *theta, uint64_t seed, uint64_t seq);
void orc_grid_encode(const orc_grid_spec *s, const float *theta, const float p01[3], float *out);

/* ---- mlp.hpp:12-18, mlp.cpp:7-72 (hidden 32, 3 hidden layers, leaky 0.01) */
int orc_mlp_param_count(int in, int out);
int orc_mlp_head_offset(int in, int out);
void orc_mlp_init(int in, int out, float *theta, uint64_t seed, uint64_t seq);
void orc_mlp_forward(int in, int out, const float *theta, const float *x, float *y);

/* ---- networks.cpp: snapshot inference ----------------------------------- */
enum { ORC_VARIANT_NRRS = 0, ORC_VARIANT_AID = 1 };
typedef struct {
    int variant;
    orc_grid_spec grid;
    const float *stat_grid; /* snapshot StatNet grid theta */
    const float *stat_mlp;  /* snapshot StatNet MLP theta (in = L*F+16, out = 6) */
    const float *rrs_grid;  /* snapshot RRS grid theta (AID only) */
    const float *rrs_mlp;   /* snapshot RRSNet MLP theta (in = 11 or L*F+16, out = 1) */
} orc_nets;
int orc_stat_input_dim(const orc_nets *n);
int orc_rrs_input_dim(const orc_nets *n);
void orc_build_stat_tail(const float wo01[2], float roughness, float *out);
void orc_build_nrrs_input(const float mean[3], const float m2[3], const float t_x[3],
                          const float i_pixel[3], float roughness, float *out);
void orc_build_aid_tail(const float wo01[2], const float t_x[3], const float i_pixel[3],
                        float roughness, float *out);
void orc_predict_stats(const orc_nets *n, const float p01[3], const float wo01[2], float roughness,
                       float stats[6]);
float orc_predict_q(const orc_nets *n, const float p01[3], const float wo01[2], float roughness,
                    const float t_x[3], const float i_pixel[3]);

/* ---- rrs.hpp / rrs.cpp --------------------------------------------------- */
enum {
    ORC_FIXED = 0, ORC_THROUGHPUT = 1, ORC_ADRRS_TREE = 2, ORC_ADRRS_NN = 3, ORC_NRRS = 4,
    ORC_AID_NRRS = 5
};
float orc_adrrs_factor(const float w[3], const float lo_hat[3], const float i_pixel[3], float eps_div);
float orc_strategy_factor(int kind, float fixed_value, const orc_nets *nets, const float w[3],
                          const float p01[3], const float wo01[2], float roughness,
                          const float i_pixel[3], float eps_div);
/* returns F_norm; *err = 1 where the reference throws */
double orc_normalize_factors(float *q, size_t n, uint64_t n_pixels, int *err);
uint64_t orc_realize_counts(const float *q, const float *u, int *counts, size_t n, int *err);
double orc_bernstein_bound(double f_rate, uint64_t n_pixels);
uint32_t orc_queue_capacity_for(uint32_t n_pixels);
/* plan_spawns (wavefront.cpp:141-154) */
void orc_plan_spawns(const int *counts, size_t n, uint32_t capacity, uint32_t *offset,
                     uint32_t *spawned, uint64_t *dropped, int *err);

/* ---- the RRS decision block of trace_frame (wavefront.cpp:363-411, 413-425, 488-497) ---- */
typedef struct {
    const float *p01;      /* [3n] */
    const float *wo01;     /* [2n] */
    const float *roughness;/* [n]  */
    const float *weight;   /* [3n] path weight w (= t_x) */
    const float *i_pixel;  /* [3n] film.i_acc[pixel] gathered per vertex */
    const uint64_t *path_key; /* [n] */
} orc_vertices;

typedef struct {
    uint32_t depth, n_pixels, capacity;
    int kind;
    float fixed_value;
    float gain;        /* rc.gain() evaluated by the caller; applied iff depth>=2 && adaptive */
    float eps_div;
    uint64_t seed;
    int threads;       /* factor pass threads (reference: parallel_for_blocks) */
} orc_stage_params;

typedef struct {
    float *q_orig;   /* [n] raw sanitized factor */
    float *q_norm;   /* [n] */
    float *q_real;   /* [n] */
    float *u;        /* [n] */
    int *k;          /* [n] */
    uint32_t *offset;/* [n] */
    uint8_t *decided;/* [n] */
    uint32_t *slots; /* [2*capacity] (parent j, child c) in slot order */
    double f_norm;
    double sum_q;
    uint64_t total;
    uint32_t spawned;
    uint64_t dropped;
    uint64_t nonfinite;
} orc_stage_out;

void orc_rrs_stage(const orc_vertices *v, size_t n, const orc_stage_params *p, const orc_nets *nets,
                   orc_stage_out *out);
/* order-preserving compaction (wavefront.cpp:488-497) of 2-word slot records */
uint32_t orc_compact_slots(const uint32_t *slots, const uint8_t *used, uint32_t count, uint32_t *out);

/* ---- suffix side of trace_frame ---- */
/* dst[key[i]] += term[i] (f64 x3) in item order, negative keys skipped: the frame / parent
 * folds (wavefront.cpp:299-319, :355, :485) and one depth of the reverse pass (:505-507). */
void orc_fold_ordered(double *dst, const int32_t *keys, const double *terms, size_t n);
/* TrainSample (networks.hpp:20-32), 80 bytes */
typedef struct {
    float position[3], omega_o[2], roughness, t_x[3], i_pixel[3], lo_sample[3], q_norm, q_real;
    uint32_t pixel;
    float k_i;
    uint16_t depth, pad;
} orc_train_sample;
/* one depth of the emission loop (wavefront.cpp:512-537); returns the records written */
size_t orc_emit_train(uint32_t depth, size_t n, const float *p01, const float *wo01, const float *rough,
                      const float *weight, const uint32_t *pixel, const float *q_norm, const float *q_real,
                      const uint8_t *decided, const double *s, const float *i_acc, orc_train_sample *out,
                      uint64_t *nonfinite);
/* k_i = per-pixel count over out[start, end) (wavefront.cpp:539-543) */
void orc_train_k_i(orc_train_sample *s, size_t start, size_t end, uint32_t n_pixels);
/* Film::add_frame / roll_acc (wavefront.cpp:104-116) */
void orc_film_add_frame(double *sum, uint32_t *samples, float *i_cur, const double *frame, size_t n_pixels);
void orc_film_roll_acc(float *i_acc, const float *i_cur, size_t n_pixels);

/* ---- StatNet training step ---- */
/* RelL2 (networks.cpp:110-114) */
void orc_relative_l2(float pred, float target, float eps, float *value, float *d_pred);
/* NeuralRrs::stat_loss_impl (networks.cpp:349-391): batch-mean relative L2 of the 6 stats
 * against (lo, lo^2); with g_mlp / g_grid non-NULL also the gradients (scaled by d_scale),
 * through Mlp::backward (mlp.cpp:74-111) and HashGrid::encode_backward (hashgrid.cpp:84-103). */
double orc_stat_loss(const orc_grid_spec *g, const float *stat_grid, const float *stat_mlp,
                     const orc_train_sample *batch, size_t n, float eps, float d_scale,
                     float *g_mlp, float *g_grid);
/* PixelError (networks.hpp:86-92) and the RRSNet loss parts (networks.hpp:219-224) */
typedef struct { float e, inv_denom; } orc_pixel_error;
typedef struct { double min, avg, rrs, total; uint32_t skipped; } orc_rrs_parts;
/* NeuralRrs::rrs_loss_impl (networks.cpp:418-460): snapshot stats from (snap_stat_grid,
 * snap_stat_mlp), RRSNet on the live (rrs_grid, rrs_mlp) of `variant`; phase 0 = Warmup,
 * 1 = Full.  Gradients (scaled by d_scale) into g_mlp / g_grid when non-NULL. */
void orc_rrs_loss(int variant, const orc_grid_spec *g, const float *snap_stat_grid, const float *snap_stat_mlp,
                  const float *rrs_grid, const float *rrs_mlp, const orc_train_sample *batch, size_t n,
                  const orc_pixel_error *errors, size_t n_errors, float e_avg, int phase, float gamma_min,
                  float gamma_avg, float gamma_rrs, float eps, float d_scale, float *g_mlp, float *g_grid,
                  orc_rrs_parts *parts);
/* Adam::step (optimizer.hpp:21-32) with the step counter already incremented to t */
void orc_adam_step(float *theta, const float *grad, float *m, float *v, size_t n, int64_t t, float lr,
                   float beta1, float beta2, float eps);
/* EmaTracker::update (optimizer.hpp:54-61) */
void orc_ema_update(float *shadow, const float *theta, size_t n, float decay);

/* ---- render front-end (first part) ---- */
/* Camera::generate_ray (scene.cpp:10-21) */
void orc_camera_ray(const float pos[3], const float look_at[3], const float up[3], float vfov_deg, float u, float v,
                    float aspect, float o[3], float d[3]);
/* path_stream(seed, key, depth, purpose) first two next_float() (rng.hpp:78-82) */
void orc_path_floats2(uint64_t seed, uint64_t key, uint32_t depth, uint64_t purpose, float *a, float *b);
/* intersect_triangle over every triangle in index order (geometry.cpp:46-70, Bvh::intersect_brute_force) */
void orc_intersect_brute(const float *pos, const uint32_t *idx, uint32_t n_tri, const float o[3], const float d[3],
                         float t_max, float *t, uint32_t *tri, float *u, float *v);
/* trace_frame's depth-1 front end (wavefront.cpp:253-268, :282-345): camera rays with jitter, closest hit
 * (brute force), dispatch (:125-138: 0 miss, 1 light, 2 surface) and the surface fields
 * (Scene::interaction scene.cpp:50-64, normalize_position :93-96, dir_to_spherical01 core.hpp:52-58). */
typedef struct {
    const float *pos; const uint32_t *idx; const uint32_t *mat_of_tri; uint32_t n_vert, n_tri;
    const int32_t *mat_kind; const float *mat_albedo; const float *mat_roughness; const float *mat_emission;
    float cam_pos[3], cam_look[3], cam_up[3], vfov;
} orc_scene;
void orc_render_depth1(const orc_scene *s, uint32_t width, uint32_t height, uint64_t seed, uint32_t frame,
                       float *ray_o, float *ray_d, float *hit_t, uint32_t *hit_tri, uint8_t *cls, float *p01,
                       float *wo01, float *roughness, uint64_t *path_key);

/* ---- trace_frame: wavefront.cpp:217-551 sequentially, brute-force hits ---- */
typedef struct {
    float o[3], d[3], t_max, w[3];
    uint64_t key;
    float prev_pdf, rrs;
    uint32_t pixel;
    int32_t parent;
    uint16_t depth, pad16;
    uint32_t pad;
} orc_path_state; /* PathState (wavefront.hpp:17-26), 72 bytes */
typedef struct { int kind; float fixed_value; } orc_strategy;
typedef struct { float f_rate, alpha, eps; int enabled; uint64_t overflow_events; } orc_rate_control;
typedef struct {
    uint32_t width, height;
    int max_depth;
    uint32_t capacity;        /* 0 = queue_capacity_for(W*H) */
    uint64_t seed;
    uint32_t frame_index;
    float adrrs_eps_scale;    /* TraceConfig (wavefront.hpp:128-140) */
    int collect_training;
    float env[3];             /* Scene::env_emission */
} orc_trace_cfg;
typedef struct {
    uint64_t camera_rays, scatter_rays, shadow_rays, nonfinite_drops, overflow_events, bias_drop_events,
        train_samples;
    uint32_t depth_counts[32];
} orc_frame_report;
/* One frame into frame[3*npx] (f64, zero on entry) and normals[3*npx]; i_acc is Film::i_acc.
 * Appends TrainSamples to train[*n_train..train_cap).  Returns 0, or -1 where the reference throws. */
int orc_trace_frame(const orc_scene *s, const orc_trace_cfg *cfg, const orc_strategy *assignment,
                    const orc_nets *nets, orc_rate_control *rc, const float *i_acc, double *frame, float *normals,
                    orc_train_sample *train, size_t train_cap, size_t *n_train, orc_frame_report *rep);
/* bsdf_sample (bsdf.cpp:85-133) for one material: kind, albedo, roughness */
int orc_bsdf_sample(int kind, const float albedo[3], float roughness, const float n[3], const float wo[3], float u1,
                    float u2, float wi[3], float *pdf, float thr[3]);

/* ---- synthetic inputs (generator follows test_networks.cpp:37-51) ---- */
void orc_gen_vertices(size_t n, uint32_t n_pixels, uint32_t frame, float *p01, float *wo01,
                      float *rough, float *t_x, float *i_pixel, uint64_t *path_key,
                      uint32_t *pixel);
void orc_gen_split_bound_factors(size_t n, float *q); /* RngStream(0xACC02, i).next_float()*4 */
/* NeuralRrs constructor init (networks.cpp:159-197) followed by the benchmark's
 * randomization (test_networks.cpp:407-410 style heads, RRSNet head bias
 * softplus_inv(2), grid *= 1e4). randomize = 0 gives the fresh constructor state. */
void orc_init_nets(int variant, const orc_grid_spec *g, uint64_t seed, int randomize,
                   float *stat_grid, float *stat_mlp, float *rrs_grid, float *rrs_mlp);

#ifdef __cplusplus
}
#endif
#endif
