/*
 * nrrs_oracle.c -- CPU ORACLE (test infrastructure only; see nrrs_oracle.h).
 *
 * A line-by-line restatement of the reference's NRRS decision path in plain C.
 * Build flags must keep IEEE semantics: -O2 -ffp-contract=off -fno-fast-math
 * (the reference's Release build on x86-64 does not contract a*b+c).
 * Citations are relative to /root/reference/proj.
 */
#include "nrrs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

/* ======================= rng.hpp ======================================== */

/* rng.hpp:8-13 SplitMix64 finalizer */
uint64_t orc_mix_bits(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* rng.hpp:15-17 */
uint64_t orc_mix_bits2(uint64_t a, uint64_t b) { return orc_mix_bits(a ^ orc_mix_bits(b)); }

/* rng.hpp:43-56 PCG32 step */
uint32_t orc_rng_next_u32(orc_rng *r) {
    const uint64_t old = r->state;
    r->state = old * 6364136223846793005ull + r->inc;
    const uint32_t xorshifted = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    const uint32_t rot = (uint32_t)(old >> 59u);
    return (xorshifted >> rot) | (xorshifted << ((32u - rot) & 31u));
}

/* rng.hpp:37-41 constructor */
void orc_rng_init(orc_rng *r, uint64_t seed, uint64_t sequence) {
    r->inc = (sequence << 1u) | 1u;
    r->state = 0u;
    orc_rng_next_u32(r);
    r->state += orc_mix_bits(seed);
    orc_rng_next_u32(r);
}

/* rng.hpp:59-61 */
float orc_rng_next_float(orc_rng *r) { return (float)(orc_rng_next_u32(r) >> 8) * 0x1p-24f; }

/* rng.hpp:70-72 */
uint64_t orc_child_path_key(uint64_t parent_key, uint32_t child_index) {
    return orc_mix_bits2(parent_key, 0xc2b2ae3d27d4eb4full + child_index);
}

/* rng.hpp:74-76 */
uint64_t orc_root_path_key(uint32_t pixel, uint32_t frame) {
    return orc_mix_bits(((uint64_t)frame << 32) | pixel);
}

/* rng.hpp:78-82 */
void orc_path_stream(orc_rng *r, uint64_t seed, uint64_t path_key, uint32_t depth, uint64_t purpose) {
    const uint64_t seq = orc_mix_bits2(path_key, ((uint64_t)depth << 8) ^ purpose);
    orc_rng_init(r, seed, seq);
}

/* wavefront.cpp:397-399, Draw::RrsRound = 0x55 (rng.hpp:27) */
float orc_rrs_uniform(uint64_t seed, uint64_t path_key, uint32_t depth) {
    orc_rng r;
    orc_path_stream(&r, seed, path_key, depth, 0x55);
    return orc_rng_next_float(&r);
}

void orc_fill_uniform(uint64_t seed, uint64_t sequence, float *out, size_t n, float lo, float hi) {
    orc_rng r;
    orc_rng_init(&r, seed, sequence);
    for (size_t i = 0; i < n; ++i)
        out[i] = lo + (hi - lo) * orc_rng_next_float(&r);
}

/* ======================= core.hpp / encodings.hpp ======================= */

/* core.hpp:24-26 */
float orc_luminance(const float c[3]) { return 0.2126f * c[0] + 0.7152f * c[1] + 0.0722f * c[2]; }

static _Atomic uint64_t g_box_cox_clamps;
uint64_t orc_box_cox_clamps(void) { return atomic_load(&g_box_cox_clamps); }
void orc_reset_box_cox_clamps(void) { atomic_store(&g_box_cox_clamps, 0); }

/* encodings.hpp:21-27 */
int orc_stochastic_round(float q, float u) {
    if (!(q >= 0.0f) || !isfinite(q))
        return -1;
    const float fl = floorf(q);
    const float r = q - fl;
    return (int)fl + (u < r ? 1 : 0);
}

/* encodings.hpp:31-44 */
void orc_one_blob(float x, int bins, float *out) {
    const float sigma = 1.0f / (float)bins;
    const float inv_two_sigma2 = 1.0f / (2.0f * sigma * sigma);
    float sum = 0.0f;
    for (int i = 0; i < bins; ++i) {
        const float c = ((float)i + 0.5f) / (float)bins;
        const float d = x - c;
        out[i] = expf(-d * d * inv_two_sigma2);
        sum += out[i];
    }
    const float inv = 1.0f / sum;
    for (int i = 0; i < bins; ++i)
        out[i] *= inv;
}

/* encodings.hpp:54-62, lambda = 0.5 */
float orc_box_cox(float x) {
    if (x < 0.0f) {
        atomic_fetch_add(&g_box_cox_clamps, 1);
        x = 0.0f;
    }
    return (powf(x, 0.5f) - 1.0f) / 0.5f;
}

/* encodings.hpp:65-67 */
float orc_roughness_remap(float a) { return 1.0f - expf(-a); }

/* encodings.hpp:71-75 */
float orc_softplus_mod(float x) {
    if (x < 0.0f)
        return log1pf(expf(x));
    return 0.5f * x + 0.6931471805599453f;
}

/* encodings.hpp:85-88 */
float orc_softplus_mod_inverse_pos(float y) { return 2.0f * (y - 0.6931471805599453f); }

/* ======================= hashgrid.cpp ==================================== */

static const uint32_t kPrimeY = 2654435761u; /* hashgrid.cpp:10-11 */
static const uint32_t kPrimeZ = 805459861u;

size_t orc_grid_param_count(const orc_grid_spec *s) {
    return (size_t)s->levels * ((size_t)1 << s->log2_table_size) * (size_t)s->features;
}

/* hashgrid.cpp:25-28 */
void orc_grid_init(const orc_grid_spec *s, float *theta, uint64_t seed, uint64_t seq) {
    orc_rng r;
    orc_rng_init(&r, seed, seq);
    const size_t n = orc_grid_param_count(s);
    for (size_t i = 0; i < n; ++i)
        theta[i] = (orc_rng_next_float(&r) * 2.0f - 1.0f) * 1e-4f;
}

/* hashgrid.cpp:30-36 */
static uint32_t grid_vertex_index(const orc_grid_spec *s, int level, uint32_t x, uint32_t y, uint32_t z) {
    const uint64_t res = (uint64_t)(s->base_resolution << level);
    const uint32_t table = 1u << s->log2_table_size;
    if ((res + 1) * (res + 1) * (res + 1) <= table) { /* dense level, hashgrid.cpp:16-22 */
        const uint32_t n = (uint32_t)res + 1;
        return (x * n + y) * n + z;
    }
    return (x ^ (y * kPrimeY) ^ (z * kPrimeZ)) & (table - 1);
}

static float clamp01(float v) { return v < 0.0f ? 0.0f : (1.0f < v ? 1.0f : v); }

/* hashgrid.cpp:38-82 (one point) */
void orc_grid_encode(const orc_grid_spec *s, const float *theta, const float p01[3], float *out) {
    const int F = s->features, L = s->levels;
    const uint32_t stride = (1u << s->log2_table_size) * (uint32_t)F;
    for (int l = 0; l < L; ++l) {
        const int res = s->base_resolution << l;
        const float fx = clamp01(p01[0]) * (float)res;
        const float fy = clamp01(p01[1]) * (float)res;
        const float fz = clamp01(p01[2]) * (float)res;
        uint32_t cx = (uint32_t)fx, cy = (uint32_t)fy, cz = (uint32_t)fz;
        if (cx > (uint32_t)(res - 1)) cx = (uint32_t)(res - 1);
        if (cy > (uint32_t)(res - 1)) cy = (uint32_t)(res - 1);
        if (cz > (uint32_t)(res - 1)) cz = (uint32_t)(res - 1);
        const float tx = fx - (float)cx, ty = fy - (float)cy, tz = fz - (float)cz;
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        for (int c = 0; c < 8; ++c) {
            const uint32_t ox = (c & 1), oy = (c >> 1) & 1, oz = (c >> 2) & 1;
            const float w = (ox ? tx : 1.0f - tx) * (oy ? ty : 1.0f - ty) * (oz ? tz : 1.0f - tz);
            const uint32_t idx = grid_vertex_index(s, l, cx + ox, cy + oy, cz + oz);
            const uint32_t base = (uint32_t)l * stride + idx * (uint32_t)F;
            for (int f = 0; f < F; ++f)
                acc[f] += w * theta[base + f];
        }
        for (int f = 0; f < F; ++f)
            out[l * F + f] = acc[f];
    }
}

/* ======================= mlp.cpp ========================================= */
#define HID 32
#define HLAYERS 3

static int layer_in(int in, int l) { return l == 0 ? in : HID; }
static int layer_out(int out, int l) { return l == HLAYERS ? out : HID; }

/* mlp.cpp:7-16 */
static int layer_offset(int in, int out, int layer) {
    int off = 0;
    for (int l = 0; l < layer; ++l)
        off += layer_out(out, l) * layer_in(in, l) + layer_out(out, l);
    return off;
}
int orc_mlp_param_count(int in, int out) { return layer_offset(in, out, HLAYERS + 1); }
int orc_mlp_head_offset(int in, int out) { return layer_offset(in, out, HLAYERS); }

/* mlp.cpp:34-44: He-uniform hidden layers (column-major W), zero head */
void orc_mlp_init(int in, int out, float *theta, uint64_t seed, uint64_t seq) {
    orc_rng r;
    orc_rng_init(&r, seed, seq);
    memset(theta, 0, sizeof(float) * (size_t)orc_mlp_param_count(in, out));
    for (int l = 0; l < HLAYERS; ++l) {
        const int li = layer_in(in, l), lo = layer_out(out, l);
        const float bound = sqrtf(6.0f / (float)li);
        float *w = theta + layer_offset(in, out, l);
        for (int c = 0; c < li; ++c)
            for (int rr = 0; rr < lo; ++rr)
                w[c * lo + rr] = (orc_rng_next_float(&r) * 2.0f - 1.0f) * bound;
    }
}

/* mlp.cpp:52-72: z = W a + b ; a = max(z, slope z) ; head linear */
void orc_mlp_forward(int in, int out, const float *theta, const float *x, float *y) {
    float a[64], z[64];
    const float slope = 0.01f;
    for (int i = 0; i < in; ++i)
        a[i] = x[i];
    for (int l = 0; l <= HLAYERS; ++l) {
        const int li = layer_in(in, l), lo = layer_out(out, l);
        const float *w = theta + layer_offset(in, out, l);
        const float *b = w + lo * li;
        for (int r = 0; r < lo; ++r) {
            float s = 0.0f;
            for (int c = 0; c < li; ++c)
                s += w[c * lo + r] * a[c];
            z[r] = s + b[r];
        }
        if (l < HLAYERS) {
            for (int r = 0; r < lo; ++r) {
                const float zs = z[r] * slope;
                a[r] = z[r] < zs ? zs : z[r]; /* cwiseMax(z, z*slope) */
            }
        } else {
            for (int r = 0; r < lo; ++r)
                y[r] = z[r];
        }
    }
}

/* ======================= networks.cpp ==================================== */

int orc_stat_input_dim(const orc_nets *n) { return n->grid.levels * n->grid.features + 16; }
int orc_rrs_input_dim(const orc_nets *n) {
    return n->variant == ORC_VARIANT_NRRS ? 11 : n->grid.levels * n->grid.features + 16;
}

/* Eigen Vector3f::mean(): redux x + (y + z), then / 3 */
static float mean3(const float v[3]) { return (v[0] + (v[1] + v[2])) / 3.0f; }

/* networks.cpp:131-135 */
void orc_build_stat_tail(const float wo01[2], float roughness, float *out) {
    orc_one_blob(wo01[0], 4, out);
    orc_one_blob(wo01[1], 4, out + 4);
    orc_one_blob(orc_roughness_remap(roughness), 8, out + 8);
}

/* networks.cpp:137-147 */
void orc_build_nrrs_input(const float mean[3], const float m2[3], const float t_x[3],
                          const float i_pixel[3], float roughness, float *out) {
    for (int c = 0; c < 3; ++c)
        out[c] = orc_box_cox(mean[c]);
    for (int c = 0; c < 3; ++c)
        out[3 + c] = orc_box_cox(m2[c]);
    for (int c = 0; c < 3; ++c)
        out[6 + c] = orc_box_cox(t_x[c]);
    out[9] = orc_box_cox(mean3(i_pixel));
    out[10] = orc_roughness_remap(roughness);
}

/* networks.cpp:149-157 */
void orc_build_aid_tail(const float wo01[2], const float t_x[3], const float i_pixel[3],
                        float roughness, float *out) {
    orc_one_blob(wo01[0], 4, out);
    orc_one_blob(wo01[1], 4, out + 4);
    for (int c = 0; c < 3; ++c)
        out[8 + c] = orc_box_cox(t_x[c]);
    out[11] = orc_box_cox(mean3(i_pixel));
    orc_one_blob(orc_roughness_remap(roughness), 4, out + 12);
}

/* networks.cpp:206-224 + 252-264: StatNet on the snapshot */
void orc_predict_stats(const orc_nets *n, const float p01[3], const float wo01[2], float roughness,
                       float stats[6]) {
    float x[64];
    const int gd = n->grid.levels * n->grid.features;
    orc_grid_encode(&n->grid, n->stat_grid, p01, x);
    orc_build_stat_tail(wo01, roughness, x + gd);
    orc_mlp_forward(gd + 16, 6, n->stat_mlp, x, stats);
}

/* networks.cpp:266-281.  AID also runs StatNet and discards the result
 * (networks.cpp:276); its only side effect is nothing (StatNet has no
 * box_cox), so the restatement skips it. */
float orc_predict_q(const orc_nets *n, const float p01[3], const float wo01[2], float roughness,
                    const float t_x[3], const float i_pixel[3]) {
    float x[64], y[8];
    if (n->variant == ORC_VARIANT_NRRS) {
        float st[6];
        orc_predict_stats(n, p01, wo01, roughness, st);
        orc_build_nrrs_input(st, st + 3, t_x, i_pixel, roughness, x);
        orc_mlp_forward(11, 1, n->rrs_mlp, x, y);
    } else {
        const int gd = n->grid.levels * n->grid.features;
        orc_grid_encode(&n->grid, n->rrs_grid, p01, x);
        orc_build_aid_tail(wo01, t_x, i_pixel, roughness, x + gd);
        orc_mlp_forward(gd + 16, 1, n->rrs_mlp, x, y);
    }
    return orc_softplus_mod(y[0]);
}

/* ======================= rrs.hpp / rrs.cpp ============================== */

static float fmin_std(float a, float b) { return (b < a) ? b : a; } /* std::min(a,b) */

/* rrs.hpp:56-61 */
float orc_adrrs_factor(const float w[3], const float lo_hat[3], const float i_pixel[3], float eps_div) {
    const float prod[3] = {w[0] * lo_hat[0], w[1] * lo_hat[1], w[2] * lo_hat[2]};
    const float num = orc_luminance(prod);
    const float q = num / (orc_luminance(i_pixel) + eps_div);
    return q < 0.05f ? 0.05f : (20.0f < q ? 20.0f : q); /* std::clamp */
}

/* wavefront.cpp:186-215 (AdrrsTree is out of scope: returns NaN, sanitized to 0) */
float orc_strategy_factor(int kind, float fixed_value, const orc_nets *nets, const float w[3],
                          const float p01[3], const float wo01[2], float roughness,
                          const float i_pixel[3], float eps_div) {
    const float eps = (eps_div < 1e-8f) ? 1e-8f : eps_div; /* std::max(eps_div, 1e-8f) */
    switch (kind) {
    case ORC_FIXED:
        return fixed_value;
    case ORC_THROUGHPUT:
        return fmin_std(1.0f, orc_luminance(w)); /* rrs.hpp:49-51 */
    case ORC_ADRRS_NN: {
        float st[6];
        orc_predict_stats(nets, p01, wo01, roughness, st);
        return orc_adrrs_factor(w, st, i_pixel, eps);
    }
    case ORC_NRRS:
    case ORC_AID_NRRS:
        return orc_predict_q(nets, p01, wo01, roughness, w, i_pixel);
    default:
        return NAN;
    }
}

/* rrs.cpp:8-24 */
double orc_normalize_factors(float *q, size_t n, uint64_t n_pixels, int *err) {
    double sum = 0.0;
    *err = 0;
    for (size_t i = 0; i < n; ++i) {
        if (!(q[i] >= 0.0f) || !isfinite(q[i])) {
            *err = 1;
            return 0.0;
        }
        sum += q[i];
    }
    if (sum <= 0.0)
        return 1.0;
    const double f_norm = (double)n_pixels / sum;
    if (f_norm < 1.0) {
        const float s = (float)f_norm;
        for (size_t i = 0; i < n; ++i)
            q[i] *= s;
    }
    return f_norm;
}

/* rrs.cpp:26-33 */
double orc_bernstein_bound(double f_rate, uint64_t n_pixels) {
    if (f_rate >= 1.0)
        return 1.0;
    const double gap = 1.0 - f_rate;
    const double exponent = gap * gap * (double)n_pixels / (2.0 * f_rate + (2.0 / 3.0) * gap);
    return exp(-exponent);
}

/* rrs.cpp:35-45 */
uint64_t orc_realize_counts(const float *q, const float *u, int *counts, size_t n, int *err) {
    uint64_t total = 0;
    *err = 0;
    for (size_t i = 0; i < n; ++i) {
        counts[i] = orc_stochastic_round(q[i], u[i]);
        if (counts[i] < 0) {
            *err = 1;
            return 0;
        }
        total += (uint64_t)counts[i];
    }
    return total;
}

/* wavefront.cpp:82-84 */
uint32_t orc_queue_capacity_for(uint32_t n_pixels) { return n_pixels + (n_pixels + 7u) / 8u; }

/* wavefront.cpp:141-154 */
void orc_plan_spawns(const int *counts, size_t n, uint32_t capacity, uint32_t *offset,
                     uint32_t *spawned, uint64_t *dropped, int *err) {
    uint64_t cum = 0;
    *err = 0;
    for (size_t i = 0; i < n; ++i) {
        if (counts[i] < 0) {
            *err = 1;
            return;
        }
        offset[i] = (uint32_t)(cum < capacity ? cum : capacity);
        cum += (uint64_t)counts[i];
    }
    *spawned = (uint32_t)(cum < capacity ? cum : capacity);
    *dropped = cum - *spawned;
}

/* ======================= trace_frame RRS block ========================== */

typedef struct {
    const orc_vertices *v;
    const orc_stage_params *p;
    const orc_nets *nets;
    orc_stage_out *out;
    size_t n;
    _Atomic size_t next_block;
    _Atomic uint64_t nonfinite;
} factor_job;

/* wavefront.cpp:368-389 body, one parallel_for_blocks block (parallel.hpp:28-63) */
static void factor_block(factor_job *job, size_t begin, size_t end) {
    const orc_vertices *v = job->v;
    const orc_stage_params *p = job->p;
    uint64_t nonfinite = 0;
    for (size_t j = begin; j < end; ++j) {
        float q = 0.0f;
        int decided = 0;
        const float *w = v->weight + 3 * j;
        if (p->depth == 1) {
            q = 1.0f;
            decided = 1;
        } else if (orc_luminance(w) > 0.0f) {
            q = orc_strategy_factor(p->kind, p->fixed_value, job->nets, w, v->p01 + 3 * j,
                                    v->wo01 + 2 * j, v->roughness[j], v->i_pixel + 3 * j, p->eps_div);
            decided = 1;
        }
        if (!isfinite(q) || q < 0.0f) {
            q = 0.0f;
            decided = 0;
            ++nonfinite;
        }
        if (job->out->decided)
            job->out->decided[j] = (uint8_t)decided;
        job->out->q_orig[j] = q;
    }
    atomic_fetch_add(&job->nonfinite, nonfinite);
}

static void *factor_worker(void *arg) {
    factor_job *job = (factor_job *)arg;
    const size_t block = 4096; /* parallel.hpp kParallelBlock */
    for (;;) {
        const size_t b = atomic_fetch_add(&job->next_block, 1);
        const size_t begin = b * block;
        if (begin >= job->n)
            return NULL;
        factor_block(job, begin, begin + block < job->n ? begin + block : job->n);
    }
}

void orc_rrs_stage(const orc_vertices *v, size_t n, const orc_stage_params *p, const orc_nets *nets,
                   orc_stage_out *out) {
    /* factor pass: parallel_for_blocks over ns surface vertices (wavefront.cpp:368-389) */
    factor_job job;
    job.v = v;
    job.p = p;
    job.nets = nets;
    job.out = out;
    job.n = n;
    atomic_init(&job.next_block, 0);
    atomic_init(&job.nonfinite, 0);
    int threads = p->threads < 1 ? 1 : p->threads;
    if (threads > 256)
        threads = 256;
    pthread_t pool[256];
    int spawned_threads = 0;
    for (int t = 1; t < threads; ++t)
        if (pthread_create(&pool[spawned_threads], NULL, factor_worker, &job) == 0)
            ++spawned_threads;
    factor_worker(&job);
    for (int t = 0; t < spawned_threads; ++t)
        pthread_join(pool[t], NULL);
    out->nonfinite = atomic_load(&job.nonfinite);

    /* serial part: normalize (:390), gain (:391), RNG + q_real (:393-402), realize (:403-404),
     * plan (:406) */
    memcpy(out->q_norm, out->q_orig, n * sizeof(float));
    double sum = 0.0;
    for (size_t j = 0; j < n; ++j)
        sum += out->q_norm[j];
    out->sum_q = sum;
    int err = 0;
    out->f_norm = orc_normalize_factors(out->q_norm, n, p->n_pixels, &err);
    const int adaptive = p->kind != ORC_FIXED;
    const float gain = (p->depth >= 2 && adaptive) ? p->gain : 1.0f;
    uint64_t total = 0;
    for (size_t j = 0; j < n; ++j) {
        out->q_real[j] = out->q_norm[j] * gain;
        out->u[j] = orc_rrs_uniform(p->seed, v->path_key[j], p->depth);
        out->k[j] = orc_stochastic_round(out->q_real[j], out->u[j]);
        total += (uint64_t)out->k[j];
    }
    out->total = total;
    orc_plan_spawns(out->k, n, p->capacity, out->offset, &out->spawned, &out->dropped, &err);
    /* child slot layout (wavefront.cpp:421-425, :436): slot off+c <- (j, c) */
    if (out->slots) {
        for (size_t j = 0; j < n; ++j) {
            const uint32_t off = out->offset[j];
            const uint32_t rem = out->spawned - (out->spawned < off ? out->spawned : off);
            const uint32_t kept = (uint32_t)out->k[j] < rem ? (uint32_t)out->k[j] : rem;
            for (uint32_t c = 0; c < kept; ++c) {
                out->slots[2 * (size_t)(off + c)] = (uint32_t)j;
                out->slots[2 * (size_t)(off + c) + 1] = c;
            }
        }
    }
}

/* wavefront.cpp:488-497 */
uint32_t orc_compact_slots(const uint32_t *slots, const uint8_t *used, uint32_t count, uint32_t *out) {
    uint32_t write = 0;
    for (uint32_t s = 0; s < count; ++s) {
        if (!used[s])
            continue;
        out[2 * (size_t)write] = slots[2 * (size_t)s];
        out[2 * (size_t)write + 1] = slots[2 * (size_t)s + 1];
        ++write;
    }
    return write;
}

/* ======================= synthetic inputs =============================== */

/* vertex i draws from RngStream(0xC0FFEE, i) in the order of
 * test_networks.cpp:37-51 (position, omega_o, roughness, t_x, i_pixel),
 * each vector component drawn left to right. */
/* ---- StatNet training step (networks.cpp:349-391, mlp.cpp:74-111, hashgrid.cpp:84-103,
 * optimizer.hpp) ---- */

void orc_relative_l2(float pred, float target, float eps, float *value, float *d_pred) {
    const float d = pred - target;
    const float inv = 1.0f / (target * target + eps);
    *value = d * d * inv;
    *d_pred = 2.0f * d * inv;
}

/* Mlp::forward keeping the workspace (pre / post activations of the hidden layers) */
static void mlp_forward_ws(int in, int out, const float *theta, const float *x, float pre[HLAYERS][HID],
                           float post[HLAYERS][HID], float *y) {
    const float slope = 0.01f;
    const float *a = x;
    for (int l = 0; l <= HLAYERS; ++l) {
        const int li = layer_in(in, l), lo = layer_out(out, l);
        const float *w = theta + layer_offset(in, out, l);
        const float *b = w + lo * li;
        float z[HID];
        for (int r = 0; r < lo; ++r) {
            float s = 0.0f;
            for (int c2 = 0; c2 < li; ++c2)
                s += w[c2 * lo + r] * a[c2];
            z[r] = s + b[r];
        }
        if (l < HLAYERS) {
            for (int r = 0; r < lo; ++r) {
                pre[l][r] = z[r];
                const float zs = z[r] * slope;
                post[l][r] = z[r] < zs ? zs : z[r];
            }
            a = post[l];
        } else {
            for (int r = 0; r < lo; ++r)
                y[r] = z[r];
        }
    }
}

/* Mlp::backward for one sample, accumulating into grad (mlp.cpp:74-111) */
static void mlp_backward_1(int in, int out, const float *theta, const float *x, float pre[HLAYERS][HID],
                           float post[HLAYERS][HID], const float *d_y, float *grad, float *d_x) {
    const float slope = 0.01f;
    float delta[HID], d_a[HID];
    for (int r = 0; r < out; ++r)
        delta[r] = d_y[r];
    int lo = out;
    for (int l = HLAYERS; l >= 0; --l) {
        const int li = layer_in(in, l);
        const float *w = theta + layer_offset(in, out, l);
        float *gw = grad + layer_offset(in, out, l);
        float *gb = gw + lo * li;
        const float *below = l == 0 ? x : post[l - 1];
        for (int c2 = 0; c2 < li; ++c2)
            for (int r = 0; r < lo; ++r)
                gw[c2 * lo + r] += delta[r] * below[c2];
        for (int r = 0; r < lo; ++r)
            gb[r] += delta[r];
        for (int c2 = 0; c2 < li; ++c2) {  /* d_a = W^T delta */
            float s = 0.0f;
            for (int r = 0; r < lo; ++r)
                s += w[c2 * lo + r] * delta[r];
            d_a[c2] = s;
        }
        if (l == 0) {
            for (int c2 = 0; c2 < li; ++c2)
                d_x[c2] = d_a[c2];
        } else {
            for (int r = 0; r < HID; ++r)  /* leaky-ReLU derivative on the stored pre-activation */
                delta[r] = pre[l - 1][r] <= 0.0f ? d_a[r] * slope : d_a[r];
            lo = HID;
        }
    }
}

double orc_stat_loss(const orc_grid_spec *g, const float *stat_grid, const float *stat_mlp,
                     const orc_train_sample *batch, size_t n, float eps, float d_scale,
                     float *g_mlp, float *g_grid) {
    const int F = g->features, L = g->levels, gd = L * F, in = gd + 16;
    const uint32_t stride = (1u << g->log2_table_size) * (uint32_t)F;
    if (g_mlp)
        memset(g_mlp, 0, sizeof(float) * (size_t)orc_mlp_param_count(in, 6));
    if (g_grid)
        memset(g_grid, 0, sizeof(float) * orc_grid_param_count(g));
    if (n == 0)
        return 0.0;
    const float inv_n = 1.0f / (float)n;
    double loss = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const orc_train_sample *s = batch + i;
        float x[64], pre[HLAYERS][HID], post[HLAYERS][HID], y[6];
        orc_grid_encode(g, stat_grid, s->position, x);
        orc_build_stat_tail(s->omega_o, s->roughness, x + gd);
        mlp_forward_ws(in, 6, stat_mlp, x, pre, post, y);
        float d_y[6];
        for (int c2 = 0; c2 < 3; ++c2) {
            float vm, dm, v2, d2;
            orc_relative_l2(y[c2], s->lo_sample[c2], eps, &vm, &dm);
            orc_relative_l2(y[3 + c2], s->lo_sample[c2] * s->lo_sample[c2], eps, &v2, &d2);
            loss += (double)vm + (double)v2;
            d_y[c2] = dm * inv_n * d_scale;
            d_y[3 + c2] = d2 * inv_n * d_scale;
        }
        if (!g_mlp)
            continue;
        float d_x[64];
        mlp_backward_1(in, 6, stat_mlp, x, pre, post, d_y, g_mlp, d_x);
        for (int l = 0; l < L; ++l) {  /* HashGrid::encode_backward: grad[base + f] += w * d_out */
            const int res = g->base_resolution << l;
            const float fx = clamp01(s->position[0]) * (float)res, fy = clamp01(s->position[1]) * (float)res,
                        fz = clamp01(s->position[2]) * (float)res;
            uint32_t cx = (uint32_t)fx, cy = (uint32_t)fy, cz = (uint32_t)fz;
            if (cx > (uint32_t)(res - 1)) cx = (uint32_t)(res - 1);
            if (cy > (uint32_t)(res - 1)) cy = (uint32_t)(res - 1);
            if (cz > (uint32_t)(res - 1)) cz = (uint32_t)(res - 1);
            const float tx = fx - (float)cx, ty = fy - (float)cy, tz = fz - (float)cz;
            for (int c2 = 0; c2 < 8; ++c2) {
                const uint32_t ox = (c2 & 1), oy = (c2 >> 1) & 1, oz = (c2 >> 2) & 1;
                const float w = (ox ? tx : 1.0f - tx) * (oy ? ty : 1.0f - ty) * (oz ? tz : 1.0f - tz);
                const uint32_t base = (uint32_t)l * stride + grid_vertex_index(g, l, cx + ox, cy + oy, cz + oz) * (uint32_t)F;
                for (int f = 0; f < F; ++f)
                    g_grid[base + f] += w * d_x[l * F + f];
            }
        }
    }
    return loss * (double)inv_n;
}

/* grad_pixelvar_wrt_rr / _split (networks.cpp:116-130) */
static float grad_pixelvar_wrt_rr(const float weight[3], const float h_sample[3], float p_rr) {
    const float w = orc_luminance(weight), h = orc_luminance(h_sample);
    return -(w * w) * (h * h) / (p_rr * p_rr);
}
static float grad_pixelvar_wrt_split(const float weight[3], float h_variance_lum, float n_s) {
    const float w = orc_luminance(weight);
    return -(w * w) * h_variance_lum / (n_s * n_s);
}
/* encodings.hpp:77-83 */
static float softplus_mod_grad(float x) {
    if (x < 0.0f) {
        const float e = expf(x);
        return e / (1.0f + e);
    }
    return 0.5f;
}

void orc_rrs_loss(int variant, const orc_grid_spec *g, const float *snap_stat_grid, const float *snap_stat_mlp,
                  const float *rrs_grid, const float *rrs_mlp, const orc_train_sample *batch, size_t n,
                  const orc_pixel_error *errors, size_t n_errors, float e_avg, int phase, float gamma_min,
                  float gamma_avg, float gamma_rrs, float eps, float d_scale, float *g_mlp, float *g_grid,
                  orc_rrs_parts *parts) {
    const int F = g->features, L = g->levels, gd = L * F;
    const int in = variant == ORC_VARIANT_NRRS ? 11 : gd + 16;
    const uint32_t stride = (1u << g->log2_table_size) * (uint32_t)F;
    memset(parts, 0, sizeof *parts);
    if (g_mlp)
        memset(g_mlp, 0, sizeof(float) * (size_t)orc_mlp_param_count(in, 1));
    if (g_grid && variant == ORC_VARIANT_AID)
        memset(g_grid, 0, sizeof(float) * orc_grid_param_count(g));
    if (n == 0)
        return;
    const float inv_n = 1.0f / (float)n;
    for (size_t i = 0; i < n; ++i) {
        const orc_train_sample *s = batch + i;
        /* snapshot_stats_batch (networks.cpp:219-224) */
        float xs[64], stats[6];
        orc_grid_encode(g, snap_stat_grid, s->position, xs);
        orc_build_stat_tail(s->omega_o, s->roughness, xs + gd);
        orc_mlp_forward(gd + 16, 6, snap_stat_mlp, xs, stats);
        /* encode_rrs_inputs (networks.cpp:226-250) */
        float x[64];
        if (variant == ORC_VARIANT_NRRS) {
            orc_build_nrrs_input(stats, stats + 3, s->t_x, s->i_pixel, s->roughness, x);
        } else {
            orc_grid_encode(g, rrs_grid, s->position, x);
            orc_build_aid_tail(s->omega_o, s->t_x, s->i_pixel, s->roughness, x + gd);
        }
        float pre[HLAYERS][HID], post[HLAYERS][HID], y[1];
        mlp_forward_ws(in, 1, rrs_mlp, x, pre, post, y);
        const float z = y[0], q = orc_softplus_mod(z);
        float d_q = 0.0f;
        if (phase == 0) {
            float v, d;
            orc_relative_l2(q, 1.0f, eps, &v, &d);
            parts->rrs += v;
            d_q = d * inv_n;
        } else {
            const size_t px = s->pixel;
            const float inv_k = s->k_i > 0.0f ? 1.0f / s->k_i : 1.0f;
            if (px < n_errors) {
                const orc_pixel_error *pe = errors + px;
                float gvar = 0.0f;
                if (s->q_real < 1.0f) {
                    if (s->q_real > 0.0f)
                        gvar = grad_pixelvar_wrt_rr(s->t_x, s->lo_sample, s->q_real);
                } else {
                    float var[3];
                    for (int c2 = 0; c2 < 3; ++c2) {
                        const float vv = stats[3 + c2] - stats[c2] * stats[c2];
                        var[c2] = vv < 0.0f ? 0.0f : vv;  /* cwiseMax(0) */
                    }
                    gvar = grad_pixelvar_wrt_split(s->t_x, orc_luminance(var), s->q_real);
                }
                const float de_dq = pe->inv_denom * gvar * inv_k;
                parts->min += pe->e * inv_k;
                const float dev = pe->e - e_avg;
                parts->avg += dev * dev * inv_k;
                d_q += (gamma_min * de_dq + gamma_avg * 2.0f * dev * de_dq) * inv_n;
            } else {
                ++parts->skipped;
            }
            const float dq_gap = q - s->q_norm;
            parts->rrs += dq_gap * dq_gap;
            d_q += gamma_rrs * 2.0f * dq_gap * inv_n;
        }
        if (!g_mlp)
            continue;
        const float dy = d_q * softplus_mod_grad(z) * d_scale;
        float d_x[64];
        mlp_backward_1(in, 1, rrs_mlp, x, pre, post, &dy, g_mlp, d_x);
        if (variant == ORC_VARIANT_AID && g_grid) {
            for (int l = 0; l < L; ++l) {
                const int res = g->base_resolution << l;
                const float fx = clamp01(s->position[0]) * (float)res, fy = clamp01(s->position[1]) * (float)res,
                            fz = clamp01(s->position[2]) * (float)res;
                uint32_t cx = (uint32_t)fx, cy = (uint32_t)fy, cz = (uint32_t)fz;
                if (cx > (uint32_t)(res - 1)) cx = (uint32_t)(res - 1);
                if (cy > (uint32_t)(res - 1)) cy = (uint32_t)(res - 1);
                if (cz > (uint32_t)(res - 1)) cz = (uint32_t)(res - 1);
                const float tx = fx - (float)cx, ty = fy - (float)cy, tz = fz - (float)cz;
                for (int c2 = 0; c2 < 8; ++c2) {
                    const uint32_t ox = (c2 & 1), oy = (c2 >> 1) & 1, oz = (c2 >> 2) & 1;
                    const float w = (ox ? tx : 1.0f - tx) * (oy ? ty : 1.0f - ty) * (oz ? tz : 1.0f - tz);
                    const uint32_t base = (uint32_t)l * stride +
                                          grid_vertex_index(g, l, cx + ox, cy + oy, cz + oz) * (uint32_t)F;
                    for (int f = 0; f < F; ++f)
                        g_grid[base + f] += w * d_x[l * F + f];
                }
            }
        }
    }
    parts->min *= (double)inv_n;
    parts->avg *= (double)inv_n;
    parts->rrs *= (double)inv_n;
    parts->total = phase == 0 ? parts->rrs
                              : (double)gamma_min * parts->min + (double)gamma_avg * parts->avg +
                                    (double)gamma_rrs * parts->rrs;
}

void orc_adam_step(float *theta, const float *grad, float *m, float *v, size_t n, int64_t t, float lr,
                   float beta1, float beta2, float eps) {
    const float c1 = 1.0f / (1.0f - powf(beta1, (float)t));
    const float c2 = 1.0f / (1.0f - powf(beta2, (float)t));
    for (size_t i = 0; i < n; ++i) {
        m[i] = beta1 * m[i] + (1.0f - beta1) * grad[i];
        v[i] = beta2 * v[i] + (1.0f - beta2) * (grad[i] * grad[i]);
        theta[i] -= lr * (m[i] * c1) / (sqrtf(v[i] * c2) + eps);
    }
}

void orc_ema_update(float *shadow, const float *theta, size_t n, float decay) {
    for (size_t i = 0; i < n; ++i)
        shadow[i] = decay * shadow[i] + (1.0f - decay) * theta[i];
}

/* ---- render front-end (first part) ---- */

static void v3_sub(const float a[3], const float b[3], float r[3]) { r[0] = a[0] - b[0]; r[1] = a[1] - b[1]; r[2] = a[2] - b[2]; }
static float v3_dot(const float a[3], const float b[3]) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }
static void v3_cross(const float a[3], const float b[3], float r[3]) {
    const float x = a[1] * b[2] - a[2] * b[1], y = a[2] * b[0] - a[0] * b[2], z = a[0] * b[1] - a[1] * b[0];
    r[0] = x; r[1] = y; r[2] = z;
}
static void v3_normalize(float v[3]) {  /* Eigen normalized(): v / sqrt(squaredNorm) if > 0 */
    const float sq = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
    if (sq > 0.0f) {
        const float n = sqrtf(sq);
        v[0] = v[0] / n; v[1] = v[1] / n; v[2] = v[2] / n;
    }
}

void orc_camera_ray(const float pos[3], const float look_at[3], const float up[3], float vfov_deg, float u, float v,
                    float aspect, float o[3], float d[3]) {
    float fwd[3], right[3], cup[3];
    v3_sub(look_at, pos, fwd);
    v3_normalize(fwd);
    v3_cross(fwd, up, right);
    v3_normalize(right);
    v3_cross(right, fwd, cup);
    const float tan_half = tanf(0.5f * vfov_deg * 3.14159265358979323846f / 180.0f);
    const float px = (2.0f * u - 1.0f) * tan_half * aspect;
    const float py = (1.0f - 2.0f * v) * tan_half;
    for (int a = 0; a < 3; ++a) {
        o[a] = pos[a];
        d[a] = (fwd[a] + px * right[a]) + py * cup[a];
    }
    v3_normalize(d);
}

void orc_path_floats2(uint64_t seed, uint64_t key, uint32_t depth, uint64_t purpose, float *a, float *b) {
    orc_rng r;
    orc_rng_init(&r, seed, orc_mix_bits2(key, ((uint64_t)depth << 8) ^ purpose));
    *a = orc_rng_next_float(&r);
    *b = orc_rng_next_float(&r);
}

/* geometry.cpp:46-70 */
static int tri_hit(const float *pos, const uint32_t *idx, uint32_t tri, const float o[3], const float d[3],
                   float t_min, float t_max, float *t, float *u, float *v) {
    const float *p0 = pos + 3 * idx[3 * tri], *p1 = pos + 3 * idx[3 * tri + 1], *p2 = pos + 3 * idx[3 * tri + 2];
    float e1[3], e2[3], pv[3], tv[3], qv[3];
    v3_sub(p1, p0, e1);
    v3_sub(p2, p0, e2);
    v3_cross(d, e2, pv);
    const float det = v3_dot(e1, pv);
    if (fabsf(det) < 1e-12f)
        return 0;
    const float inv_det = 1.0f / det;
    v3_sub(o, p0, tv);
    const float uu = v3_dot(tv, pv) * inv_det;
    if (uu < 0.0f || uu > 1.0f)
        return 0;
    v3_cross(tv, e1, qv);
    const float vv = v3_dot(d, qv) * inv_det;
    if (vv < 0.0f || uu + vv > 1.0f)
        return 0;
    const float tt = v3_dot(e2, qv) * inv_det;
    if (tt <= t_min || tt >= *t || tt >= t_max)
        return 0;
    *t = tt; *u = uu; *v = vv;
    return 1;
}

void orc_intersect_brute(const float *pos, const uint32_t *idx, uint32_t n_tri, const float o[3], const float d[3],
                         float t_max, float *t, uint32_t *tri, float *u, float *v) {
    *t = INFINITY; *tri = 0xFFFFFFFFu; *u = 0.0f; *v = 0.0f;
    for (uint32_t k = 0; k < n_tri; ++k)
        if (tri_hit(pos, idx, k, o, d, 1e-4f, t_max, t, u, v))
            *tri = k;
}

void orc_render_depth1(const orc_scene *s, uint32_t width, uint32_t height, uint64_t seed, uint32_t frame,
                       float *ray_o, float *ray_d, float *hit_t, uint32_t *hit_tri, uint8_t *cls, float *p01,
                       float *wo01, float *roughness, uint64_t *path_key) {
    /* Scene::finalize normalization (scene.cpp:23-37) */
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (uint32_t i = 0; i < s->n_vert; ++i)
        for (int a = 0; a < 3; ++a) {
            lo[a] = s->pos[3 * i + a] < lo[a] ? s->pos[3 * i + a] : lo[a];
            hi[a] = s->pos[3 * i + a] > hi[a] ? s->pos[3 * i + a] : hi[a];
        }
    float span = 0.0f;
    for (int a = 0; a < 3; ++a)
        span = (hi[a] - lo[a]) > span ? (hi[a] - lo[a]) : span;
    if (span < 1e-6f)
        span = 1e-6f;
    const float scale = 1.0f / (span * 1.02f);
    float off[3];
    for (int a = 0; a < 3; ++a)
        off[a] = lo[a] - span * 0.01f;
    const float aspect = (float)width / (float)height;
    for (uint32_t p = 0; p < width * height; ++p) {
        const uint64_t key = orc_root_path_key(p, frame);
        path_key[p] = key;
        float j0, j1;
        orc_path_floats2(seed, key, 1, 0x11, &j0, &j1);  /* Draw::CameraJitter */
        const float u = ((float)(p % width) + j0) / (float)width;
        const float v = ((float)(p / width) + j1) / (float)height;
        float *o = ray_o + 3 * p, *d = ray_d + 3 * p;
        orc_camera_ray(s->cam_pos, s->cam_look, s->cam_up, s->vfov, u, v, aspect, o, d);
        float t, uu, vv;
        uint32_t tri;
        orc_intersect_brute(s->pos, s->idx, s->n_tri, o, d, INFINITY, &t, &tri, &uu, &vv);
        hit_t[p] = t;
        hit_tri[p] = tri;
        p01[3 * p] = p01[3 * p + 1] = p01[3 * p + 2] = 0.0f;
        wo01[2 * p] = wo01[2 * p + 1] = 0.0f;
        roughness[p] = 0.0f;
        if (tri == 0xFFFFFFFFu) {
            cls[p] = 0;
            continue;
        }
        const uint32_t m = s->mat_of_tri[tri];
        const float *alb = s->mat_albedo + 3 * m;
        const float amax = alb[0] > alb[1] ? (alb[0] > alb[2] ? alb[0] : alb[2]) : (alb[1] > alb[2] ? alb[1] : alb[2]);
        const int scattering = s->mat_kind[m] == 1 || amax > 0.0f;
        cls[p] = scattering ? 2 : 1;
        if (!scattering)
            continue;
        float pt[3], wo[3];
        for (int a = 0; a < 3; ++a) {
            pt[a] = o[a] + t * d[a];
            wo[a] = -d[a];
        }
        for (int a = 0; a < 3; ++a) {
            float q = (pt[a] - off[a]) * scale;
            q = q < 0.0f ? 0.0f : q;
            p01[3 * p + a] = q > 1.0f ? 1.0f : q;
        }
        const float z = wo[2] < -1.0f ? -1.0f : (wo[2] > 1.0f ? 1.0f : wo[2]);
        const float theta = acosf(z);
        float phi = atan2f(wo[1], wo[0]);
        if (phi < 0.0f)
            phi += 2.0f * 3.14159265358979323846f;
        wo01[2 * p] = theta * 0.31830988618379067154f;
        wo01[2 * p + 1] = phi * (0.5f * 0.31830988618379067154f);
        roughness[p] = s->mat_kind[m] == 1 ? s->mat_roughness[m] : 1.0f;
    }
}

/* ---- suffix side of trace_frame ---- */

/* wavefront.cpp:299 / :317 / :355 / :485 (frame[pixel] += term), :301 / :319
 * (parent.s += term), :505-507 (verts[d-1][v.parent].s += v.s): sequential f64. */
void orc_fold_ordered(double *dst, const int32_t *keys, const double *terms, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        if (keys[i] < 0)
            continue;
        for (int c = 0; c < 3; ++c)
            dst[3 * (size_t)keys[i] + c] += terms[3 * i + c];
    }
}

/* wavefront.cpp:512-537: decided vertices with finite lo = float(s / weight) */
size_t orc_emit_train(uint32_t depth, size_t n, const float *p01, const float *wo01, const float *rough,
                      const float *weight, const uint32_t *pixel, const float *q_norm, const float *q_real,
                      const uint8_t *decided, const double *s, const float *i_acc, orc_train_sample *out,
                      uint64_t *nonfinite) {
    size_t w = 0;
    for (size_t j = 0; j < n; ++j) {
        if (!decided[j])
            continue;
        float lo[3];
        for (int c = 0; c < 3; ++c)
            lo[c] = weight[3 * j + c] > 0.0f ? (float)(s[3 * j + c] / (double)weight[3 * j + c]) : 0.0f;
        if (!(isfinite(lo[0]) && isfinite(lo[1]) && isfinite(lo[2]))) {
            ++*nonfinite;
            continue;
        }
        orc_train_sample t;
        memset(&t, 0, sizeof t);
        for (int c = 0; c < 3; ++c) {
            t.position[c] = p01[3 * j + c];
            t.t_x[c] = weight[3 * j + c];
            t.i_pixel[c] = i_acc[3 * (size_t)pixel[j] + c];
            t.lo_sample[c] = lo[c];
        }
        t.omega_o[0] = wo01[2 * j];
        t.omega_o[1] = wo01[2 * j + 1];
        t.roughness = rough[j];
        t.q_norm = q_norm[j];
        t.q_real = q_real[j];
        t.pixel = pixel[j];
        t.k_i = 1.0f;
        t.depth = (uint16_t)depth;
        out[w++] = t;
    }
    return w;
}

/* wavefront.cpp:539-543 */
void orc_train_k_i(orc_train_sample *s, size_t start, size_t end, uint32_t n_pixels) {
    uint32_t *per_pixel = (uint32_t *)calloc(n_pixels ? n_pixels : 1, sizeof(uint32_t));
    for (size_t i = start; i < end; ++i)
        per_pixel[s[i].pixel] += 1u;
    for (size_t i = start; i < end; ++i)
        s[i].k_i = (float)per_pixel[s[i].pixel];
    free(per_pixel);
}

/* Film::add_frame (wavefront.cpp:104-111) */
void orc_film_add_frame(double *sum, uint32_t *samples, float *i_cur, const double *frame, size_t n_pixels) {
    for (size_t i = 0; i < n_pixels; ++i) {
        for (int c = 0; c < 3; ++c) {
            sum[3 * i + c] += frame[3 * i + c];
            i_cur[3 * i + c] = (float)frame[3 * i + c];
        }
        samples[i] += 1u;
    }
}

/* Film::roll_acc (wavefront.cpp:113-116) */
void orc_film_roll_acc(float *i_acc, const float *i_cur, size_t n_pixels) {
    for (size_t i = 0; i < 3 * n_pixels; ++i) {
        const float a = 0.5f * i_acc[i];
        const float b = 0.5f * i_cur[i];
        i_acc[i] = a + b;
    }
}

void orc_gen_vertices(size_t n, uint32_t n_pixels, uint32_t frame, float *p01, float *wo01,
                      float *rough, float *t_x, float *i_pixel, uint64_t *path_key,
                      uint32_t *pixel) {
    for (size_t i = 0; i < n; ++i) {
        orc_rng g;
        orc_rng_init(&g, 0xC0FFEEull, (uint64_t)i);
        for (int c = 0; c < 3; ++c) p01[3 * i + c] = orc_rng_next_float(&g);
        for (int c = 0; c < 2; ++c) wo01[2 * i + c] = orc_rng_next_float(&g);
        rough[i] = orc_rng_next_float(&g);
        for (int c = 0; c < 3; ++c) t_x[3 * i + c] = 0.2f + orc_rng_next_float(&g);
        for (int c = 0; c < 3; ++c) i_pixel[3 * i + c] = 0.5f + orc_rng_next_float(&g);
        const uint32_t px = (uint32_t)(i % (n_pixels ? n_pixels : 1));
        if (pixel) pixel[i] = px;
        path_key[i] = orc_root_path_key(px, frame);
    }
}

/* nrrs_cli.cpp:121-125 per-index convention with acceptance.cpp:99-102's seed */
void orc_gen_split_bound_factors(size_t n, float *q) {
    for (size_t i = 0; i < n; ++i) {
        orc_rng r;
        orc_rng_init(&r, 0xACC02ull, (uint64_t)i);
        q[i] = orc_rng_next_float(&r) * 4.0f;
    }
}

void orc_init_nets(int variant, const orc_grid_spec *g, uint64_t seed, int randomize,
                   float *stat_grid, float *stat_mlp, float *rrs_grid, float *rrs_mlp) {
    const int gd = g->levels * g->features;
    const int stat_in = gd + 16, rrs_in = variant == ORC_VARIANT_NRRS ? 11 : gd + 16;
    /* networks.cpp:177-190 */
    orc_grid_init(g, stat_grid, seed, 0);
    orc_mlp_init(stat_in, 6, stat_mlp, seed, 1);
    if (variant == ORC_VARIANT_AID)
        orc_grid_init(g, rrs_grid, seed, 2);
    orc_mlp_init(rrs_in, 1, rrs_mlp, seed, 3);
    const int rrs_head = orc_mlp_head_offset(rrs_in, 1);
    rrs_mlp[orc_mlp_param_count(rrs_in, 1) - 1] = orc_softplus_mod_inverse_pos(1.0f);
    if (!randomize)
        return;
    /* benchmark randomization: heads (w, b) ~ U(-0.5, 0.5) as in
     * test_networks.cpp:407-410, StatNet head bias 1 (mostly positive stats),
     * RRSNet head bias softplus_inv(2) (mean q ~ 2 so F < 1), grids x 1e4
     * (test_networks.cpp:337-339). */
    const int stat_head = orc_mlp_head_offset(stat_in, 6), stat_n = orc_mlp_param_count(stat_in, 6);
    orc_rng r;
    orc_rng_init(&r, seed, 100);
    for (int k = stat_head; k < stat_n; ++k)
        stat_mlp[k] = (orc_rng_next_float(&r) * 2.0f - 1.0f) * 0.5f;
    for (int k = stat_n - 6; k < stat_n; ++k)
        stat_mlp[k] = 1.0f;
    const int rrs_n = orc_mlp_param_count(rrs_in, 1);
    orc_rng_init(&r, seed, 101);
    for (int k = rrs_head; k < rrs_n; ++k)
        rrs_mlp[k] = (orc_rng_next_float(&r) * 2.0f - 1.0f) * 0.5f;
    rrs_mlp[rrs_n - 1] = orc_softplus_mod_inverse_pos(2.0f);
    const size_t gn = orc_grid_param_count(g);
    for (size_t i = 0; i < gn; ++i)
        stat_grid[i] *= 1e4f;
    if (variant == ORC_VARIANT_AID)
        for (size_t i = 0; i < gn; ++i)
            rrs_grid[i] *= 1e4f;
}

/* ---- trace_frame ---- */
#define ORC_PI 3.14159265358979323846f
#define ORC_INV_PI 0.31830988618379067154f

static void face_normal(const orc_scene *s, uint32_t tri, float n[3]) { /* geometry.cpp:22-28 */
    const float *p0 = s->pos + 3 * s->idx[3 * tri], *p1 = s->pos + 3 * s->idx[3 * tri + 1],
                *p2 = s->pos + 3 * s->idx[3 * tri + 2];
    float e1[3], e2[3], c[3];
    v3_sub(p1, p0, e1);
    v3_sub(p2, p0, e2);
    v3_cross(e1, e2, c);
    const float len = sqrtf(v3_dot(c, c));
    if (len > 0.0f) {
        n[0] = c[0] / len; n[1] = c[1] / len; n[2] = c[2] / len;
    } else {
        n[0] = 0.0f; n[1] = 0.0f; n[2] = 1.0f;
    }
}
static float tri_area(const orc_scene *s, uint32_t tri) { /* geometry.cpp:16-20 */
    const float *p0 = s->pos + 3 * s->idx[3 * tri], *p1 = s->pos + 3 * s->idx[3 * tri + 1],
                *p2 = s->pos + 3 * s->idx[3 * tri + 2];
    float e1[3], e2[3], c[3];
    v3_sub(p1, p0, e1);
    v3_sub(p2, p0, e2);
    v3_cross(e1, e2, c);
    return 0.5f * sqrtf(v3_dot(c, c));
}
static float fmaxf3(const float v[3]) { /* Eigen maxCoeff */
    float m = v[0];
    if (v[1] > m) m = v[1];
    if (v[2] > m) m = v[2];
    return m;
}
static float stdmaxf(float a, float b) { return a < b ? b : a; }
static float stdminf(float a, float b) { return b < a ? b : a; }

static float mis_power2(float a, float b) { /* wavefront.cpp:15-21 */
    const double a2 = (double)a * (double)a, b2 = (double)b * (double)b;
    if (a2 + b2 <= 0.0)
        return 0.0f;
    return (float)(a2 / (a2 + b2));
}
static void build_frame(const float n[3], float t[3], float b[3]) { /* core.hpp:43-50 */
    const float sign = copysignf(1.0f, n[2]);
    const float a = -1.0f / (sign + n[2]);
    const float c = n[0] * n[1] * a;
    t[0] = 1.0f + sign * n[0] * n[0] * a; t[1] = sign * c; t[2] = -sign * n[0];
    b[0] = c; b[1] = sign + n[1] * n[1] * a; b[2] = -n[1];
}
static void to_world(const float n[3], const float l[3], float w[3]) { /* bsdf.cpp:35-39 */
    float t[3], b[3];
    build_frame(n, t, b);
    for (int a = 0; a < 3; ++a)
        w[a] = (l[0] * t[a] + l[1] * b[a]) + l[2] * n[a];
}
static float ggx_d(float cos_h, float alpha) {
    if (cos_h <= 0.0f)
        return 0.0f;
    const float a2 = alpha * alpha;
    const float d = stdmaxf(cos_h * cos_h * (a2 - 1.0f) + 1.0f, 1e-12f);
    return a2 / (ORC_PI * d * d);
}
static float smith_g1(float cos_v, float alpha) {
    if (cos_v <= 0.0f)
        return 0.0f;
    const float a2 = alpha * alpha;
    return 2.0f * cos_v / (cos_v + sqrtf(a2 + (1.0f - a2) * cos_v * cos_v));
}
static void schlick(const float f0[3], float cos_i, float out[3]) {
    float m = 1.0f - cos_i;
    m = m < 0.0f ? 0.0f : (1.0f < m ? 1.0f : m); /* std::clamp */
    const float m2 = m * m;
    for (int a = 0; a < 3; ++a)
        out[a] = f0[a] + (1.0f - f0[a]) * (m2 * m2 * m);
}
static void half_vec(const float wo[3], const float wi[3], float h[3]) {
    for (int a = 0; a < 3; ++a)
        h[a] = wo[a] + wi[a];
    v3_normalize(h);
}
static void bsdf_eval(int kind, const float alb[3], float rough, const float n[3], const float wo[3],
                      const float wi[3], float f[3]) { /* bsdf.cpp:43-61 */
    f[0] = f[1] = f[2] = 0.0f;
    const float cos_o = v3_dot(n, wo), cos_i = v3_dot(n, wi);
    if (cos_o <= 0.0f || cos_i <= 0.0f)
        return;
    if (kind == 0) {
        for (int a = 0; a < 3; ++a)
            f[a] = alb[a] * ORC_INV_PI;
        return;
    }
    float h[3], fr[3];
    half_vec(wo, wi, h);
    const float alpha = stdmaxf(rough, 1e-3f);
    const float d = ggx_d(v3_dot(n, h), alpha);
    const float g = smith_g1(cos_o, alpha) * smith_g1(cos_i, alpha);
    schlick(alb, v3_dot(wo, h), fr);
    const float sc = d * g / (4.0f * cos_o * cos_i);
    for (int a = 0; a < 3; ++a)
        f[a] = fr[a] * sc;
}
static float bsdf_pdf(int kind, float rough, const float n[3], const float wo[3], const float wi[3]) {
    const float cos_o = v3_dot(n, wo), cos_i = v3_dot(n, wi); /* bsdf.cpp:63-83 */
    if (cos_o <= 0.0f || cos_i <= 0.0f)
        return 0.0f;
    if (kind == 0)
        return cos_i * ORC_INV_PI;
    float h[3];
    half_vec(wo, wi, h);
    const float cos_h = v3_dot(n, h);
    const float alpha = stdmaxf(rough, 1e-3f);
    const float d = ggx_d(cos_h, alpha);
    const float dot_oh = v3_dot(wo, h);
    if (dot_oh <= 0.0f)
        return 0.0f;
    return d * cos_h / (4.0f * dot_oh);
}

int orc_bsdf_sample(int kind, const float alb[3], float rough, const float n[3], const float wo[3], float u1,
                    float u2, float wi[3], float *pdf, float thr[3]) { /* bsdf.cpp:85-133 */
    const float cos_o = v3_dot(n, wo);
    if (cos_o <= 0.0f)
        return 0;
    if (kind == 0) {
        const float r = sqrtf(u1);
        const float phi = 2.0f * ORC_PI * u2;
        const float loc[3] = {r * cosf(phi), r * sinf(phi), sqrtf(stdmaxf(0.0f, 1.0f - u1))};
        to_world(n, loc, wi);
        const float cos_i = v3_dot(n, wi);
        if (cos_i <= 0.0f)
            return 0;
        *pdf = cos_i * ORC_INV_PI;
        thr[0] = alb[0]; thr[1] = alb[1]; thr[2] = alb[2];
        return 1;
    }
    const float alpha = stdmaxf(rough, 1e-3f);
    const float tan2 = alpha * alpha * u1 / stdmaxf(1.0f - u1, 1e-12f);
    const float cos_h = 1.0f / sqrtf(1.0f + tan2);
    const float sin_h = sqrtf(stdmaxf(0.0f, 1.0f - cos_h * cos_h));
    const float phi = 2.0f * ORC_PI * u2;
    const float loc[3] = {sin_h * cosf(phi), sin_h * sinf(phi), cos_h};
    float h[3], fr[3];
    to_world(n, loc, h);
    const float dot_oh = v3_dot(wo, h);
    if (dot_oh <= 0.0f)
        return 0;
    for (int a = 0; a < 3; ++a)
        wi[a] = 2.0f * dot_oh * h[a] - wo[a];
    const float cos_i = v3_dot(n, wi);
    if (cos_i <= 0.0f)
        return 0;
    const float nh = v3_dot(n, h);
    *pdf = ggx_d(nh, alpha) * nh / (4.0f * dot_oh);
    if (!(*pdf > 0.0f) || !isfinite(*pdf))
        return 0;
    const float g = smith_g1(cos_o, alpha) * smith_g1(cos_i, alpha);
    schlick(alb, dot_oh, fr);
    const float sc = g * dot_oh / (cos_o * nh);
    for (int a = 0; a < 3; ++a)
        thr[a] = fr[a] * sc;
    return 1;
}

static int occluded_brute(const orc_scene *s, const float o[3], const float d[3], float t_max) {
    for (uint32_t k = 0; k < s->n_tri; ++k) { /* Bvh::occluded: any hit in (kRayEps, t_max) */
        float t = t_max, u, v;
        if (tri_hit(s->pos, s->idx, k, o, d, 1e-4f, t_max, &t, &u, &v))
            return 1;
    }
    return 0;
}

typedef struct {
    uint32_t n;
    uint32_t *tris;
    float *areas;
    int32_t *index_of_tri;
} orc_lights;

static void light_pdf(const orc_lights *L, uint32_t tri, float *pdf) { /* scene.cpp:84-91 */
    const int32_t i = L->index_of_tri[tri];
    *pdf = i < 0 ? 0.0f : 1.0f / ((float)L->n * L->areas[i]);
}

static void hit_emission(const orc_scene *s, const orc_lights *L, const float d[3], uint32_t tri, float dist,
                         float prev_pdf, float out[3]) { /* wavefront.cpp:28-41 */
    const float *e = s->mat_emission + 3 * s->mat_of_tri[tri];
    out[0] = out[1] = out[2] = 0.0f;
    if (!(fmaxf3(e) > 0.0f))
        return;
    float mis = 1.0f;
    if (prev_pdf >= 0.0f) {
        float pdf_area;
        light_pdf(L, tri, &pdf_area);
        if (pdf_area > 0.0f) {
            float nl[3];
            face_normal(s, tri, nl);
            const float cos_l = fabsf(v3_dot(nl, d));
            const float pdf_sa = pdf_area * dist * dist / stdmaxf(cos_l, 1e-8f);
            mis = mis_power2(prev_pdf, pdf_sa);
        }
    }
    for (int a = 0; a < 3; ++a)
        out[a] = e[a] * mis;
}

typedef struct {
    float p[3], n_s[3], wo[3], weight[3], p01[3], wo01[2], roughness;
    uint32_t material, pixel;
    int32_t parent;
    uint64_t key;
    float rrs, q_norm, q_real;
    int decided;
    double emit[3], nee[3], s[3];
} orc_vrec;

int orc_trace_frame(const orc_scene *s, const orc_trace_cfg *cfg, const orc_strategy *assignment,
                    const orc_nets *nets, orc_rate_control *rc, const float *i_acc, double *frame, float *normals,
                    orc_train_sample *train, size_t train_cap, size_t *n_train, orc_frame_report *rep) {
    const int B = cfg->max_depth;
    if (B < 1 || B > 32)
        return -1;
    const uint32_t npx = cfg->width * cfg->height;
    if (npx == 0)
        return -1;
    const uint32_t cap = cfg->capacity ? cfg->capacity : orc_queue_capacity_for(npx);
    if (cap < npx)
        return -1;
    memset(rep, 0, sizeof *rep);
    /* Scene::finalize: lights + normalization (scene.cpp:23-48) */
    orc_lights L;
    L.n = 0;
    L.tris = (uint32_t *)malloc(sizeof(uint32_t) * (s->n_tri + 1));
    L.areas = (float *)malloc(sizeof(float) * (s->n_tri + 1));
    L.index_of_tri = (int32_t *)malloc(sizeof(int32_t) * (s->n_tri + 1));
    for (uint32_t t = 0; t < s->n_tri; ++t) {
        L.index_of_tri[t] = -1;
        const float a = tri_area(s, t);
        if (fmaxf3(s->mat_emission + 3 * s->mat_of_tri[t]) > 0.0f && a > 0.0f) {
            L.index_of_tri[t] = (int32_t)L.n;
            L.tris[L.n] = t;
            L.areas[L.n] = a;
            ++L.n;
        }
    }
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (uint32_t i = 0; i < s->n_vert; ++i)
        for (int a = 0; a < 3; ++a) {
            lo[a] = stdminf(lo[a], s->pos[3 * i + a]);
            hi[a] = stdmaxf(hi[a], s->pos[3 * i + a]);
        }
    if (s->n_vert == 0) {
        lo[0] = lo[1] = lo[2] = 0.0f;
        hi[0] = hi[1] = hi[2] = 1.0f;
    }
    float span = stdmaxf(stdmaxf(hi[0] - lo[0], hi[1] - lo[1]), hi[2] - lo[2]);
    span = stdmaxf(span, 1e-6f);
    const float nscale = 1.0f / (span * 1.02f);
    float noff[3];
    for (int a = 0; a < 3; ++a)
        noff[a] = lo[a] - span * 0.01f;

    double lum_acc = 0.0;
    for (uint32_t p = 0; p < npx; ++p)
        lum_acc += (double)orc_luminance(i_acc + 3 * p);
    const float eps_div = cfg->adrrs_eps_scale * (float)(lum_acc / (double)npx);

    orc_path_state *queue = (orc_path_state *)calloc(cap, sizeof(orc_path_state));
    orc_path_state *next = (orc_path_state *)calloc(cap, sizeof(orc_path_state));
    uint8_t *used = (uint8_t *)calloc(cap, 1);
    orc_vrec *verts[33] = {0};
    uint32_t nverts[33] = {0};
    float *hit_t = (float *)malloc(sizeof(float) * cap);
    uint32_t *hit_tri = (uint32_t *)malloc(sizeof(uint32_t) * cap);
    uint8_t *cls = (uint8_t *)malloc(cap);
    const float aspect = (float)cfg->width / (float)cfg->height;
    for (uint32_t p = 0; p < npx; ++p) { /* wavefront.cpp:253-268 */
        orc_path_state *q = &queue[p];
        memset(q, 0, sizeof *q);
        q->pixel = p;
        q->key = orc_root_path_key(p, cfg->frame_index);
        float j0, j1;
        orc_path_floats2(cfg->seed, q->key, 1, 0x11, &j0, &j1);
        const float u = ((float)(p % cfg->width) + j0) / (float)cfg->width;
        const float v = ((float)(p / cfg->width) + j1) / (float)cfg->height;
        orc_camera_ray(s->cam_pos, s->cam_look, s->cam_up, s->vfov, u, v, aspect, q->o, q->d);
        q->t_max = INFINITY;
        q->w[0] = q->w[1] = q->w[2] = 1.0f;
        q->prev_pdf = -1.0f;
        q->rrs = 1.0f;
        q->parent = -1;
        q->depth = 1;
    }
    uint32_t n = npx;
    rep->camera_rays = npx;
    memset(normals, 0, sizeof(float) * 3 * npx);
    int rc_err = 0;

    for (int depth = 1; depth <= B; ++depth) {
        if (n == 0)
            break;
        rep->depth_counts[depth - 1] = n;
        if (depth >= 2)
            rep->scatter_rays += n;
        for (uint32_t i = 0; i < n; ++i) {
            float u, v;
            orc_intersect_brute(s->pos, s->idx, s->n_tri, queue[i].o, queue[i].d, queue[i].t_max, &hit_t[i],
                                &hit_tri[i], &u, &v);
            if (hit_tri[i] == 0xFFFFFFFFu) {
                cls[i] = 0;
            } else {
                const uint32_t m = s->mat_of_tri[hit_tri[i]];
                const int scat = s->mat_kind[m] == 1 || fmaxf3(s->mat_albedo + 3 * m) > 0.0f;
                cls[i] = scat ? 2 : 1;
            }
        }
        orc_vrec *up = depth >= 2 ? verts[depth - 1] : NULL;
        for (uint32_t i = 0; i < n; ++i) { /* misses (:295-303) */
            if (cls[i] != 0 || !(fmaxf3(cfg->env) > 0.0f))
                continue;
            const orc_path_state *q = &queue[i];
            double term[3];
            for (int a = 0; a < 3; ++a)
                term[a] = (double)(q->w[a] * cfg->env[a]);
            for (int a = 0; a < 3; ++a)
                frame[3 * q->pixel + a] += term[a];
            if (up && q->parent >= 0)
                for (int a = 0; a < 3; ++a)
                    up[q->parent].s[a] += term[a];
        }
        for (uint32_t i = 0; i < n; ++i) { /* pure emitters (:305-321) */
            if (cls[i] != 1)
                continue;
            const orc_path_state *q = &queue[i];
            if (depth == 1) {
                float nl[3];
                face_normal(s, hit_tri[i], nl);
                if (v3_dot(nl, q->d) > 0.0f)
                    for (int a = 0; a < 3; ++a)
                        nl[a] = -nl[a];
                memcpy(normals + 3 * q->pixel, nl, sizeof nl);
            }
            float em[3];
            hit_emission(s, &L, q->d, hit_tri[i], hit_t[i], q->prev_pdf, em);
            if (fmaxf3(em) > 0.0f) {
                double term[3];
                for (int a = 0; a < 3; ++a)
                    term[a] = (double)(q->w[a] * em[a]);
                for (int a = 0; a < 3; ++a)
                    frame[3 * q->pixel + a] += term[a];
                if (up && q->parent >= 0)
                    for (int a = 0; a < 3; ++a)
                        up[q->parent].s[a] += term[a];
            }
        }
        uint32_t ns = 0;
        for (uint32_t i = 0; i < n; ++i)
            ns += cls[i] == 2;
        orc_vrec *vd = (orc_vrec *)calloc(ns ? ns : 1, sizeof(orc_vrec));
        verts[depth] = vd;
        nverts[depth] = ns;
        uint32_t j = 0;
        for (uint32_t i = 0; i < n; ++i) { /* surface vertices (:324-352) */
            if (cls[i] != 2)
                continue;
            const orc_path_state *q = &queue[i];
            orc_vrec *v = &vd[j++];
            const uint32_t tri = hit_tri[i];
            float ns_[3];
            face_normal(s, tri, ns_); /* shading_normal without per-vertex normals */
            for (int a = 0; a < 3; ++a) {
                v->p[a] = q->o[a] + hit_t[i] * q->d[a];
                v->wo[a] = -q->d[a];
            }
            if (v3_dot(ns_, v->wo) < 0.0f)
                for (int a = 0; a < 3; ++a)
                    ns_[a] = -ns_[a];
            memcpy(v->n_s, ns_, sizeof ns_);
            memcpy(v->weight, q->w, sizeof q->w);
            v->material = s->mat_of_tri[tri];
            v->pixel = q->pixel;
            v->parent = q->parent;
            v->key = q->key;
            v->rrs = q->rrs;
            v->q_norm = 1.0f;
            v->q_real = 1.0f;
            for (int a = 0; a < 3; ++a) {
                float qq = (v->p[a] - noff[a]) * nscale;
                qq = stdmaxf(qq, 0.0f);
                v->p01[a] = stdminf(qq, 1.0f);
            }
            const float z = v->wo[2] < -1.0f ? -1.0f : (v->wo[2] > 1.0f ? 1.0f : v->wo[2]);
            const float theta = acosf(z);
            float phi = atan2f(v->wo[1], v->wo[0]);
            if (phi < 0.0f)
                phi += 2.0f * ORC_PI;
            v->wo01[0] = theta * ORC_INV_PI;
            v->wo01[1] = phi * (0.5f * ORC_INV_PI);
            v->roughness = s->mat_kind[v->material] == 1 ? s->mat_roughness[v->material] : 1.0f;
            float em[3];
            hit_emission(s, &L, q->d, tri, hit_t[i], q->prev_pdf, em);
            if (fmaxf3(em) > 0.0f)
                for (int a = 0; a < 3; ++a)
                    v->emit[a] = (double)(q->w[a] * em[a]);
            if (depth == 1)
                memcpy(normals + 3 * q->pixel, v->n_s, sizeof v->n_s);
        }
        for (j = 0; j < ns; ++j)
            for (int a = 0; a < 3; ++a) {
                vd[j].s[a] = vd[j].emit[a];
                frame[3 * vd[j].pixel + a] += vd[j].emit[a];
            }
        if (depth == B)
            break;

        /* the RRS decision block (:363-425) */
        const orc_strategy st = assignment[depth - 1];
        float *p01 = (float *)malloc(sizeof(float) * 3 * (ns + 1)), *wo01 = (float *)malloc(sizeof(float) * 2 * (ns + 1));
        float *rough = (float *)malloc(sizeof(float) * (ns + 1)), *wgt = (float *)malloc(sizeof(float) * 3 * (ns + 1));
        float *ipx = (float *)malloc(sizeof(float) * 3 * (ns + 1));
        uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (ns + 1));
        for (j = 0; j < ns; ++j) {
            memcpy(p01 + 3 * j, vd[j].p01, 12);
            memcpy(wo01 + 2 * j, vd[j].wo01, 8);
            rough[j] = vd[j].roughness;
            memcpy(wgt + 3 * j, vd[j].weight, 12);
            memcpy(ipx + 3 * j, i_acc + 3 * vd[j].pixel, 12);
            keys[j] = vd[j].key;
        }
        orc_vertices ov = {p01, wo01, rough, wgt, ipx, keys};
        orc_stage_params sp;
        memset(&sp, 0, sizeof sp);
        sp.depth = (uint32_t)depth;
        sp.n_pixels = npx;
        sp.capacity = cap;
        sp.kind = st.kind;
        sp.fixed_value = st.fixed_value;
        sp.gain = rc->enabled ? rc->f_rate * rc->alpha : 1.0f;
        sp.eps_div = eps_div;
        sp.seed = cfg->seed;
        sp.threads = 1;
        orc_stage_out so;
        memset(&so, 0, sizeof so);
        const size_t nn = ns + 1;
        so.q_orig = (float *)malloc(sizeof(float) * nn);
        so.q_norm = (float *)malloc(sizeof(float) * nn);
        so.q_real = (float *)malloc(sizeof(float) * nn);
        so.u = (float *)malloc(sizeof(float) * nn);
        so.k = (int *)malloc(sizeof(int) * nn);
        so.offset = (uint32_t *)malloc(sizeof(uint32_t) * nn);
        so.decided = (uint8_t *)malloc(nn);
        so.slots = (uint32_t *)malloc(sizeof(uint32_t) * 2 * (size_t)cap);
        orc_rrs_stage(&ov, ns, &sp, nets, &so);
        rep->nonfinite_drops += so.nonfinite;
        if (so.dropped > 0) {
            rc->overflow_events += 1;
            rc->alpha *= (1.0f - rc->eps);
            rep->overflow_events += 1;
            rep->bias_drop_events += so.dropped;
        }
        for (j = 0; j < ns; ++j) {
            vd[j].q_norm = so.q_norm[j];
            vd[j].q_real = so.q_real[j];
            vd[j].decided = so.decided[j];
        }
        /* children (:413-482) */
        memset(used, 0, so.spawned);
        for (j = 0; j < ns; ++j) {
            orc_vrec *v = &vd[j];
            const uint32_t off = so.offset[j];
            const uint32_t rem = so.spawned - (so.spawned < off ? so.spawned : off);
            const uint32_t kept = (uint32_t)so.k[j] < rem ? (uint32_t)so.k[j] : rem;
            const int kind = s->mat_kind[v->material];
            const float *alb = s->mat_albedo + 3 * v->material;
            const float mrough = s->mat_roughness[v->material];
            const float qr = v->q_real;
            for (uint32_t c = 0; c < kept; ++c) {
                const uint64_t ck = orc_child_path_key(v->key, c);
                float pick, l1, l2, b1, b2, dummy;
                orc_path_floats2(cfg->seed, ck, (uint32_t)depth, 0x33, &pick, &dummy);
                orc_path_floats2(cfg->seed, ck, (uint32_t)depth, 0x44, &l1, &l2);
                /* sample_nee (:155-184) over Scene::sample_light (scene.cpp:66-82) */
                if (L.n > 0) {
                    uint32_t li = (uint32_t)(pick * (float)L.n);
                    if (li > L.n - 1)
                        li = L.n - 1;
                    const uint32_t lt = L.tris[li];
                    const float su = sqrtf(l1);
                    const float bu = 1.0f - su, bv = l2 * su;
                    const float *q0 = s->pos + 3 * s->idx[3 * lt], *q1 = s->pos + 3 * s->idx[3 * lt + 1],
                                *q2 = s->pos + 3 * s->idx[3 * lt + 2];
                    float lp[3], ln[3], wl[3];
                    for (int a = 0; a < 3; ++a)
                        lp[a] = ((1.0f - bu - bv) * q0[a] + bu * q1[a]) + bv * q2[a];
                    face_normal(s, lt, ln);
                    const float *le = s->mat_emission + 3 * s->mat_of_tri[lt];
                    const float pdf_area = 1.0f / ((float)L.n * L.areas[li]);
                    if (pdf_area > 0.0f) {
                        v3_sub(lp, v->p, wl);
                        const float dist2 = v3_dot(wl, wl);
                        if (dist2 > 1e-12f) {
                            const float dist = sqrtf(dist2);
                            for (int a = 0; a < 3; ++a)
                                wl[a] = wl[a] / dist;
                            const float cos_l = fabsf(v3_dot(ln, wl));
                            if (cos_l > 1e-7f) {
                                float f[3];
                                bsdf_eval(kind, alb, mrough, v->n_s, v->wo, wl, f);
                                const float cos_v = v3_dot(v->n_s, wl);
                                if (!(cos_v <= 0.0f || fmaxf3(f) <= 0.0f || fmaxf3(le) <= 0.0f)) {
                                    const float scale = cos_v * cos_l / (dist2 * pdf_area);
                                    const float pdf_l = pdf_area * dist2 / stdmaxf(cos_l, 1e-8f);
                                    const float pdf_b = bsdf_pdf(kind, mrough, v->n_s, v->wo, wl);
                                    rep->shadow_rays += 1;
                                    if (!occluded_brute(s, v->p, wl, dist * (1.0f - 1e-3f))) {
                                        const float mis = mis_power2(pdf_l, pdf_b);
                                        for (int a = 0; a < 3; ++a) {
                                            const float wq = v->weight[a] / qr;
                                            v->nee[a] += (double)(wq * ((f[a] * le[a]) * scale * mis));
                                        }
                                    }
                                }
                            }
                        }
                    }
                }
                orc_path_floats2(cfg->seed, ck, (uint32_t)depth, 0x22, &b1, &b2);
                float wi[3], pdf, thr[3];
                if (!orc_bsdf_sample(kind, alb, mrough, v->n_s, v->wo, b1, b2, wi, &pdf, thr))
                    continue;
                orc_path_state *ch = &next[off + c];
                memset(ch, 0, sizeof *ch);
                for (int a = 0; a < 3; ++a) {
                    ch->o[a] = v->p[a];
                    ch->d[a] = wi[a];
                    ch->w[a] = v->weight[a] * thr[a] / qr;
                }
                ch->t_max = INFINITY;
                if (!(isfinite(ch->w[0]) && isfinite(ch->w[1]) && isfinite(ch->w[2]))) {
                    rep->nonfinite_drops += 1;
                    continue;
                }
                ch->key = ck;
                ch->prev_pdf = pdf;
                ch->rrs = v->rrs * qr;
                ch->pixel = v->pixel;
                ch->parent = (int32_t)j;
                ch->depth = (uint16_t)(depth + 1);
                used[off + c] = 1;
            }
        }
        for (j = 0; j < ns; ++j)
            for (int a = 0; a < 3; ++a) {
                frame[3 * vd[j].pixel + a] += vd[j].nee[a];
                vd[j].s[a] += vd[j].nee[a];
            }
        uint32_t w = 0;
        for (uint32_t slot = 0; slot < so.spawned; ++slot)
            if (used[slot])
                queue[w++] = next[slot];
        n = w;
        free(p01); free(wo01); free(rough); free(wgt); free(ipx); free(keys);
        free(so.q_orig); free(so.q_norm); free(so.q_real); free(so.u); free(so.k); free(so.offset);
        free(so.decided); free(so.slots);
    }
    /* reverse pass (:504-507) */
    for (int d = B; d >= 2; --d)
        for (uint32_t j = 0; j < nverts[d]; ++j)
            if (verts[d][j].parent >= 0)
                for (int a = 0; a < 3; ++a)
                    verts[d - 1][verts[d][j].parent].s[a] += verts[d][j].s[a];
    if (cfg->collect_training && train) { /* :511-544 */
        const size_t start = *n_train;
        for (int d = 1; d < B; ++d) {
            const orc_vrec *vd = verts[d];
            for (uint32_t j = 0; vd && j < nverts[d]; ++j) {
                const orc_vrec *v = &vd[j];
                if (!v->decided)
                    continue;
                float lo_[3];
                for (int a = 0; a < 3; ++a)
                    lo_[a] = v->weight[a] > 0.0f ? (float)(v->s[a] / (double)v->weight[a]) : 0.0f;
                if (!(isfinite(lo_[0]) && isfinite(lo_[1]) && isfinite(lo_[2]))) {
                    rep->nonfinite_drops += 1;
                    continue;
                }
                if (*n_train >= train_cap) {
                    rc_err = -1;
                    continue;
                }
                orc_train_sample *t = &train[(*n_train)++];
                memset(t, 0, sizeof *t);
                memcpy(t->position, v->p01, 12);
                memcpy(t->omega_o, v->wo01, 8);
                t->roughness = v->roughness;
                memcpy(t->t_x, v->weight, 12);
                memcpy(t->i_pixel, i_acc + 3 * v->pixel, 12);
                memcpy(t->lo_sample, lo_, 12);
                t->q_norm = v->q_norm;
                t->q_real = v->q_real;
                t->pixel = v->pixel;
                t->k_i = 1.0f;
                t->depth = (uint16_t)d;
            }
        }
        orc_train_k_i(train, start, *n_train, npx);
        rep->train_samples = *n_train - start;
    }
    for (int d = 0; d <= B; ++d)
        free(verts[d]);
    free(queue); free(next); free(used); free(hit_t); free(hit_tri); free(cls);
    free(L.tris); free(L.areas); free(L.index_of_tri);
    return rc_err;
}
