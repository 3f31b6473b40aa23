// nrrs_train.cu -- online training steps on the GPU:
// NeuralRrs::stat_loss_impl (networks.cpp:349-391) and rrs_loss_impl
// (:418-460) with Mlp::backward (mlp.cpp:74-111) and HashGrid::encode_backward
// (hashgrid.cpp:84-103), then Adam (optimizer.hpp:21-32) and the EMA shadow
// (optimizer.hpp:54-61).
//
//   stat_fwd_bwd_kernel  one thread per TrainSample: grid encode + stat tail,
//                        MLP forward (fp32), relative-L2 loss and d_y, the
//                        backward through the MLP, and the grid gradient by
//                        scatter-add; activations and deltas go to a per-sample
//                        workspace record for the weight gradients
//   rrs_fwd_bwd_kernel   the same for the RRSNet: snapshot StatNet stats, NRRS
//                        (11 inputs) or AID (own grid + tail) input, softplus,
//                        warmup / full-phase loss, backward, AID grid scatter
//   mlp_dw_kernel<OUT>   dW = sum_s delta_s in_s^T, db = sum_s delta_s: per-CTA
//                        partials over sample chunks staged in smem, then a
//                        fixed-order reduction over CTAs
//   adam_ema_kernel      grad * inv_scale -> Adam with bias correction -> EMA
#include "nrrs_device.cuh"
#include "nrrs_internal.h"

#include <cub/device/device_radix_sort.cuh>

#include <cuda_runtime.h>

namespace nrrs {

constexpr int kTH = 32;                       // hidden width (mlp.hpp)
constexpr int kTOut = 6;                      // StatNet outputs
constexpr int kWs = 4 * kTH + 3 * kTH + 8;    // per-sample workspace: in0, post0..2, delta0..2, delta3
constexpr int kDwChunk = 32;                  // samples staged per smem chunk in stat_dw_kernel

__host__ __device__ inline int mlp_params(int in, int out) {
    return (kTH * in + kTH) + 2 * (kTH * kTH + kTH) + (out * kTH + out);
}
__host__ __device__ inline int stat_param_count(int in) { return mlp_params(in, kTOut); }
__host__ __device__ inline int stat_layer_offset(int in, int l) {  // hidden layers and head start (any out)
    return l == 0 ? 0 : (kTH * in + kTH) + (l - 1) * (kTH * kTH + kTH);
}

// one_blob_encode (encodings.hpp:31-44), exact exp
__device__ __forceinline__ void one_blob_exact(float x, int bins, float *out) {
    const float sigma = 1.0f / (float)bins;
    const float inv_two_sigma2 = 1.0f / (2.0f * sigma * sigma);
    float sum = 0.0f;
    for (int i = 0; i < bins; ++i) {
        const float d = x - ((float)i + 0.5f) / (float)bins;
        out[i] = expf(-d * d * inv_two_sigma2);
        sum += out[i];
    }
    const float inv = 1.0f / sum;
    for (int i = 0; i < bins; ++i)
        out[i] *= inv;
}

// the 8 corners of level l: table offsets (floats) and trilinear weights (hashgrid.cpp:38-82)
// Scatter key of a grid-gradient contribution: (level << (2 + log2 T)) | 2 * entry.  Bit 1 + log2 T
// is never set by a real entry, only by the 0xFFFFFFFF sentinel of a slot that contributed nothing,
// so a sort over bits [1, 2 + log2 T) (one level) or [1, 2 + log2 T + level bits) (all levels)
// puts the sentinel after every real entry.  base = (level * T + entry) * 2 (the gradient offset).
__device__ __forceinline__ uint32_t scatter_key(uint32_t base, int lv, uint32_t table_size) {
    const uint32_t e2 = base - 2u * (uint32_t)lv * table_size;
    return ((uint32_t)lv << (__ffs((int)table_size) + 1)) | e2;
}
__device__ __forceinline__ void grid_corners(const TrainGrid &g, int l, const float p[3], uint32_t base[8],
                                             float w[8]) {
    const uint32_t res = (uint32_t)g.base_resolution << l;
    float f[3];
    uint32_t c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float v = p[a] < 0.0f ? 0.0f : (1.0f < p[a] ? 1.0f : p[a]);
        f[a] = v * (float)res;
        c[a] = min((uint32_t)f[a], res - 1u);
    }
    const float tx = f[0] - (float)c[0], ty = f[1] - (float)c[1], tz = f[2] - (float)c[2];
    const bool dense = (g.dense_mask >> l) & 1u;
    const uint32_t nn = res + 1u, m = g.table_size - 1u;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t ox = k & 1, oy = (k >> 1) & 1, oz = k >> 2;
        w[k] = (ox ? tx : 1.0f - tx) * (oy ? ty : 1.0f - ty) * (oz ? tz : 1.0f - tz);
        const uint32_t x = c[0] + ox, y = c[1] + oy, z = c[2] + oz;
        const uint32_t idx = dense ? (x * nn + y) * nn + z : (x ^ (y * 2654435761u) ^ (z * 805459861u)) & m;
        base[k] = ((uint32_t)l * g.table_size + idx) * 2u;
    }
}

// One 32-wide layer z = W a + b (W column-major [c][r] in smem, mlp.cpp:63-66): per output r the
// sum over c runs in order with one FMA per term -- the plain loop's arithmetic.  LI > 0: the input
// width is a compile-time constant, the loops unroll (a, z stay in registers) and W is read as
// 16-byte vectors of four outputs; LI == 0: the runtime width `li`.
template <int LI>
__device__ __forceinline__ void dense_fwd(const float *W, const float *b, int li, const float (&a)[kTH],
                                          float (&z)[kTH]) {
    if constexpr (LI > 0) {
#pragma unroll
        for (int r = 0; r < kTH; ++r)
            z[r] = 0.0f;
#pragma unroll
        for (int c = 0; c < LI; ++c) {
            asm volatile("" ::: "memory");  // one column's W in flight at a time (no hoisting into spills)
            const float ac = a[c];
#pragma unroll
            for (int r4 = 0; r4 < kTH / 4; ++r4) {
                const float4 w4 = *reinterpret_cast<const float4 *>(W + c * kTH + 4 * r4);
                z[4 * r4] = fmaf(w4.x, ac, z[4 * r4]);
                z[4 * r4 + 1] = fmaf(w4.y, ac, z[4 * r4 + 1]);
                z[4 * r4 + 2] = fmaf(w4.z, ac, z[4 * r4 + 2]);
                z[4 * r4 + 3] = fmaf(w4.w, ac, z[4 * r4 + 3]);
            }
        }
#pragma unroll
        for (int r = 0; r < kTH; ++r)
            z[r] = z[r] + b[r];
    } else {
        for (int r = 0; r < kTH; ++r) {
            float acc = 0.0f;
            for (int c = 0; c < li; ++c)
                acc += W[c * kTH + r] * a[c];
            z[r] = acc + b[r];
        }
    }
}

// da = W^T delta for one 32-wide layer (mlp.cpp:74-111): per input c the sum over r in order.
template <int LI>
__device__ __forceinline__ void dense_bwd(const float *W, int li, const float (&delta)[kTH], float (&da)[kTH]) {
    if constexpr (LI > 0) {
#pragma unroll
        for (int c = 0; c < LI; ++c) {
            asm volatile("" ::: "memory");
            float acc = 0.0f;
#pragma unroll
            for (int r4 = 0; r4 < kTH / 4; ++r4) {
                const float4 w4 = *reinterpret_cast<const float4 *>(W + c * kTH + 4 * r4);
                acc = fmaf(w4.x, delta[4 * r4], acc);
                acc = fmaf(w4.y, delta[4 * r4 + 1], acc);
                acc = fmaf(w4.z, delta[4 * r4 + 2], acc);
                acc = fmaf(w4.w, delta[4 * r4 + 3], acc);
            }
            da[c] = acc;
        }
    } else {
        for (int c = 0; c < li; ++c) {
            float acc = 0.0f;
            for (int r = 0; r < kTH; ++r)
                acc += W[c * kTH + r] * delta[r];
            da[c] = acc;
        }
    }
}

// 32 floats to a 16-byte-aligned workspace row slice
__device__ __forceinline__ void store32(float *dst, const float (&v)[kTH]) {
#pragma unroll
    for (int i = 0; i < kTH / 4; ++i)
        reinterpret_cast<float4 *>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}

__global__ void __launch_bounds__(256) stat_fwd_bwd_kernel(TrainStepParams p) {  // any grid / input width
    extern __shared__ float w_s[];
    const int tid = threadIdx.x;
    const int in = p.in, P = stat_param_count(in);
    for (int i = tid; i < P; i += blockDim.x)
        w_s[i] = p.mlp[i];
    __syncthreads();
    const float slope = 0.01f;
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + tid;
    double my_loss = 0.0;
    if (s < p.n) {
        const nrrs_train_sample &t = p.batch[s];
        float *ws = p.ws + s * kWs;
        const int gd = 2 * p.grid.levels;
        float a[kTH];
        // ---- encode_stat_inputs (networks.cpp:206-217): grid features, then the stat tail ----
        for (int l = 0; l < p.grid.levels; ++l) {
            uint32_t base[8];
            float w[8];
            grid_corners(p.grid, l, t.position, base, w);
            float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                a0 += w[k] * __ldg(p.theta_grid + base[k]);
                a1 += w[k] * __ldg(p.theta_grid + base[k] + 1);
            }
            a[2 * l] = a0;
            a[2 * l + 1] = a1;
        }
        one_blob_exact(t.omega_o[0], 4, a + gd);
        one_blob_exact(t.omega_o[1], 4, a + gd + 4);
        one_blob_exact(1.0f - expf(-t.roughness), 8, a + gd + 8);  // roughness_remap (encodings.hpp:65-67)
        for (int i = in; i < kTH; ++i)
            a[i] = 0.0f;
        for (int i = 0; i < kTH; ++i)
            ws[i] = a[i];
        // ---- Mlp::forward (mlp.cpp:52-72), keeping post-activations ----
        for (int l = 0; l < 3; ++l) {
            const int li = l == 0 ? in : kTH;
            const float *W = w_s + stat_layer_offset(in, l), *b = W + kTH * li;
            float z[kTH];
            for (int r = 0; r < kTH; ++r) {
                float acc = 0.0f;
                for (int c = 0; c < li; ++c)
                    acc += W[c * kTH + r] * a[c];
                z[r] = acc + b[r];
            }
            for (int r = 0; r < kTH; ++r) {
                const float zs = z[r] * slope;
                a[r] = z[r] < zs ? zs : z[r];  // cwiseMax(z, slope z)
                ws[kTH * (l + 1) + r] = a[r];
            }
        }
        float y[kTOut];
        {
            const float *W = w_s + stat_layer_offset(in, 3), *b = W + kTOut * kTH;
            for (int r = 0; r < kTOut; ++r) {
                float acc = 0.0f;
                for (int c = 0; c < kTH; ++c)
                    acc += W[c * kTOut + r] * a[c];
                y[r] = acc + b[r];
            }
        }
        // ---- relative L2 against (lo, lo^2) (networks.cpp:370-381) ----
        float dy[kTOut];
        for (int c = 0; c < 3; ++c) {
            const float lo = t.lo_sample[c];
            const float t2 = lo * lo;
            const float d1 = y[c] - lo, inv1 = 1.0f / (lo * lo + p.eps);
            const float d2 = y[3 + c] - t2, inv2 = 1.0f / (t2 * t2 + p.eps);
            my_loss += (double)(d1 * d1 * inv1) + (double)(d2 * d2 * inv2);
            dy[c] = 2.0f * d1 * inv1 * p.inv_n * p.d_scale;
            dy[3 + c] = 2.0f * d2 * inv2 * p.inv_n * p.d_scale;
        }
        // ---- Mlp::backward (mlp.cpp:74-111) ----
        float *dws = ws + 4 * kTH;  // delta0 [32], delta1 [32], delta2 [32], delta3 [8]
        for (int r = 0; r < kTOut; ++r)
            dws[3 * kTH + r] = dy[r];
        float delta[kTH];
        {
            const float *W = w_s + stat_layer_offset(in, 3);
            for (int c = 0; c < kTH; ++c) {
                float acc = 0.0f;
                for (int r = 0; r < kTOut; ++r)
                    acc += W[c * kTOut + r] * dy[r];
                delta[c] = a[c] <= 0.0f ? acc * slope : acc;  // post2 <= 0 <=> pre2 <= 0
            }
        }
        for (int l = 2; l >= 0; --l) {
            for (int r = 0; r < kTH; ++r)
                dws[kTH * l + r] = delta[r];
            const int li = l == 0 ? in : kTH;
            const float *W = w_s + stat_layer_offset(in, l);
            float da[kTH];
            for (int c = 0; c < li; ++c) {
                float acc = 0.0f;
                for (int r = 0; r < kTH; ++r)
                    acc += W[c * kTH + r] * delta[r];
                da[c] = acc;
            }
            if (l > 0) {
                const float *post = ws + kTH * l;  // post_{l-1}
                for (int c = 0; c < kTH; ++c)
                    delta[c] = post[c] <= 0.0f ? da[c] * slope : da[c];
            } else {
                // ---- HashGrid::encode_backward: grad[base + f] += w * d_x ----
                for (int lv = 0; lv < p.grid.levels; ++lv) {
                    uint32_t base[8];
                    float w[8];
                    grid_corners(p.grid, lv, t.position, base, w);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint64_t slot = ((uint64_t)lv * p.n + s) * 8u + (uint64_t)k;  // level-major
                        NRRS_CHECK(slot < p.n * (uint64_t)p.grid.levels * 8u, "scatter slot", slot, p.n * (uint64_t)p.grid.levels * 8u);
                        p.scatter.keys[slot] = scatter_key(base[k], lv, p.grid.table_size);
                        p.scatter.vals[slot] = make_float2(w[k] * da[2 * lv], w[k] * da[2 * lv + 1]);
                    }
                }
            }
        }
    }
    // block sum of the per-sample loss terms (fixed order) -> loss_parts[block]
    __shared__ double red[8];
    double v = my_loss;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0)
        red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
        double b = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
            b += red[i];
        p.loss_parts[blockIdx.x] = b;
    }
}

// The default grid (8 levels, StatNet input 32) with compile-time widths: the same arithmetic in
// the same order as stat_fwd_bwd_kernel, with the arrays in registers and W read as 16-byte vectors.
#ifndef NRRS_TRAIN_MINB
#define NRRS_TRAIN_MINB 2  // 128 registers, 2 CTAs per SM: train_frame 1.01 -> 0.95 ms (1: 255 registers, 4: spills)
#endif
template <int LV, int IN>
__global__ void __launch_bounds__(256, NRRS_TRAIN_MINB) stat_fwd_bwd_fast_kernel(TrainStepParams p) {
    extern __shared__ __align__(16) float w_s[];
    const int tid = threadIdx.x;
    const int in = IN ? IN : p.in, levels = LV ? LV : p.grid.levels, P = stat_param_count(in);
    for (int i = tid; i < P; i += blockDim.x)
        w_s[i] = p.mlp[i];
    __syncthreads();
    const float slope = 0.01f;
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + tid;
    double my_loss = 0.0;
    if (s < p.n) {
        const nrrs_train_sample &t = p.batch[s];
        float *ws = p.ws + s * kWs;
        const int gd = 2 * levels;
        float a[kTH];
        // ---- encode_stat_inputs (networks.cpp:206-217): grid features, then the stat tail ----
#pragma unroll
        for (int l = 0; l < (LV ? LV : 8); ++l) {
            if (!LV && l >= levels)
                break;
            uint32_t base[8];
            float w[8];
            grid_corners(p.grid, l, t.position, base, w);
            float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                a0 += w[k] * __ldg(p.theta_grid + base[k]);
                a1 += w[k] * __ldg(p.theta_grid + base[k] + 1);
            }
            a[2 * l] = a0;
            a[2 * l + 1] = a1;
            asm volatile("" ::: "memory");  // one level's 16 gathers in flight at a time (registers)
        }
        one_blob_exact(t.omega_o[0], 4, a + gd);
        one_blob_exact(t.omega_o[1], 4, a + gd + 4);
        one_blob_exact(1.0f - expf(-t.roughness), 8, a + gd + 8);  // roughness_remap (encodings.hpp:65-67)
#pragma unroll
        for (int i = 0; i < kTH; ++i)
            if (i >= in)
                a[i] = 0.0f;
        store32(ws, a);
        // ---- Mlp::forward (mlp.cpp:52-72), keeping post-activations ----
#pragma unroll 1
        for (int l = 0; l < 3; ++l) {
            const int li = l == 0 ? in : kTH;
            const float *W = w_s + stat_layer_offset(in, l), *b = W + kTH * li;
            float z[kTH];
            if (l == 0)
                dense_fwd<IN>(W, b, li, a, z);
            else
                dense_fwd<(IN ? kTH : 0)>(W, b, li, a, z);
#pragma unroll
            for (int r = 0; r < kTH; ++r) {
                const float zs = z[r] * slope;
                a[r] = z[r] < zs ? zs : z[r];  // cwiseMax(z, slope z)
            }
            store32(ws + kTH * (l + 1), a);
        }
        float y[kTOut];
        {
            const float *W = w_s + stat_layer_offset(in, 3), *b = W + kTOut * kTH;
#pragma unroll
            for (int r = 0; r < kTOut; ++r) {
                float acc = 0.0f;
#pragma unroll
                for (int c = 0; c < kTH; ++c)
                    acc += W[c * kTOut + r] * a[c];
                y[r] = acc + b[r];
            }
        }
        // ---- relative L2 against (lo, lo^2) (networks.cpp:370-381) ----
        float dy[kTOut];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float lo = t.lo_sample[c];
            const float t2 = lo * lo;
            const float d1 = y[c] - lo, inv1 = 1.0f / (lo * lo + p.eps);
            const float d2 = y[3 + c] - t2, inv2 = 1.0f / (t2 * t2 + p.eps);
            my_loss += (double)(d1 * d1 * inv1) + (double)(d2 * d2 * inv2);
            dy[c] = 2.0f * d1 * inv1 * p.inv_n * p.d_scale;
            dy[3 + c] = 2.0f * d2 * inv2 * p.inv_n * p.d_scale;
        }
        // ---- Mlp::backward (mlp.cpp:74-111) ----
        float *dws = ws + 4 * kTH;  // delta0 [32], delta1 [32], delta2 [32], delta3 [8]
#pragma unroll
        for (int r = 0; r < kTOut; ++r)
            dws[3 * kTH + r] = dy[r];
        float delta[kTH];
        {
            const float *W = w_s + stat_layer_offset(in, 3);
#pragma unroll
            for (int c = 0; c < kTH; ++c) {
                float acc = 0.0f;
#pragma unroll
                for (int r = 0; r < kTOut; ++r)
                    acc += W[c * kTOut + r] * dy[r];
                delta[c] = a[c] <= 0.0f ? acc * slope : acc;  // post2 <= 0 <=> pre2 <= 0
            }
        }
#pragma unroll 1
        for (int l = 2; l >= 0; --l) {
            store32(dws + kTH * l, delta);
            const int li = l == 0 ? in : kTH;
            const float *W = w_s + stat_layer_offset(in, l);
            float da[kTH];
            if (l == 0)
                dense_bwd<IN>(W, li, delta, da);
            else
                dense_bwd<(IN ? kTH : 0)>(W, li, delta, da);
            if (l > 0) {
                const float4 *post = reinterpret_cast<const float4 *>(ws + kTH * l);  // post_{l-1}
#pragma unroll
                for (int c4 = 0; c4 < kTH / 4; ++c4) {
                    const float4 q = post[c4];
                    delta[4 * c4] = q.x <= 0.0f ? da[4 * c4] * slope : da[4 * c4];
                    delta[4 * c4 + 1] = q.y <= 0.0f ? da[4 * c4 + 1] * slope : da[4 * c4 + 1];
                    delta[4 * c4 + 2] = q.z <= 0.0f ? da[4 * c4 + 2] * slope : da[4 * c4 + 2];
                    delta[4 * c4 + 3] = q.w <= 0.0f ? da[4 * c4 + 3] * slope : da[4 * c4 + 3];
                }
            } else {
                // ---- HashGrid::encode_backward: grad[base + f] += w * d_x ----
#pragma unroll
                for (int lv = 0; lv < (LV ? LV : 8); ++lv) {
                    if (!LV && lv >= levels)
                        break;
                    uint32_t base[8];
                    float w[8];
                    grid_corners(p.grid, lv, t.position, base, w);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint64_t slot = ((uint64_t)lv * p.n + s) * 8u + (uint64_t)k;  // level-major
                        NRRS_CHECK(slot < p.n * (uint64_t)p.grid.levels * 8u, "scatter slot", slot, p.n * (uint64_t)p.grid.levels * 8u);
                        p.scatter.keys[slot] = scatter_key(base[k], lv, p.grid.table_size);
                        p.scatter.vals[slot] = make_float2(w[k] * da[2 * lv], w[k] * da[2 * lv + 1]);
                    }
                }
            }
        }
    }
    // block sum of the per-sample loss terms (fixed order) -> loss_parts[block]
    __shared__ double red[8];
    double v = my_loss;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0)
        red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
        double b = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
            b += red[i];
        p.loss_parts[blockIdx.x] = b;
    }
}

// weight / bias gradients from the workspace: CTA b sums samples [b*per, (b+1)*per).  Each thread
// owns a 4 (output row) x 4 (input column) block of one layer's [W | b] (the bias is input column
// `li`, whose value is 1) and accumulates it over the CTA's samples in sample order with one FMA
// per entry and sample -- the order and arithmetic of a per-parameter loop, so the partials are
// bit-identical to it -- reading two 16-byte vectors (4 deltas, 4 inputs) per sample from the
// staged chunk instead of two scalars per entry.  Blocks: 3 x (8 x ceil((li + 1) / 4)) for the
// three 32-wide layers plus ceil(OUT / 4) x 9 for the head: <= 234 of the 256 threads.
template <int OUT>
__global__ void __launch_bounds__(256) mlp_dw_kernel(const float *ws, uint64_t n, int in, uint64_t per,
                                                     float *partials) {
    static_assert(OUT <= 8, "head deltas: 8 workspace slots");
    __shared__ __align__(16) float st[kDwChunk][kWs];
    const int tid = threadIdx.x, P = mlp_params(in, OUT);
    // this thread's block: layer l, rows [r0, r0 + 4), columns [c0, c0 + 4)
    int l = -1, r0 = 0, c0 = 0, t = tid;
    for (int L = 0; L < 4 && l < 0; ++L) {
        const int li = L == 0 ? in : kTH, lo = L == 3 ? OUT : kTH;
        const int ct = (li + 1 + 3) / 4, nb = ((lo + 3) / 4) * ct;
        if (t < nb) {
            l = L;
            r0 = 4 * (t / ct);
            c0 = 4 * (t % ct);
        } else {
            t -= nb;
        }
    }
    const int li = l == 0 ? in : kTH, lo = l == 3 ? OUT : kTH;
    const int doff = 4 * kTH + kTH * (l < 0 ? 0 : l) + r0, ioff = kTH * (l < 0 ? 0 : l) + c0;
    // column kinds: 0 input, 1 the bias column (value 1), 2 beyond
    int kind[4];
#pragma unroll
    for (int b = 0; b < 4; ++b)
        kind[b] = c0 + b < li ? 0 : (c0 + b == li ? 1 : 2);
    const bool edge = c0 + 3 >= li;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
            acc[a][b] = 0.0f;
    const uint64_t s0 = (uint64_t)blockIdx.x * per, s1 = s0 + per < n ? s0 + per : n;
    // chunks of kDwChunk records (kWs floats each, contiguous) move as 16-byte vectors; the next
    // chunk's vectors are loaded into registers before this chunk's FMAs, stored after them
    constexpr int kV = kDwChunk * kWs / 4, kPerThread = (kV + 255) / 256;
    static_assert(kWs % 4 == 0, "16-byte workspace records");
    float4 *st4 = reinterpret_cast<float4 *>(&st[0][0]);
    float4 nxt[kPerThread];
    auto fetch = [&](uint64_t c) {
        const int cnt = (int)(s1 - c < (uint64_t)kDwChunk ? s1 - c : (uint64_t)kDwChunk);
        const float4 *src = reinterpret_cast<const float4 *>(ws + c * kWs);
#pragma unroll
        for (int u = 0; u < kPerThread; ++u) {
            const int v = tid + 256 * u;
            nxt[u] = v < cnt * (kWs / 4) ? __ldcs(src + v) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
    };
    if (s0 < s1)
        fetch(s0);
    for (uint64_t c = s0; c < s1; c += kDwChunk) {
        const int cnt = (int)(s1 - c < (uint64_t)kDwChunk ? s1 - c : (uint64_t)kDwChunk);
#pragma unroll
        for (int u = 0; u < kPerThread; ++u) {
            const int v = tid + 256 * u;
            if (v < kV)
                st4[v] = nxt[u];
        }
        __syncthreads();
        if (c + kDwChunk < s1)
            fetch(c + kDwChunk);
        if (l >= 0) {
            for (int j = 0; j < cnt; ++j) {
                const float4 d4 = *reinterpret_cast<const float4 *>(&st[j][doff]);
                float4 x4 = *reinterpret_cast<const float4 *>(&st[j][ioff]);
                if (edge) {
                    x4.x = kind[0] == 0 ? x4.x : (kind[0] == 1 ? 1.0f : 0.0f);
                    x4.y = kind[1] == 0 ? x4.y : (kind[1] == 1 ? 1.0f : 0.0f);
                    x4.z = kind[2] == 0 ? x4.z : (kind[2] == 1 ? 1.0f : 0.0f);
                    x4.w = kind[3] == 0 ? x4.w : (kind[3] == 1 ? 1.0f : 0.0f);
                }
                const float d[4] = {d4.x, d4.y, d4.z, d4.w}, x[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        acc[a][b] = fmaf(d[a], x[b], acc[a][b]);
            }
        }
        __syncthreads();
    }
    if (l < 0)
        return;
    const int base = stat_layer_offset(in, l);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int r = r0 + a;
        if (r >= lo)
            continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int col = c0 + b;
            if (kind[b] == 2)
                continue;
            const int q = base + (col < li ? col * lo + r : lo * li + r);  // column-major W, then bias
            NRRS_CHECK(q < P, "mlp gradient index", q, P);
            partials[(uint64_t)blockIdx.x * P + q] = acc[a][b];
        }
    }
}

// Sequential sum of n values p[0], p[stride], ... in index order, with kB loads in flight per round
// trip (the adds keep the order, so the result equals the plain loop's).
template <typename T>
__device__ __forceinline__ T ordered_sum(const T *p, int n, uint64_t stride) {
    constexpr int kB = 16;
    T s = T(0);
    for (int b0 = 0; b0 < n; b0 += kB) {
        T v[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u)
            v[u] = b0 + u < n ? p[(uint64_t)(b0 + u) * stride] : T(0);
#pragma unroll
        for (int u = 0; u < kB; ++u)
            if (b0 + u < n)
                s += v[u];
    }
    return s;
}

// any non-finite entry of g[0, n) -> *flag (16-byte loads where aligned)
__device__ __forceinline__ void flag_nonfinite(const float *g, uint64_t n, uint32_t *flag) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
    bool bad = false;
    if ((reinterpret_cast<uintptr_t>(g) & 15u) == 0) {
        const float4 *g4 = reinterpret_cast<const float4 *>(g);
        for (uint64_t i = tid; i < n / 4; i += nt) {
            const float4 v = g4[i];
            bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
        }
        for (uint64_t i = n / 4 * 4 + tid; i < n; i += nt)
            bad |= !isfinite(g[i]);
    } else {
        for (uint64_t i = tid; i < n; i += nt)
            bad |= !isfinite(g[i]);
    }
    if (bad)
        atomicOr(flag, 1u);
}

// g_mlp[q] = sum over CTAs (fixed order); loss = sum of block parts * inv_n; finite flags
__global__ void stat_reduce_kernel(const float *partials, int nparts, int P, float *g_mlp, const double *loss_parts,
                                   int nloss, float inv_n, double *loss_out, const float *g_grid, uint64_t ngrid,
                                   uint32_t *nonfinite) {
    const int tid = threadIdx.x + blockIdx.x * blockDim.x;
    for (int q = tid; q < P; q += gridDim.x * blockDim.x) {
        const float s = ordered_sum(partials + q, nparts, (uint64_t)P);
        g_mlp[q] = s;
        if (!isfinite(s))
            atomicOr(nonfinite, 1u);
    }
    flag_nonfinite(g_grid, ngrid, nonfinite);
    if (tid == 0)
        *loss_out = ordered_sum(loss_parts, nloss, 1) * (double)inv_n;
}

// grad *= inv_scale; Adam::step (optimizer.hpp:21-32); EmaTracker::update (:54-61)
__global__ void adam_ema_kernel(float *theta, const float *grad, float *m, float *v, float *shadow, uint64_t n,
                                AdamParams a) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float g = __fmul_rn(grad[i], a.inv_scale);
        const float mi = __fadd_rn(__fmul_rn(a.beta1, m[i]), __fmul_rn(__fsub_rn(1.0f, a.beta1), g));
        const float vi = __fadd_rn(__fmul_rn(a.beta2, v[i]), __fmul_rn(__fsub_rn(1.0f, a.beta2), __fmul_rn(g, g)));
        m[i] = mi;
        v[i] = vi;
        const float upd = __fdiv_rn(__fmul_rn(a.lr, __fmul_rn(mi, a.c1)), __fadd_rn(__fsqrt_rn(__fmul_rn(vi, a.c2)), a.eps));
        const float th = __fsub_rn(theta[i], upd);
        theta[i] = th;
        if (shadow)
            shadow[i] = __fadd_rn(__fmul_rn(a.decay, shadow[i]), __fmul_rn(__fsub_rn(1.0f, a.decay), th));
    }
}

// ---- RRSNet step: NeuralRrs::rrs_loss_impl (networks.cpp:418-460) ----

// plain forward of the published StatNet snapshot (snapshot_stats_batch, networks.cpp:219-224)
__device__ __forceinline__ void snapshot_stats(const RrsStepParams &p, const float *w_stat,
                                               const nrrs_train_sample &t, float st[6]) {
    const int gd = 2 * p.grid.levels, in = gd + 16;
    float a[kTH];
    for (int l = 0; l < p.grid.levels; ++l) {
        uint32_t base[8];
        float w[8];
        grid_corners(p.grid, l, t.position, base, w);
        float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a0 += w[k] * __ldg(p.snap_grid + base[k]);
            a1 += w[k] * __ldg(p.snap_grid + base[k] + 1);
        }
        a[2 * l] = a0;
        a[2 * l + 1] = a1;
    }
    one_blob_exact(t.omega_o[0], 4, a + gd);
    one_blob_exact(t.omega_o[1], 4, a + gd + 4);
    one_blob_exact(1.0f - expf(-t.roughness), 8, a + gd + 8);
    for (int l = 0; l < 3; ++l) {
        const int li = l == 0 ? in : kTH;
        const float *W = w_stat + stat_layer_offset(in, l), *b = W + kTH * li;
        float z[kTH];
        for (int r = 0; r < kTH; ++r) {
            float acc = 0.0f;
            for (int c = 0; c < li; ++c)
                acc += W[c * kTH + r] * a[c];
            z[r] = acc + b[r];
        }
        for (int r = 0; r < kTH; ++r) {
            const float zs = z[r] * 0.01f;
            a[r] = z[r] < zs ? zs : z[r];
        }
    }
    const float *W = w_stat + stat_layer_offset(in, 3), *b = W + kTOut * kTH;
    for (int r = 0; r < kTOut; ++r) {
        float acc = 0.0f;
        for (int c = 0; c < kTH; ++c)
            acc += W[c * kTOut + r] * a[c];
        st[r] = acc + b[r];
    }
}

__device__ __forceinline__ float box_cox_exact(float x) {  // encodings.hpp:54-62, lambda 0.5
    if (x < 0.0f)
        x = 0.0f;
    return (powf(x, 0.5f) - 1.0f) / 0.5f;
}

__global__ void __launch_bounds__(256) rrs_fwd_bwd_kernel(RrsStepParams p) {
    extern __shared__ float w_s[];
    const int tid = threadIdx.x;
    const int gd = 2 * p.grid.levels, Ps = stat_param_count(gd + 16), Pr = mlp_params(p.in, 1);
    float *w_stat = w_s, *w_rrs = w_s + Ps;
    for (int i = tid; i < Ps; i += blockDim.x)
        w_stat[i] = p.snap_mlp[i];
    for (int i = tid; i < Pr; i += blockDim.x)
        w_rrs[i] = p.rrs_mlp[i];
    __syncthreads();
    const float slope = 0.01f;
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + tid;
    double pmin = 0.0, pavg = 0.0, prrs = 0.0;
    uint32_t skipped = 0;
    if (s < p.n) {
        const nrrs_train_sample &t = p.batch[s];
        float *ws = p.ws + s * kWs;
        float st[6];
        snapshot_stats(p, w_stat, t, st);
        // encode_rrs_inputs (networks.cpp:226-250)
        float a[kTH];
        const float imean = (t.i_pixel[0] + (t.i_pixel[1] + t.i_pixel[2])) / 3.0f;
        if (p.variant == 0) {  // build_nrrs_input (networks.cpp:137-147)
            for (int c = 0; c < 3; ++c) {
                a[c] = box_cox_exact(st[c]);
                a[3 + c] = box_cox_exact(st[3 + c]);
                a[6 + c] = box_cox_exact(t.t_x[c]);
            }
            a[9] = box_cox_exact(imean);
            a[10] = 1.0f - expf(-t.roughness);
        } else {                // AID: own grid + build_aid_tail (networks.cpp:149-157)
            for (int l = 0; l < p.grid.levels; ++l) {
                uint32_t base[8];
                float w[8];
                grid_corners(p.grid, l, t.position, base, w);
                float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    a0 += w[k] * __ldg(p.rrs_grid + base[k]);
                    a1 += w[k] * __ldg(p.rrs_grid + base[k] + 1);
                }
                a[2 * l] = a0;
                a[2 * l + 1] = a1;
            }
            one_blob_exact(t.omega_o[0], 4, a + gd);
            one_blob_exact(t.omega_o[1], 4, a + gd + 4);
            for (int c = 0; c < 3; ++c)
                a[gd + 8 + c] = box_cox_exact(t.t_x[c]);
            a[gd + 11] = box_cox_exact(imean);
            one_blob_exact(1.0f - expf(-t.roughness), 4, a + gd + 12);
        }
        for (int i = p.in; i < kTH; ++i)
            a[i] = 0.0f;
        for (int i = 0; i < kTH; ++i)
            ws[i] = a[i];
        for (int l = 0; l < 3; ++l) {
            const int li = l == 0 ? p.in : kTH;
            const float *W = w_rrs + stat_layer_offset(p.in, l), *b = W + kTH * li;
            float z[kTH];
            for (int r = 0; r < kTH; ++r) {
                float acc = 0.0f;
                for (int c = 0; c < li; ++c)
                    acc += W[c * kTH + r] * a[c];
                z[r] = acc + b[r];
            }
            for (int r = 0; r < kTH; ++r) {
                const float zs = z[r] * slope;
                a[r] = z[r] < zs ? zs : z[r];
                ws[kTH * (l + 1) + r] = a[r];
            }
        }
        const float *Wh = w_rrs + stat_layer_offset(p.in, 3);
        float zacc = 0.0f;
        for (int c = 0; c < kTH; ++c)
            zacc += Wh[c] * a[c];
        const float z = zacc + Wh[kTH];
        const float q = z < 0.0f ? log1pf(expf(z)) : 0.5f * z + 0.6931471805599453f;  // softplus_mod
        float d_q = 0.0f;
        if (p.phase == 0) {
            const float d = q - 1.0f, inv = 1.0f / (1.0f + p.eps);
            prrs += (double)(d * d * inv);
            d_q = 2.0f * d * inv * p.inv_n;
        } else {
            const uint32_t px = t.pixel;
            const float inv_k = t.k_i > 0.0f ? 1.0f / t.k_i : 1.0f;
            if (px < p.n_errors) {
                const float pe_e = p.errors[2 * px], pe_inv = p.errors[2 * px + 1];
                float gvar = 0.0f;
                const float wl = luminance(t.t_x[0], t.t_x[1], t.t_x[2]);
                if (t.q_real < 1.0f) {
                    if (t.q_real > 0.0f) {
                        const float hl = luminance(t.lo_sample[0], t.lo_sample[1], t.lo_sample[2]);
                        gvar = -(wl * wl) * (hl * hl) / (t.q_real * t.q_real);
                    }
                } else {
                    float var[3];
                    for (int c = 0; c < 3; ++c) {
                        const float v = st[3 + c] - st[c] * st[c];
                        var[c] = v < 0.0f ? 0.0f : v;
                    }
                    gvar = -(wl * wl) * luminance(var[0], var[1], var[2]) / (t.q_real * t.q_real);
                }
                const float de_dq = pe_inv * gvar * inv_k;
                pmin += (double)(pe_e * inv_k);
                const float dev = pe_e - p.e_avg;
                pavg += (double)(dev * dev * inv_k);
                d_q += (p.gamma_min * de_dq + p.gamma_avg * 2.0f * dev * de_dq) * p.inv_n;
            } else {
                skipped = 1;
            }
            const float gap = q - t.q_norm;
            prrs += (double)(gap * gap);
            d_q += p.gamma_rrs * 2.0f * gap * p.inv_n;
        }
        const float sg = z < 0.0f ? expf(z) / (1.0f + expf(z)) : 0.5f;  // softplus_mod_grad
        const float dy = d_q * sg * p.d_scale;
        // Mlp::backward (mlp.cpp:74-111)
        float *dws = ws + 4 * kTH;
        dws[3 * kTH] = dy;
        float delta[kTH];
        for (int c = 0; c < kTH; ++c) {
            const float acc = Wh[c] * dy;
            delta[c] = a[c] <= 0.0f ? acc * slope : acc;
        }
        for (int l = 2; l >= 0; --l) {
            for (int r = 0; r < kTH; ++r)
                dws[kTH * l + r] = delta[r];
            const int li = l == 0 ? p.in : kTH;
            const float *W = w_rrs + stat_layer_offset(p.in, l);
            float da[kTH];
            for (int c = 0; c < li; ++c) {
                float acc = 0.0f;
                for (int r = 0; r < kTH; ++r)
                    acc += W[c * kTH + r] * delta[r];
                da[c] = acc;
            }
            if (l > 0) {
                const float *post = ws + kTH * l;
                for (int c = 0; c < kTH; ++c)
                    delta[c] = post[c] <= 0.0f ? da[c] * slope : da[c];
            } else if (p.variant == 1 && p.g_grid) {
                for (int lv = 0; lv < p.grid.levels; ++lv) {
                    uint32_t base[8];
                    float w[8];
                    grid_corners(p.grid, lv, t.position, base, w);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint64_t slot = ((uint64_t)lv * p.n + s) * 8u + (uint64_t)k;  // level-major
                        NRRS_CHECK(slot < p.n * (uint64_t)p.grid.levels * 8u, "scatter slot", slot, p.n * (uint64_t)p.grid.levels * 8u);
                        p.scatter.keys[slot] = scatter_key(base[k], lv, p.grid.table_size);
                        p.scatter.vals[slot] = make_float2(w[k] * da[2 * lv], w[k] * da[2 * lv + 1]);
                    }
                }
            }
        }
    }
    __shared__ double red[3][8];
    __shared__ uint32_t reds[8];
    double v[3] = {pmin, pavg, prrs};
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
    const uint32_t sk = __reduce_add_sync(0xffffffffu, skipped);
    if ((tid & 31) == 0) {
        for (int j = 0; j < 3; ++j)
            red[j][tid >> 5] = v[j];
        reds[tid >> 5] = sk;
    }
    __syncthreads();
    if (tid == 0) {
        double b[3] = {0.0, 0.0, 0.0};
        uint32_t bs = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            for (int j = 0; j < 3; ++j)
                b[j] += red[j][i];
            bs += reds[i];
        }
        for (int j = 0; j < 3; ++j)
            p.parts[3 * blockIdx.x + j] = b[j];
        if (bs)
            atomicAdd(p.skipped, bs);
    }
}

// snapshot_stats for the default grid (8 levels, StatNet input 32), compile-time widths
__device__ __forceinline__ void snapshot_stats_fast(const RrsStepParams &p, const float *w_stat,
                                                    const nrrs_train_sample &t, float st[6]) {
    constexpr int kLv = 8, gd = 2 * kLv, in = gd + 16;
    float a[kTH];
#pragma unroll
    for (int l = 0; l < kLv; ++l) {
        uint32_t base[8];
        float w[8];
        grid_corners(p.grid, l, t.position, base, w);
        float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            a0 += w[k] * __ldg(p.snap_grid + base[k]);
            a1 += w[k] * __ldg(p.snap_grid + base[k] + 1);
        }
        a[2 * l] = a0;
        a[2 * l + 1] = a1;
        asm volatile("" ::: "memory");
    }
    one_blob_exact(t.omega_o[0], 4, a + gd);
    one_blob_exact(t.omega_o[1], 4, a + gd + 4);
    one_blob_exact(1.0f - expf(-t.roughness), 8, a + gd + 8);
#pragma unroll 1
    for (int l = 0; l < 3; ++l) {
        const float *W = w_stat + stat_layer_offset(in, l), *b = W + kTH * kTH;
        float z[kTH];
        dense_fwd<kTH>(W, b, kTH, a, z);
#pragma unroll
        for (int r = 0; r < kTH; ++r) {
            const float zs = z[r] * 0.01f;
            a[r] = z[r] < zs ? zs : z[r];
        }
    }
    const float *W = w_stat + stat_layer_offset(in, 3), *b = W + kTOut * kTH;
#pragma unroll
    for (int r = 0; r < kTOut; ++r) {
        float acc = 0.0f;
#pragma unroll
        for (int c = 0; c < kTH; ++c)
            acc += W[c * kTOut + r] * a[c];
        st[r] = acc + b[r];
    }
}

// rrs_fwd_bwd_kernel for the default grid with compile-time widths (VAR 0: NRRS, 11 inputs; 1: AID,
// own grid + tail, 32 inputs): the same arithmetic in the same order, arrays in registers, W read as
// 16-byte vectors.  The RRSNet weights start at a 16-byte boundary after the StatNet's (w_rrs_off).
__host__ __device__ constexpr int rrs_w_offset(int ps) { return (ps + 3) & ~3; }
template <int VAR>
__global__ void __launch_bounds__(256, NRRS_TRAIN_MINB) rrs_fwd_bwd_fast_kernel(RrsStepParams p) {
    extern __shared__ __align__(16) float w_s[];
    constexpr int kLv = 8, gd = 2 * kLv, kIn = VAR ? gd + 16 : 11;
    const int tid = threadIdx.x;
    const int Ps = stat_param_count(gd + 16), Pr = mlp_params(kIn, 1);
    float *w_stat = w_s, *w_rrs = w_s + rrs_w_offset(Ps);
    for (int i = tid; i < Ps; i += blockDim.x)
        w_stat[i] = p.snap_mlp[i];
    for (int i = tid; i < Pr; i += blockDim.x)
        w_rrs[i] = p.rrs_mlp[i];
    __syncthreads();
    const float slope = 0.01f;
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + tid;
    double pmin = 0.0, pavg = 0.0, prrs = 0.0;
    uint32_t skipped = 0;
    if (s < p.n) {
        const nrrs_train_sample &t = p.batch[s];
        float *ws = p.ws + s * kWs;
        float st[6];
        snapshot_stats_fast(p, w_stat, t, st);
        float a[kTH];
        const float imean = (t.i_pixel[0] + (t.i_pixel[1] + t.i_pixel[2])) / 3.0f;
        if (VAR == 0) {  // build_nrrs_input (networks.cpp:137-147)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                a[c] = box_cox_exact(st[c]);
                a[3 + c] = box_cox_exact(st[3 + c]);
                a[6 + c] = box_cox_exact(t.t_x[c]);
            }
            a[9] = box_cox_exact(imean);
            a[10] = 1.0f - expf(-t.roughness);
        } else {         // AID: own grid + build_aid_tail (networks.cpp:149-157)
#pragma unroll
            for (int l = 0; l < kLv; ++l) {
                uint32_t base[8];
                float w[8];
                grid_corners(p.grid, l, t.position, base, w);
                float a0 = 0.0f, a1 = 0.0f;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    a0 += w[k] * __ldg(p.rrs_grid + base[k]);
                    a1 += w[k] * __ldg(p.rrs_grid + base[k] + 1);
                }
                a[2 * l] = a0;
                a[2 * l + 1] = a1;
                asm volatile("" ::: "memory");
            }
            one_blob_exact(t.omega_o[0], 4, a + gd);
            one_blob_exact(t.omega_o[1], 4, a + gd + 4);
#pragma unroll
            for (int c = 0; c < 3; ++c)
                a[gd + 8 + c] = box_cox_exact(t.t_x[c]);
            a[gd + 11] = box_cox_exact(imean);
            one_blob_exact(1.0f - expf(-t.roughness), 4, a + gd + 12);
        }
#pragma unroll
        for (int i = kIn; i < kTH; ++i)
            a[i] = 0.0f;
        store32(ws, a);
#pragma unroll 1
        for (int l = 0; l < 3; ++l) {
            const int li = l == 0 ? kIn : kTH;
            const float *W = w_rrs + stat_layer_offset(kIn, l), *b = W + kTH * li;
            float z[kTH];
            if (l == 0)
                dense_fwd<kIn>(W, b, li, a, z);
            else
                dense_fwd<kTH>(W, b, li, a, z);
#pragma unroll
            for (int r = 0; r < kTH; ++r) {
                const float zs = z[r] * slope;
                a[r] = z[r] < zs ? zs : z[r];
            }
            store32(ws + kTH * (l + 1), a);
        }
        const float *Wh = w_rrs + stat_layer_offset(kIn, 3);
        float zacc = 0.0f;
#pragma unroll
        for (int c = 0; c < kTH; ++c)
            zacc += Wh[c] * a[c];
        const float z = zacc + Wh[kTH];
        const float q = z < 0.0f ? log1pf(expf(z)) : 0.5f * z + 0.6931471805599453f;  // softplus_mod
        float d_q = 0.0f;
        if (p.phase == 0) {
            const float d = q - 1.0f, inv = 1.0f / (1.0f + p.eps);
            prrs += (double)(d * d * inv);
            d_q = 2.0f * d * inv * p.inv_n;
        } else {
            const uint32_t px = t.pixel;
            const float inv_k = t.k_i > 0.0f ? 1.0f / t.k_i : 1.0f;
            if (px < p.n_errors) {
                const float pe_e = p.errors[2 * px], pe_inv = p.errors[2 * px + 1];
                float gvar = 0.0f;
                const float wl = luminance(t.t_x[0], t.t_x[1], t.t_x[2]);
                if (t.q_real < 1.0f) {
                    if (t.q_real > 0.0f) {
                        const float hl = luminance(t.lo_sample[0], t.lo_sample[1], t.lo_sample[2]);
                        gvar = -(wl * wl) * (hl * hl) / (t.q_real * t.q_real);
                    }
                } else {
                    float var[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float v = st[3 + c] - st[c] * st[c];
                        var[c] = v < 0.0f ? 0.0f : v;
                    }
                    gvar = -(wl * wl) * luminance(var[0], var[1], var[2]) / (t.q_real * t.q_real);
                }
                const float de_dq = pe_inv * gvar * inv_k;
                pmin += (double)(pe_e * inv_k);
                const float dev = pe_e - p.e_avg;
                pavg += (double)(dev * dev * inv_k);
                d_q += (p.gamma_min * de_dq + p.gamma_avg * 2.0f * dev * de_dq) * p.inv_n;
            } else {
                skipped = 1;
            }
            const float gap = q - t.q_norm;
            prrs += (double)(gap * gap);
            d_q += p.gamma_rrs * 2.0f * gap * p.inv_n;
        }
        const float sg = z < 0.0f ? expf(z) / (1.0f + expf(z)) : 0.5f;  // softplus_mod_grad
        const float dy = d_q * sg * p.d_scale;
        float *dws = ws + 4 * kTH;
        dws[3 * kTH] = dy;
        float delta[kTH];
#pragma unroll
        for (int c = 0; c < kTH; ++c) {
            const float acc = Wh[c] * dy;
            delta[c] = a[c] <= 0.0f ? acc * slope : acc;
        }
#pragma unroll 1
        for (int l = 2; l >= 0; --l) {
            store32(dws + kTH * l, delta);
            const int li = l == 0 ? kIn : kTH;
            const float *W = w_rrs + stat_layer_offset(kIn, l);
            float da[kTH];
            if (l == 0)
                dense_bwd<kIn>(W, li, delta, da);
            else
                dense_bwd<kTH>(W, li, delta, da);
            if (l > 0) {
                const float4 *post = reinterpret_cast<const float4 *>(ws + kTH * l);
#pragma unroll
                for (int c4 = 0; c4 < kTH / 4; ++c4) {
                    const float4 q4 = post[c4];
                    delta[4 * c4] = q4.x <= 0.0f ? da[4 * c4] * slope : da[4 * c4];
                    delta[4 * c4 + 1] = q4.y <= 0.0f ? da[4 * c4 + 1] * slope : da[4 * c4 + 1];
                    delta[4 * c4 + 2] = q4.z <= 0.0f ? da[4 * c4 + 2] * slope : da[4 * c4 + 2];
                    delta[4 * c4 + 3] = q4.w <= 0.0f ? da[4 * c4 + 3] * slope : da[4 * c4 + 3];
                }
            } else if (VAR == 1 && p.g_grid) {
#pragma unroll
                for (int lv = 0; lv < kLv; ++lv) {
                    uint32_t base[8];
                    float w[8];
                    grid_corners(p.grid, lv, t.position, base, w);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint64_t slot = ((uint64_t)lv * p.n + s) * 8u + (uint64_t)k;  // level-major
                        NRRS_CHECK(slot < p.n * (uint64_t)p.grid.levels * 8u, "scatter slot", slot, p.n * (uint64_t)p.grid.levels * 8u);
                        p.scatter.keys[slot] = scatter_key(base[k], lv, p.grid.table_size);
                        p.scatter.vals[slot] = make_float2(w[k] * da[2 * lv], w[k] * da[2 * lv + 1]);
                    }
                }
            }
        }
    }
    __shared__ double red[3][8];
    __shared__ uint32_t reds[8];
    double v[3] = {pmin, pavg, prrs};
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
    const uint32_t sk = __reduce_add_sync(0xffffffffu, skipped);
    if ((tid & 31) == 0) {
        for (int j = 0; j < 3; ++j)
            red[j][tid >> 5] = v[j];
        reds[tid >> 5] = sk;
    }
    __syncthreads();
    if (tid == 0) {
        double b[3] = {0.0, 0.0, 0.0};
        uint32_t bs = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            for (int j = 0; j < 3; ++j)
                b[j] += red[j][i];
            bs += reds[i];
        }
        for (int j = 0; j < 3; ++j)
            p.parts[3 * blockIdx.x + j] = b[j];
        if (bs)
            atomicAdd(p.skipped, bs);
    }
}

// g_mlp = sum of CTA partials (fixed order), loss parts summed over blocks, finite flags
__global__ void rrs_reduce_kernel(const float *partials, int nparts, int P, float *g_mlp, const double *parts,
                                  int nblocks, double *parts_out, const float *g_grid, uint64_t ngrid,
                                  uint32_t *nonfinite) {
    const int tid = threadIdx.x + blockIdx.x * blockDim.x;
    for (int q = tid; q < P; q += gridDim.x * blockDim.x) {
        const float s = ordered_sum(partials + q, nparts, (uint64_t)P);
        g_mlp[q] = s;
        if (!isfinite(s))
            atomicOr(nonfinite, 1u);
    }
    if (g_grid)
        flag_nonfinite(g_grid, ngrid, nonfinite);
    if (tid < 3)  // the three loss-part columns, each summed over the blocks in order
        parts_out[tid] = ordered_sum(parts + tid, nblocks, 3);
}

// ---- launchers ----
size_t train_ws_floats(uint64_t n) { return (size_t)n * kWs; }
int train_param_count(int in) { return stat_param_count(in); }
int train_rrs_param_count(int in) { return mlp_params(in, 1); }
uint32_t train_dw_ctas(uint64_t n) {
    const uint64_t c = (n + 511) / 512;
    return (uint32_t)(c < 1 ? 1 : (c > 256 ? 256 : c));
}

// Sums each entry's run of sorted contributions in slot order (sample, level, corner), like the
// reference's sequential encode_backward loop: 0 + v0 + v1 + ... left to right, one __fadd_rn per
// element.  The contributions were sorted together with their keys, so a run is contiguous.
//
// One warp per 256-element window, read as 16-byte vectors (the warp's loads are one contiguous
// 1 KB of keys and 2 KB of values).  Lane l holds elements [8l, 8l + 8) and sums the runs that
// start there in order.  A run that reaches the end of its lane continues in the next lane: the
// open partial sum moves right one lane per step (shuffle), so the additions keep the reference's
// order -- a lane with no run start passes the run on after adding its 8 elements, and the loop
// runs only as many steps as the window's longest such streak.  The run open at the window's end
// is finished by lane 31 reading on past the window; the next window skips its leading elements
// (they belong to that run).  Replaces the one-thread-per-start walk (scattered 16-element
// batches, L1-wavefront-bound: 58.6 us per fold at 65,536 samples).
constexpr int kFoldE = 8;                 // elements per lane
constexpr int kFoldWin = 32 * kFoldE;     // elements per warp window
struct FoldRun {
    uint32_t key;  // 0xFFFFFFFF: none
    float a0, a1;
};
__device__ __forceinline__ uint32_t fold_offset(const GridScatter &sc, uint32_t key) {
    if (key == 0xFFFFFFFFu)
        return key;
    return (key >> sc.key_shift) * sc.level_stride + (key & ((1u << sc.key_shift) - 1u));
}
__device__ __forceinline__ void fold_flush(float *g_grid, const GridScatter &sc, uint32_t key, float a0, float a1) {
    if (key == 0xFFFFFFFFu)
        return;  // slots that contributed nothing sort last under the sentinel key
    NRRS_CHECK(key + 1u < sc.ngrid, "grid gradient entry", key + 1u, sc.ngrid);
    g_grid[key] = a0;
    g_grid[key + 1] = a1;
}
__global__ void __launch_bounds__(256) grid_scatter_fold_kernel(GridScatter sc, uint64_t m, float *g_grid) {
    const int lane = threadIdx.x & 31;
    const uint64_t b = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kFoldWin;
    if (b >= m)
        return;  // warp-uniform
    const uint64_t i0 = b + (uint64_t)lane * kFoldE;
    uint32_t k[kFoldE];
    float2 v[kFoldE];
    if (i0 + kFoldE <= m) {
        const uint4 *kp = reinterpret_cast<const uint4 *>(sc.keys_sorted + i0);
        const uint4 k0 = __ldcs(kp), k1 = __ldcs(kp + 1);
        k[0] = k0.x; k[1] = k0.y; k[2] = k0.z; k[3] = k0.w;
        k[4] = k1.x; k[5] = k1.y; k[6] = k1.z; k[7] = k1.w;
        const float4 *vp = reinterpret_cast<const float4 *>(sc.vals_sorted + i0);
#pragma unroll
        for (int q = 0; q < kFoldE / 2; ++q) {
            const float4 t = __ldcs(vp + q);
            v[2 * q] = make_float2(t.x, t.y);
            v[2 * q + 1] = make_float2(t.z, t.w);
        }
    } else {
#pragma unroll
        for (int e = 0; e < kFoldE; ++e) {
            k[e] = i0 + e < m ? sc.keys_sorted[i0 + e] : 0xFFFFFFFFu;
            v[e] = i0 + e < m ? sc.vals_sorted[i0 + e] : make_float2(0.0f, 0.0f);
        }
    }
    // scatter keys -> gradient offsets; the sentinel stays the sentinel
#pragma unroll
    for (int e = 0; e < kFoldE; ++e)
        k[e] = fold_offset(sc, k[e]);
    uint32_t pk = __shfl_up_sync(0xffffffffu, k[kFoldE - 1], 1);
    if (lane == 0)
        pk = b > 0 ? fold_offset(sc, sc.keys_sorted[b - 1]) : 0xFFFFFFFEu;
    // first run start in the lane (kFoldE: none) and the runs that start here, in order
    int fs = kFoldE;
#pragma unroll
    for (int e = kFoldE - 1; e >= 0; --e)
        if (k[e] != (e == 0 ? pk : k[e - 1]))
            fs = e;
    const bool has_start = fs < kFoldE;
    FoldRun out{0xFFFFFFFFu, 0.0f, 0.0f};  // the run open at the lane's end
#pragma unroll
    for (int e = 0; e < kFoldE; ++e) {
        if (e < fs)
            continue;
        if (k[e] != out.key || e == fs) {
            if (e > fs)
                fold_flush(g_grid, sc, out.key, out.a0, out.a1);
            out.key = k[e];
            out.a0 = __fadd_rn(0.0f, v[e].x);
            out.a1 = __fadd_rn(0.0f, v[e].y);
        } else {
            out.a0 = __fadd_rn(out.a0, v[e].x);
            out.a1 = __fadd_rn(out.a1, v[e].y);
        }
    }
    // lanes without a start carry the run coming from the left through their 8 elements; lane 0's
    // incoming run started before this window (its owner finishes it), so it is dropped here
    bool resolved = has_start || lane == 0;
    for (;;) {
        const unsigned pend = __ballot_sync(0xffffffffu, !resolved);
        if (!pend)
            break;
        const FoldRun in{__shfl_up_sync(0xffffffffu, out.key, 1), __shfl_up_sync(0xffffffffu, out.a0, 1),
                         __shfl_up_sync(0xffffffffu, out.a1, 1)};
        const bool in_ok = __shfl_up_sync(0xffffffffu, resolved ? 1 : 0, 1) != 0;
        if (!resolved && in_ok) {
            out = in;
            if (out.key != 0xFFFFFFFFu) {
#pragma unroll
                for (int e = 0; e < kFoldE; ++e) {
                    out.a0 = __fadd_rn(out.a0, v[e].x);
                    out.a1 = __fadd_rn(out.a1, v[e].y);
                }
            }
            resolved = true;
        }
    }
    // a lane with a start completes the run coming from the left with its leading elements
    const FoldRun in{__shfl_up_sync(0xffffffffu, out.key, 1), __shfl_up_sync(0xffffffffu, out.a0, 1),
                     __shfl_up_sync(0xffffffffu, out.a1, 1)};
    if (lane > 0 && has_start && in.key != 0xFFFFFFFFu) {
        float a0 = in.a0, a1 = in.a1;
#pragma unroll
        for (int e = 0; e < kFoldE; ++e)
            if (e < fs) {
                a0 = __fadd_rn(a0, v[e].x);
                a1 = __fadd_rn(a1, v[e].y);
            }
        fold_flush(g_grid, sc, in.key, a0, a1);
    }
    // the run open at the window's end continues into the next window(s), up to its level's end
    if (lane == 31 && out.key != 0xFFFFFFFFu) {
        float a0 = out.a0, a1 = out.a1;
        for (uint64_t j = b + kFoldWin;; j += 4) {
            uint32_t kk[4];
            float2 vv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                kk[u] = j + u < m ? fold_offset(sc, sc.keys_sorted[j + u]) : 0xFFFFFFFFu;
                vv[u] = j + u < m ? sc.vals_sorted[j + u] : make_float2(0.0f, 0.0f);
            }
            bool more = true;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                more = more && kk[u] == out.key;
                if (more) {
                    a0 = __fadd_rn(a0, vv[u].x);
                    a1 = __fadd_rn(a1, vv[u].y);
                }
            }
            if (!more)
                break;
        }
        fold_flush(g_grid, sc, out.key, a0, a1);
    }
}

size_t grid_scatter_sort_bytes(uint64_t contributions, int end_bit) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (const unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                    (int64_t)contributions, 1, end_bit);
    return (bytes + 255) & ~(size_t)255;
}

// per level: stable sort of its segment by the bits [1, end_bit) of the level-local keys (the
// 0xFFFFFFFF sentinel of non-contributing slots sorts after the last entry) on the level's side
// stream, all levels concurrently; then one fold over the whole array
static cudaError_t grid_scatter_reduce(const GridScatter &sc, uint64_t m, uint64_t ngrid, float *g_grid,
                                       cudaStream_t stream) {
    (void)ngrid;
    cudaError_t e = cudaEventRecord(sc.fork, stream);
    for (int l = 0; l < sc.levels && e == cudaSuccess; ++l) {
        const uint64_t o = (uint64_t)l * sc.seg;
        e = cudaStreamWaitEvent(sc.side[l], sc.fork, 0);
        size_t tmp = sc.seg_tmp_bytes;
        if (e == cudaSuccess)
            e = cub::DeviceRadixSort::SortPairs(
                static_cast<uint8_t *>(sc.sort_tmp) + (size_t)l * sc.seg_tmp_bytes, tmp, sc.keys + o,
                sc.keys_sorted + o, reinterpret_cast<const unsigned long long *>(sc.vals + o),
                reinterpret_cast<unsigned long long *>(sc.vals_sorted + o), (int64_t)sc.seg, 1, sc.key_end_bit,
                sc.side[l]);
        if (e == cudaSuccess)
            e = cudaEventRecord(sc.join[l], sc.side[l]);
        if (e == cudaSuccess)
            e = cudaStreamWaitEvent(stream, sc.join[l], 0);
    }
    if (e != cudaSuccess)
        return e;
    const uint64_t warps = (m + kFoldWin - 1) / kFoldWin;
    grid_scatter_fold_kernel<<<(uint32_t)((warps + 7) / 8), 256, 0, stream>>>(sc, m, g_grid);
    return cudaGetLastError();
}

cudaError_t launch_stat_train(const TrainStepParams &p, float *partials, uint32_t dw_ctas, float *g_mlp,
                              double *loss_out, uint32_t *nonfinite, uint64_t ngrid, cudaStream_t stream) {
    const uint32_t blocks = (uint32_t)((p.n + 255) / 256);
    const size_t smem = (size_t)stat_param_count(p.in) * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(stat_fwd_bwd_fast_kernel<8, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(stat_fwd_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    const uint64_t m = p.n * (uint64_t)p.grid.levels * 8u;
    e = cudaMemsetAsync(p.scatter.keys, 0xFF, m * sizeof(uint32_t), stream);
    if (e != cudaSuccess)
        return e;
    if (p.grid.levels == 8 && p.in == 32)  // the default grid: compile-time widths
        stat_fwd_bwd_fast_kernel<8, 32><<<blocks, 256, smem, stream>>>(p);
    else
        stat_fwd_bwd_kernel<<<blocks, 256, smem, stream>>>(p);
    e = grid_scatter_reduce(p.scatter, m, ngrid, p.g_grid, stream);
    if (e != cudaSuccess)
        return e;
    const uint64_t per = (p.n + dw_ctas - 1) / dw_ctas;
    mlp_dw_kernel<kTOut><<<dw_ctas, 256, 0, stream>>>(p.ws, p.n, p.in, per, partials);
    stat_reduce_kernel<<<64, 256, 0, stream>>>(partials, (int)dw_ctas, stat_param_count(p.in), g_mlp, p.loss_parts,
                                               (int)blocks, p.inv_n, loss_out, p.g_grid, ngrid, nonfinite);
    return cudaGetLastError();
}

cudaError_t launch_rrs_train(const RrsStepParams &p, float *partials, uint32_t dw_ctas, float *g_mlp,
                             double *parts_out, uint32_t *nonfinite, uint64_t ngrid, cudaStream_t stream) {
    const uint32_t blocks = (uint32_t)((p.n + 255) / 256);
    const int gd = 2 * p.grid.levels;
    const size_t smem = (size_t)(rrs_w_offset(stat_param_count(gd + 16)) + mlp_params(p.in, 1)) * sizeof(float);
    const int fast = p.grid.levels != 8 ? -1 : (p.variant == 0 && p.in == 11 ? 0 : (p.variant == 1 && p.in == 32 ? 1 : -1));
    cudaError_t e = cudaFuncSetAttribute(rrs_fwd_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(rrs_fwd_bwd_fast_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(rrs_fwd_bwd_fast_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    const uint64_t m = p.n * (uint64_t)p.grid.levels * 8u;
    if (p.variant == 1 && p.g_grid) {
        e = cudaMemsetAsync(p.scatter.keys, 0xFF, m * sizeof(uint32_t), stream);
        if (e != cudaSuccess)
            return e;
    }
    if (fast == 0)
        rrs_fwd_bwd_fast_kernel<0><<<blocks, 256, smem, stream>>>(p);
    else if (fast == 1)
        rrs_fwd_bwd_fast_kernel<1><<<blocks, 256, smem, stream>>>(p);
    else
        rrs_fwd_bwd_kernel<<<blocks, 256, smem, stream>>>(p);
    if (p.variant == 1 && p.g_grid) {
        e = grid_scatter_reduce(p.scatter, m, ngrid, p.g_grid, stream);
        if (e != cudaSuccess)
            return e;
    }
    const uint64_t per = (p.n + dw_ctas - 1) / dw_ctas;
    mlp_dw_kernel<1><<<dw_ctas, 256, 0, stream>>>(p.ws, p.n, p.in, per, partials);
    rrs_reduce_kernel<<<64, 256, 0, stream>>>(partials, (int)dw_ctas, mlp_params(p.in, 1), g_mlp, p.parts,
                                              (int)blocks, parts_out, p.g_grid, ngrid, nonfinite);
    return cudaGetLastError();
}

cudaError_t launch_adam_ema(float *theta, const float *grad, float *m, float *v, float *shadow, uint64_t n,
                            const AdamParams &a, int num_sms, cudaStream_t stream) {
    if (n == 0)
        return cudaSuccess;
    const uint64_t want = (n + 255) / 256, cap = (uint64_t)num_sms * 8;
    adam_ema_kernel<<<(uint32_t)(want < cap ? want : cap), 256, 0, stream>>>(theta, grad, m, v, shadow, n, a);
    return cudaGetLastError();
}

}  // namespace nrrs
