// nrrs_film.cu -- the suffix side of trace_frame: the
// ordered film / parent folds, the reverse pass, TrainSample emission and the
// Film buffer updates, all bit-identical to the reference's sequential order.
//
//   fold_ordered_kernel  dst[key[i]] += term[i] in item order (f64); keys are
//                        non-decreasing (queue order is pixel and parent order,
//                        wavefront.cpp:253-268 / :421-425), so each key's run is
//                        folded by one thread in the reference's order:
//                        frame[pixel] += term (:299, :317, :355, :485),
//                        parent.s += term (:301, :319), reverse pass (:505-507)
//   emit_train_kernel    TrainSample per decided vertex with finite lo (:512-537),
//                        order-preserving (look-back scan), appended per depth
//   k_i kernels          per-pixel sample counts (:539-543)
//   film kernels         Film::add_frame / roll_acc (:104-116)
#include "nrrs_device.cuh"
#include "nrrs_internal.h"

#include <cuda_runtime.h>

namespace nrrs {

__global__ void __launch_bounds__(256) fold_ordered_kernel(double *dst, uint64_t n_dst, const int32_t *keys,
                                                           const double *terms, uint64_t n, uint32_t *err) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const int32_t key = keys[i];
    if (i > 0) {
        const int32_t prev = keys[i - 1];
        if (key < prev)
            atomicOr(err, 1u);  // not in queue order: the fold order would be undefined
        if (key == prev)
            return;             // not the first item of its run
    }
    if (key < 0)
        return;                 // no parent (camera ray): the reference skips it
    if ((uint64_t)key >= n_dst) {
        atomicOr(err, 2u);
        return;
    }
    double a0 = dst[3 * (uint64_t)key], a1 = dst[3 * (uint64_t)key + 1], a2 = dst[3 * (uint64_t)key + 2];
    for (uint64_t j = i; j < n && keys[j] == key; ++j) {  // sequential, in item order
        a0 = __dadd_rn(a0, terms[3 * j]);
        a1 = __dadd_rn(a1, terms[3 * j + 1]);
        a2 = __dadd_rn(a2, terms[3 * j + 2]);
    }
    dst[3 * (uint64_t)key] = a0;
    dst[3 * (uint64_t)key + 1] = a1;
    dst[3 * (uint64_t)key + 2] = a2;
}

// Film::add_frame: sum += frame, samples += 1, i_cur = float(frame).
__global__ void film_add_frame_kernel(double *sum, uint32_t *samples, float *i_cur, const double *frame, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double f = frame[3 * i + c];
            sum[3 * i + c] = __dadd_rn(sum[3 * i + c], f);
            i_cur[3 * i + c] = __double2float_rn(f);
        }
        samples[i] += 1u;
    }
}

// Film::roll_acc: i_acc = 0.5f * i_acc + 0.5f * i_cur (f32, no contraction).
__global__ void film_roll_acc_kernel(float *i_acc, const float *i_cur, uint64_t n3) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n3; i += (uint64_t)gridDim.x * blockDim.x)
        i_acc[i] = __fadd_rn(__fmul_rn(0.5f, i_acc[i]), __fmul_rn(0.5f, i_cur[i]));
}

// ---- TrainSample emission (one depth, order-preserving, appended) ----
constexpr int kET = 256;   // threads
constexpr int kEI = 4;     // items per thread
constexpr int kETile = kET * kEI;

__device__ __forceinline__ bool emit_lo(const TrainParams &p, uint64_t j, float lo[3], bool &nonfinite) {
    nonfinite = false;
    if (!p.decided[j])
        return false;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float w = p.weight[3 * j + c];
        // static_cast<float>(v.s[c] / v.weight[c]) for weight > 0, else 0 (wavefront.cpp:517-518)
        lo[c] = w > 0.0f ? __double2float_rn(__ddiv_rn(p.s[3 * j + c], (double)w)) : 0.0f;
    }
    if (!(isfinite(lo[0]) && isfinite(lo[1]) && isfinite(lo[2]))) {
        nonfinite = true;
        return false;
    }
    return true;
}

__global__ void __launch_bounds__(kET) emit_train_kernel(TrainParams p) {
    __shared__ uint32_t warp_tot[kET / 32];
    __shared__ unsigned long long prefix;
    __shared__ uint32_t tile_s, epoch_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0)
        tile_s = claim_tile_epoch(p.sync, &epoch_s);
    __syncthreads();
    const uint32_t tile = tile_s, epoch = epoch_s;
    const uint64_t first = (uint64_t)tile * kETile + (uint64_t)tid * kEI;
    float lo[kEI][3];
    uint32_t keep = 0, cnt = 0, nf = 0;
#pragma unroll
    for (int e = 0; e < kEI; ++e) {
        bool bad = false;
        if (first + e < p.n && emit_lo(p, first + e, lo[e], bad)) {
            keep |= 1u << e;
            ++cnt;
        }
        nf += bad ? 1u : 0u;
    }
    // block exclusive scan of the per-thread counts (thread order = vertex order)
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o)
            inc += t;
    }
    if (lane == 31)
        warp_tot[warp] = inc;
    nf = __reduce_add_sync(0xffffffffu, nf);
    if (lane == 0 && nf)
        atomicAdd(p.nonfinite, (unsigned long long)nf);
    __syncthreads();
    uint32_t before = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < kET / 32; ++w) {
        if (w < warp)
            before += warp_tot[w];
        agg += warp_tot[w];
    }
    if (warp == 0) {
        const uint64_t ex = lookback_warp(p.tile_state, tile, agg, epoch);
        if (lane == 0)
            prefix = ex;
    }
    __syncthreads();
    const uint64_t base = *p.base_in;
    uint64_t pos = base + prefix + before + inc - cnt;
#pragma unroll
    for (int e = 0; e < kEI; ++e) {
        if (!((keep >> e) & 1u))
            continue;
        const uint64_t j = first + e;
        if (pos >= p.capacity) {
            atomicOr(p.err, 4u);
            ++pos;
            continue;
        }
        nrrs_train_sample t;
        t.position[0] = p.p01[3 * j]; t.position[1] = p.p01[3 * j + 1]; t.position[2] = p.p01[3 * j + 2];
        t.omega_o[0] = p.wo01[2 * j]; t.omega_o[1] = p.wo01[2 * j + 1];
        t.roughness = p.roughness[j];
        t.t_x[0] = p.weight[3 * j]; t.t_x[1] = p.weight[3 * j + 1]; t.t_x[2] = p.weight[3 * j + 2];
        const uint32_t px = p.pixel[j];
        t.i_pixel[0] = p.i_acc[3 * (uint64_t)px]; t.i_pixel[1] = p.i_acc[3 * (uint64_t)px + 1];
        t.i_pixel[2] = p.i_acc[3 * (uint64_t)px + 2];
        t.lo_sample[0] = lo[e][0]; t.lo_sample[1] = lo[e][1]; t.lo_sample[2] = lo[e][2];
        t.q_norm = p.q_norm[j];
        t.q_real = p.q_real[j];
        t.pixel = px;
        t.k_i = 1.0f;  // set by the per-pixel count pass
        t.depth = (uint16_t)p.depth;
        t.pad = 0;
        p.out[pos] = t;
        ++pos;
    }
    if (tile == p.num_tiles - 1 && tid == 0)
        *p.base_out = base + prefix + agg;
    if (tid == 0)
        finish_launch(p.sync, p.tile_state, p.state_cap, epoch);
}

// k_i = number of this frame's samples with the sample's pixel (wavefront.cpp:539-543).
__global__ void k_i_count_kernel(const nrrs_train_sample *s, uint64_t start, const unsigned long long *end,
                                 uint64_t capacity, uint32_t *hist) {
    const uint64_t e = *end < capacity ? *end : capacity;
    for (uint64_t i = start + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e;
         i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(hist + s[i].pixel, 1u);
}

__global__ void k_i_assign_kernel(nrrs_train_sample *s, uint64_t start, const unsigned long long *end,
                                  uint64_t capacity, const uint32_t *hist) {
    const uint64_t e = *end < capacity ? *end : capacity;
    for (uint64_t i = start + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e;
         i += (uint64_t)gridDim.x * blockDim.x)
        s[i].k_i = (float)hist[s[i].pixel];
}

// ---- launchers ----
uint32_t emit_tiles(uint64_t n) { return (uint32_t)((n + kETile - 1) / kETile); }

cudaError_t launch_fold_ordered(double *dst, uint64_t n_dst, const int32_t *keys, const double *terms, uint64_t n,
                                uint32_t *err, cudaStream_t stream) {
    if (n == 0)
        return cudaSuccess;
    fold_ordered_kernel<<<(uint32_t)((n + 255) / 256), 256, 0, stream>>>(dst, n_dst, keys, terms, n, err);
    return cudaGetLastError();
}

cudaError_t launch_film_add_frame(double *sum, uint32_t *samples, float *i_cur, const double *frame, uint64_t n,
                                  int num_sms, cudaStream_t stream) {
    if (n == 0)
        return cudaSuccess;
    const uint64_t want = (n + 255) / 256, cap = (uint64_t)num_sms * 8;
    film_add_frame_kernel<<<(uint32_t)(want < cap ? want : cap), 256, 0, stream>>>(sum, samples, i_cur, frame, n);
    return cudaGetLastError();
}

cudaError_t launch_film_roll_acc(float *i_acc, const float *i_cur, uint64_t n, int num_sms, cudaStream_t stream) {
    if (n == 0)
        return cudaSuccess;
    const uint64_t want = (3 * n + 255) / 256, cap = (uint64_t)num_sms * 8;
    film_roll_acc_kernel<<<(uint32_t)(want < cap ? want : cap), 256, 0, stream>>>(i_acc, i_cur, 3 * n);
    return cudaGetLastError();
}

cudaError_t launch_emit_train(const TrainParams &p, cudaStream_t stream) {
    if (p.num_tiles == 0)
        return cudaSuccess;
    emit_train_kernel<<<p.num_tiles, kET, 0, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_k_i(nrrs_train_sample *s, uint64_t start, const unsigned long long *end, uint64_t capacity,
                       uint32_t *hist, uint32_t n_pixels, int num_sms, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)n_pixels * sizeof(uint32_t), stream);
    if (e != cudaSuccess)
        return e;
    const uint32_t grid = (uint32_t)num_sms * 4;
    k_i_count_kernel<<<grid, 256, 0, stream>>>(s, start, end, capacity, hist);
    k_i_assign_kernel<<<grid, 256, 0, stream>>>(s, start, end, capacity, hist);
    return cudaGetLastError();
}

}  // namespace nrrs
