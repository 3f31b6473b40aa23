// nrrs_kernels.cu -- sm_100a kernels of the NRRS per-bounce RRS stage.
//
//   K-A infer_ws_kernel<KIND> strategy factor per vertex (hash grid + tcgen05 MLP
//                            chain for the neural kinds), sanitize, RrsRound
//                            uniform, deterministic per-CTA double partial sums
//                            of q; the last CTA reduces them in fixed order.
//   K-B decide_kernel<SRC>   normalization (F from the rank sums), gain,
//                            stochastic rounding, single-pass decoupled
//                            look-back scan (u64), capacity clip, coalesced
//                            (parent, child) slot emission.
//   K-C compact_kernel<W,I>  order-preserving stream compaction of W-word
//                            records by a used mask, staged through smem.
//
// Reference: /root/reference/proj/src/wavefront.cpp:363-425 (+ :488-497),
// networks.cpp:131-281, hashgrid.cpp:38-82, mlp.cpp:52-72, rrs.cpp:8-45.
#include "nrrs_device.cuh"
#include "nrrs_internal.h"
#include "nrrs_ka.cuh"

#include <cuda_runtime.h>

#include <cstdlib>

namespace nrrs {

// ===========================================================================
// K-A: factor inference
//
// Heuristic factors (Fixed / Throughput, and depth 1) need no network: a plain
// streaming kernel, one thread per vertex.  The neural kinds run the
// warp-specialized tcgen05 pipeline further down (namespace ws).
// ===========================================================================
constexpr int kInferThreads = 256;    // heuristic kernel block

struct InferSmemHeader {
    uint32_t is_last;
    Fx128 warp_fx[8];
    uint32_t warp_cnt[8];
    uint32_t warp_bc[8];
};

// Position of entry e in the copy that pairs (e, e ^ (2^(t+1)-1)) into one
// aligned 16-byte pair (t = 0: the reference layout).  Mirrors pair_pos in
// nrrs_capi.cu (the host builds the copies at set_weights).
__device__ __forceinline__ uint32_t pair_pos(uint32_t e, uint32_t t) {
    const uint32_t G = 2u << t, i = e & (G - 1u), half = G >> 1;
    const uint32_t pi = i < half ? (i << 1) : (((G - 1u - i) << 1) | 1u);
    return (e & ~(G - 1u)) | pi;
}

// Table entry access for fp32 (float2, 8 B) or fp16 (half2, 4 B) grids: one
// gather returns the aligned entry pair (e, e^1) as (x0, y0, x1, y1).
template <bool kHalf>
struct GridTab {
    __device__ static __forceinline__ float4 pair(const void *base, uint64_t e_even) {
        if constexpr (kHalf) {
            const uint2 v = __ldg(reinterpret_cast<const uint2 *>(reinterpret_cast<const __half2 *>(base) + e_even));
            const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&v.x));
            const float2 b = __half22float2(*reinterpret_cast<const __half2 *>(&v.y));
            return make_float4(a.x, a.y, b.x, b.y);
        } else {
            return __ldg(reinterpret_cast<const float4 *>(reinterpret_cast<const float2 *>(base) + e_even));
        }
    }
    __device__ static __forceinline__ float2 one(const void *base, uint64_t e) {
        if constexpr (kHalf) {
            const uint32_t v = __ldg(reinterpret_cast<const uint32_t *>(reinterpret_cast<const __half2 *>(base) + e));
            return __half22float2(*reinterpret_cast<const __half2 *>(&v));
        } else {
            return __ldg(reinterpret_cast<const float2 *>(base) + e);
        }
    }
};

// HashGrid::encode (hashgrid.cpp:38-82) for levels [l0, l0+4) of one point, F = 2.
// Each cell edge (2 corners) costs one gather of an aligned entry pair from the
// matching table copy (GridDev); hashed x-edges with >= kPairCopies trailing ones
// in cx (1/32 of edges) fetch the second corner separately.
template <bool kHalf = false>
__device__ __forceinline__ void grid_encode4(const void *theta, const GridDev &g, int l0, float cpx, float cpy,
                                             float cpz, float *out) {
    using Tab = GridTab<kHalf>;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int l = l0 + i;
        if (l >= g.levels) {
            out[2 * i] = 0.0f;
            out[2 * i + 1] = 0.0f;
            continue;
        }
        const uint32_t res = (uint32_t)g.base_resolution << l;
        const float resf = (float)res;
        const float fx = cpx * resf, fy = cpy * resf, fz = cpz * resf;
        const uint32_t cx = min((uint32_t)fx, res - 1u);
        const uint32_t cy = min((uint32_t)fy, res - 1u);
        const uint32_t cz = min((uint32_t)fz, res - 1u);
        const float tx = fx - (float)cx, ty = fy - (float)cy, tz = fz - (float)cz;
        const float wx[2] = {1.0f - tx, tx}, wy[2] = {1.0f - ty, ty}, wz[2] = {1.0f - tz, tz};
        const uint64_t lb = (uint64_t)l * g.table_size;
        float a0 = 0.0f, a1 = 0.0f;
        if ((g.dense_mask >> l) & 1u) {
            // dense index (x*n + y)*n + z: edges along z; odd bases read the shifted copy
            const uint32_t nn = res + 1u;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t ox = e & 1, oy = e >> 1;
                const uint32_t e0 = ((cx + ox) * nn + cy + oy) * nn + cz;
                const uint32_t odd = e0 & 1u;
                const float4 pr = Tab::pair(theta, (odd ? g.copy_stride : 0) + lb + (e0 - odd));
                const float wxy = wx[ox] * wy[oy];
                a0 += wxy * wz[0] * pr.x + wxy * wz[1] * pr.z;
                a1 += wxy * wz[0] * pr.y + wxy * wz[1] * pr.w;
            }
        } else {
            // hashed index x ^ y*PY ^ z*PZ: edges along x, partner e ^ (2^(t+1)-1)
            const uint32_t tones = __ffs(~cx) - 1u;
            const uint32_t tc = tones >= g.pair_copies ? 0u : tones;
            const uint64_t tab = lb + (uint64_t)tc * g.copy_stride;
            const uint32_t yp[2] = {cy * 2654435761u, (cy + 1u) * 2654435761u};
            const uint32_t zp[2] = {cz * 805459861u, (cz + 1u) * 805459861u};
            const uint32_t m = g.table_size - 1u;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t oy = e & 1, oz = e >> 1;
                const uint32_t k = yp[oy] ^ zp[oz];
                const uint32_t e0 = (cx ^ k) & m;
                const uint32_t pos = pair_pos(e0, tc);
                const float4 pr = Tab::pair(theta, tab + (pos & ~1u));
                const bool sw = pos & 1u;
                const float v0x = sw ? pr.z : pr.x, v0y = sw ? pr.w : pr.y;
                float v1x = sw ? pr.x : pr.z, v1y = sw ? pr.y : pr.w;
                if (tones >= g.pair_copies) {
                    const float2 v = Tab::one(theta, lb + (((cx + 1u) ^ k) & m));
                    v1x = v.x;
                    v1y = v.y;
                }
                const float wyz = wy[oy] * wz[oz];
                a0 += wx[0] * wyz * v0x + wx[1] * wyz * v1x;
                a1 += wx[0] * wyz * v0y + wx[1] * wyz * v1y;
            }
        }
        out[2 * i] = a0;
        out[2 * i + 1] = a1;
    }
}

// ===========================================================================
// K-A0: level-sliced hash-grid encode (fp16 tables that fit in shared memory).
//
// Random 8-byte gathers from L2 run at ~1 per clock per SM (the L1TEX line
// lookup; profiles/r01_microbench_gather_bw.txt), which is what bounds the fused
// K-A.  Here each CTA owns ONE level: its table (T half2 entries, 128 KB at the
// default 2^15) is staged into shared memory once by TMA bulk copies, and the
// CTA encodes that level for a contiguous vertex range, 8 corner loads from
// smem per vertex.  CTA b serves level b % L on range b / L, so the L CTAs of
// one range run side by side and read the same p01 lines from L2.  Output:
// level planes feat[l][j] = (f0, f1) fp32, read back once by the groups of
// infer_aid_fused_kernel.  HashGrid::encode, hashgrid.cpp:38-82.
// ===========================================================================
constexpr int kLevelThreads = 1024;
#ifndef NRRS_LEVEL_PER_THREAD
#define NRRS_LEVEL_PER_THREAD 3
#endif
constexpr uint32_t kLevelPer = NRRS_LEVEL_PER_THREAD;             // vertices per thread per block
constexpr uint32_t kLevelBlock = kLevelPer * kLevelThreads;  // staged p01 block (12 B per vertex), double-buffered

// kF32: the fp32 StatNet grid, one (level, feature) table per CTA role (128 KB of fp32 at the default
// 2^15 entries, from the feature-major copy [level][feature][entry]); planes are then one float per
// (level, feature) and vertex.  Otherwise the fp16 AID grid, one level (both features) per role.
template <bool kF32>
__global__ void __launch_bounds__(kLevelThreads, 1) grid_level_kernel(GridLevelParams p) {
    extern __shared__ __align__(128) uint8_t lvl_smem[];
    __shared__ uint64_t bar[1];  // table landed
    pdl_trigger();  // K-A may start its prologue on SMs this kernel leaves
    const GridDev &g = p.g;
    const uint32_t L = (uint32_t)g.levels, R = kF32 ? 2u * L : L;  // CTA roles
    const uint32_t role = blockIdx.x % R, q = blockIdx.x / R;
    const uint32_t l = kF32 ? role >> 1 : role;
    const uint32_t nq = (gridDim.x - role + R - 1) / R;  // CTAs serving this role
    const uint32_t res = (uint32_t)g.base_resolution << l;
    const uint32_t nn = res + 1u;
    const bool dense = (g.dense_mask >> l) & 1u;
    const uint32_t entries = dense ? nn * nn * nn : g.table_size;
    const uint32_t bytes = (entries * 4u + 15u) & ~15u;
    const uint32_t tab_bytes = g.table_size * 4u;
    const uint64_t n = p.n;
    const uint64_t j0 = n * q / nq, j1 = n * (q + 1) / nq;  // this CTA's vertex range
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(&bar[0], bytes);
        const uint8_t *src = reinterpret_cast<const uint8_t *>(p.table) + (uint64_t)role * tab_bytes;
        for (uint32_t off = 0; off < bytes; off += 32768u)
            bulk_g2s(lvl_smem + off, src + off, bytes - off < 32768u ? bytes - off : 32768u, &bar[0]);
    }
    __syncthreads();
    LevelConsts c;
    c.res = res;
    c.nn = nn;
    c.m4 = (g.table_size - 1u) * 4u;
    c.resf = (float)res;
    c.dense = dense;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        c.doff4[k] = (((k & 1) * nn + ((k >> 1) & 1)) * nn + (k >> 2)) * 4u;
    // 32-bit offsets inside the CTA's range (a CTA serves < 2^32 vertices): the pointers advance once
    // per block and the bounds are one 32-bit compare per vertex
    const float *src3 = p.p01 + 3 * j0 + threadIdx.x * 3u;
    float2 *out = p.feat + (uint64_t)role * p.feat_stride + j0 + threadIdx.x;
    float *out1 = reinterpret_cast<float *>(p.feat) + (uint64_t)role * p.feat_stride + j0 + threadIdx.x;
    const uint32_t span = (uint32_t)(j1 - j0);
    // kLevelPer vertices per thread per block (t, t + 1024, ...); the next block's p01 is loaded
    // into registers before this block's gathers, so its L2 round trip hides behind them (no
    // shared-memory staging and no barrier in the loop: every thread owns its own vertices).
    float pv[kLevelPer][3];
    auto load_block = [&](uint32_t s) {  // s: block start relative to j0
        const float *g = src3 + 3u * s;
#pragma unroll
        for (int u = 0; u < (int)kLevelPer; ++u) {
            if (s + threadIdx.x + (uint32_t)u * kLevelThreads < span) {
                pv[u][0] = __ldg(g + 3u * u * kLevelThreads);
                pv[u][1] = __ldg(g + 3u * u * kLevelThreads + 1);
                pv[u][2] = __ldg(g + 3u * u * kLevelThreads + 2);
            } else {
                pv[u][0] = pv[u][1] = pv[u][2] = 0.0f;
            }
        }
    };
    load_block(0);
    mbar_wait(&bar[0], 0);
    for (uint32_t s = 0; s < span; s += kLevelBlock) {
        float cur[kLevelPer][3];
#pragma unroll
        for (int u = 0; u < (int)kLevelPer; ++u) {
            cur[u][0] = pv[u][0];
            cur[u][1] = pv[u][1];
            cur[u][2] = pv[u][2];
        }
        if (s + kLevelBlock < span)
            load_block(s + kLevelBlock);
        if constexpr (kF32) {
            float r[kLevelPer];
#pragma unroll
            for (int u = 0; u < (int)kLevelPer; ++u)
                r[u] = level_encode_f32(lvl_smem, c, cur[u][0], cur[u][1], cur[u][2]);
#pragma unroll
            for (int u = 0; u < (int)kLevelPer; ++u)
                if (s + threadIdx.x + (uint32_t)u * kLevelThreads < span)
                    __stcs(out1 + s + (uint32_t)u * kLevelThreads, r[u]);
        } else {
            float2 r[kLevelPer];
#pragma unroll
            for (int u = 0; u < (int)kLevelPer; ++u)
                r[u] = level_encode(lvl_smem, c, cur[u][0], cur[u][1], cur[u][2]);
#pragma unroll
            for (int u = 0; u < (int)kLevelPer; ++u)
                if (s + threadIdx.x + (uint32_t)u * kLevelThreads < span)
                    __stcs(out + s + (uint32_t)u * kLevelThreads, r[u]);
        }
    }
}

// nrrs_gpu_sharded_clip on the device (one thread): the rank's global slot base, kept records,
// global spawned and dropped from the all-gathered rank totals (wavefront.cpp:141-154 across ranks).
__global__ void sharded_clip_kernel(const unsigned long long *totals, int nranks, int rank, uint32_t capacity,
                                    unsigned long long *out) {
    if (threadIdx.x != 0 || blockIdx.x != 0)
        return;
    unsigned long long base = 0, all = 0;
    for (int r = 0; r < nranks; ++r) {
        if (r < rank)
            base += totals[r];
        all += totals[r];
    }
    const unsigned long long cap = capacity;
    const unsigned long long room = cap - (base < cap ? base : cap);
    const unsigned long long kept = totals[rank] < room ? totals[rank] : room;
    const unsigned long long spawned = all < cap ? all : cap;
    out[0] = base;
    out[1] = kept;
    out[2] = spawned;
    out[3] = all - spawned;
}

// PDL launches (default; env NRRS_NO_PDL at context creation turns them off): K-A after K-A0, K-B
// after K-A, K-C after K-B, so each kernel's launch and prologue overlap its predecessor's tail
// (AID stage 0.2274 -> 0.2195 ms in an interleaved A/B).
static bool g_pdl = false;
void set_pdl(bool on) { g_pdl = on; }
template <typename K, typename P>
static cudaError_t launch_maybe_pdl(K kernel, uint32_t grid, uint32_t block, size_t smem, cudaStream_t stream,
                                    const P &p) {
    if (!g_pdl) {
        kernel<<<grid, block, smem, stream>>>(p);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, p);
}

// Mailbox mode of sharded_clip_kernel: the rank totals come from the own mailbox (kind 1).
__global__ void mbox_clip_kernel(const MboxDev *m, uint32_t capacity, unsigned long long *out, double *sums_out,
                                 unsigned long long *totals_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0)
        return;
    unsigned long long base = 0, all = 0, mine = 0;
    mbox_wait(m, 1, [&](int r, unsigned long long t, unsigned long long) {
        if (r < m->rank)
            base += t;
        if (r == m->rank)
            mine = t;
        all += t;
        m->totals_seen[r] = t;
    });
    const unsigned long long cap = capacity;
    const unsigned long long room = cap - (base < cap ? base : cap);
    const unsigned long long kept = mine < room ? mine : room;
    const unsigned long long spawned = all < cap ? all : cap;
    out[0] = base;
    out[1] = kept;
    out[2] = spawned;
    out[3] = all - spawned;
    for (int r = 0; r < m->nranks; ++r) {  // the depth's rank sums (decide3 kept them) and totals
        if (sums_out)
            sums_out[r] = m->sums_seen[r];
        if (totals_out)
            totals_out[r] = m->totals_seen[r];
    }
}

__global__ void mbox_publish_kernel(const MboxDev *m, int kind, unsigned long long value) {
    if (threadIdx.x == 0 && blockIdx.x == 0)
        mbox_publish(m, kind, value, 0ull);  // an empty rank: total 0 / exact sum 0
}

cudaError_t launch_mbox_publish(const MboxDev *m, int kind, unsigned long long value, cudaStream_t stream) {
    mbox_publish_kernel<<<1, 32, 0, stream>>>(m, kind, value);
    return cudaGetLastError();
}

cudaError_t launch_mbox_clip(const MboxDev *m, uint32_t capacity, unsigned long long *out, double *sums_out,
                             unsigned long long *totals_out, cudaStream_t stream) {
    mbox_clip_kernel<<<1, 32, 0, stream>>>(m, capacity, out, sums_out, totals_out);
    return cudaGetLastError();
}

cudaError_t launch_sharded_clip(const unsigned long long *totals, int nranks, int rank, uint32_t capacity,
                                unsigned long long *out, cudaStream_t stream) {
    sharded_clip_kernel<<<1, 32, 0, stream>>>(totals, nranks, rank, capacity, out);
    return cudaGetLastError();
}

template <bool kF32>
static cudaError_t launch_grid_levels_t(const GridLevelParams &p, int num_sms, cudaStream_t stream) {
    const uint32_t R = (kF32 ? 2u : 1u) * (uint32_t)p.g.levels;
    const size_t smem = (size_t)p.g.table_size * 4u;
    cudaError_t e =
        cudaFuncSetAttribute(grid_level_kernel<kF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    // one CTA per SM; every role (level, or level x feature) gets floor or ceil of num_sms / R CTAs
    uint64_t grid = (uint64_t)num_sms < R ? R : (uint64_t)num_sms;
    const uint64_t max_useful = R * ((p.n + kLevelThreads - 1) / kLevelThreads);
    if (grid > max_useful)
        grid = max_useful < R ? R : max_useful;
    grid_level_kernel<kF32><<<(uint32_t)grid, kLevelThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_grid_levels(const GridLevelParams &p, int num_sms, cudaStream_t stream) {
    return p.f32 ? launch_grid_levels_t<true>(p, num_sms, stream) : launch_grid_levels_t<false>(p, num_sms, stream);
}

__global__ void __launch_bounds__(kInferThreads, 8) infer_kernel(InferParams p) {
    __shared__ InferSmemHeader hdr_s;
    pdl_trigger();
    InferSmemHeader *hdr = &hdr_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t n = p.n;
    // per-thread accumulators, reduced once per CTA in a fixed order (deterministic)
    Fx128 my_fx{0ull, 0ull};  // exact sum of q (fixed point)
    uint32_t my_nonfinite = 0;
    const uint32_t my_bc = 0;
    const bool depth1 = p.depth == 1u;
    for (uint64_t j = (uint64_t)blockIdx.x * kInferThreads + tid; j < n; j += (uint64_t)gridDim.x * kInferThreads) {
        const float wx = __ldg(p.weight + 3 * j), wy = __ldg(p.weight + 3 * j + 1), wz = __ldg(p.weight + 3 * j + 2);
        const float lum_w = luminance(wx, wy, wz);
        // Mix-Depth gate + zero-throughput skip (wavefront.cpp:373-380)
        const bool active = p.gate ? (!depth1 && lum_w > 0.0f) : true;
        float q = p.heur_kind == 0 ? p.fixed_value                 // Fixed (wavefront.cpp:193-194)
                                   : (lum_w < 1.0f ? lum_w : 1.0f);  // std::min(1, lum) (rrs.hpp:49-51)
        uint32_t decided = active ? 1u : 0u;
        if (p.gate) {
            if (depth1)
                q = 1.0f;  // depth-1 pin (wavefront.cpp:373-375)
            if (!active && !depth1)
                q = 0.0f;
            decided = (depth1 || active) ? 1u : 0u;
            if (!isfinite(q) || q < 0.0f) {  // sanitize (wavefront.cpp:381-385)
                q = 0.0f;
                decided = 0;
                ++my_nonfinite;
            }
        }
        p.q_out[j] = q;
        if (p.u_out)
            p.u_out[j] = rrs_uniform(p.mixed_seed, __ldg(p.path_key + j), p.depth);
        if (p.decided_out)
            p.decided_out[j] = (uint8_t)decided;
        fx_add_q(my_fx, q);
    }

    if (p.parts == nullptr)
        return;
    // ---- CTA sum in a fixed tree, then last-CTA-done reduction in CTA order ----
    constexpr int kWarps = kInferThreads / 32;
    {
        const Fx128 s = fx_warp_sum(my_fx);
        const uint32_t nf = __reduce_add_sync(0xffffffffu, my_nonfinite);
        const uint32_t bcs = __reduce_add_sync(0xffffffffu, my_bc);
        if (lane == 0) {
            hdr->warp_fx[warp] = s;
            hdr->warp_cnt[warp] = nf;
            hdr->warp_bc[warp] = bcs;
        }
        __syncthreads();
    }
    if (tid == 0) {
        Fx128 cs{0ull, 0ull};
        uint32_t cn = 0, cb = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            fx_add(cs, hdr->warp_fx[w]);
            cn += hdr->warp_cnt[w];
            cb += hdr->warp_bc[w];
        }
        reinterpret_cast<Fx128 *>(p.parts)[blockIdx.x] = cs;
        p.part_counts[2 * blockIdx.x] = cn;
        p.part_counts[2 * blockIdx.x + 1] = cb;
        __threadfence();
        const uint32_t prev = atomicAdd(p.counter, 1u);
        hdr->is_last = (prev == gridDim.x - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (!hdr->is_last)
        return;
    __threadfence();
    Fx128 s{0ull, 0ull};
    uint32_t nf = 0, bcs = 0;
    for (uint32_t b = tid; b < gridDim.x; b += kInferThreads) {
        const unsigned long long *pp = reinterpret_cast<const unsigned long long *>(p.parts) + 2 * b;
        fx_add(s, Fx128{__ldcg(pp), __ldcg(pp + 1)});
        nf += __ldcg(p.part_counts + 2 * b);
        bcs += __ldcg(p.part_counts + 2 * b + 1);
    }
    s = fx_warp_sum(s);
    nf = __reduce_add_sync(0xffffffffu, nf);
    bcs = __reduce_add_sync(0xffffffffu, bcs);
    __syncthreads();
    if (lane == 0) {
        hdr->warp_fx[warp] = s;
        hdr->warp_cnt[warp] = nf;
        hdr->warp_bc[warp] = bcs;
    }
    __syncthreads();
    if (tid == 0) {
        Fx128 fx{0ull, 0ull};
        unsigned long long tn = 0, tb = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            fx_add(fx, hdr->warp_fx[w]);
            tn += hdr->warp_cnt[w];
            tb += hdr->warp_bc[w];
        }
        const double total = fx_finish(p, fx);
        *p.sum_out = total;
        if (p.mbox)  // sharded mailbox mode: this rank's sum to every rank
            mbox_publish(p.mbox, 0, p.res->sum_fx[0], p.res->sum_fx[1]);  // the exact 128-bit sum
        if (p.accumulate) {
            p.res->sum_q = total;  // the running exact total (fx_finish)
            p.res->nonfinite += tn;
            p.res->box_cox_clamps += tb;
        } else {
            p.res->sum_q = total;
            p.res->nonfinite = tn;
            p.res->box_cox_clamps = tb;
        }
        *p.counter = 0;  // self-cleaning for the next launch
    }
}

// Teardown shared by the persistent K-A kernels: the CTA's exact sum of q (Fx128) and its
// non-finite / Box-Cox-clamp counts as one partial per CTA, then the last CTA to finish reduces the
// partials (exact, so order-free), converts the call's running total (fx_finish) and writes sum_out,
// the result counters and, in sharded mailbox mode, the rank's exact sum to every rank.  Called by
// every thread of the CTA after its last tile.
template <int kWarps>
__device__ __forceinline__ void ka_reduce_finish(const InferParams &p, ws::SmemTail *st, const Fx128 &my_fx,
                                                 uint32_t my_nonfinite, uint32_t my_bc) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    {
        const Fx128 sv = fx_warp_sum(my_fx);
        const uint32_t nf = __reduce_add_sync(0xffffffffu, my_nonfinite);
        const uint32_t bcs = __reduce_add_sync(0xffffffffu, my_bc);
        if (lane == 0) {
            st->red_fx[warp] = sv;
            st->red_nf[warp] = nf;
            st->red_bc[warp] = bcs;
        }
        __syncthreads();
    }
    if (tid == 0) {
        Fx128 cs{0ull, 0ull};
        uint32_t cn = 0, cb = 0;
        for (int w = 0; w < kWarps; ++w) {
            fx_add(cs, st->red_fx[w]);
            cn += st->red_nf[w];
            cb += st->red_bc[w];
        }
        reinterpret_cast<Fx128 *>(p.parts)[blockIdx.x] = cs;
        p.part_counts[2 * blockIdx.x] = cn;
        p.part_counts[2 * blockIdx.x + 1] = cb;
        __threadfence();
        st->is_last = atomicAdd(p.counter, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (!st->is_last)
        return;
    __threadfence();
    if (warp == 0) {
        Fx128 sv{0ull, 0ull};
        uint32_t nf = 0, bcs = 0;
        for (uint32_t b = lane; b < gridDim.x; b += 32) {
            const unsigned long long *pp = reinterpret_cast<const unsigned long long *>(p.parts) + 2 * b;
            fx_add(sv, Fx128{__ldcg(pp), __ldcg(pp + 1)});
            nf += __ldcg(p.part_counts + 2 * b);
            bcs += __ldcg(p.part_counts + 2 * b + 1);
        }
        sv = fx_warp_sum(sv);
        nf = __reduce_add_sync(0xffffffffu, nf);
        bcs = __reduce_add_sync(0xffffffffu, bcs);
        if (lane == 0) {
            const double tot = fx_finish(p, sv);
            *p.sum_out = tot;
            if (p.mbox)  // sharded mailbox mode: this rank's exact 128-bit sum to every rank
                mbox_publish(p.mbox, 0, p.res->sum_fx[0], p.res->sum_fx[1]);
            p.res->sum_q = tot;  // the running exact total (fx_finish)
            if (p.accumulate) {
                p.res->nonfinite += nf;
                p.res->box_cox_clamps += bcs;
            } else {
                p.res->nonfinite = nf;
                p.res->box_cox_clamps = bcs;
            }
            *p.counter = 0;  // self-cleaning for the next launch
        }
    }
}

// ===========================================================================
// K-A (neural kinds): warp-specialized persistent pipeline, 1 CTA per SM.
//
//  encoder group e (8 warps, 2 threads per tile row, half h):
//     inputs -> hash-grid levels [4h,4h+4) + tail[8h,8h+8) -> tcgen05.st into
//     TMEM A-slot s (hi | lo) + per-row sidecar (path key, flags, extras) in
//     smem -> arrive full[s]
//  MLP group g (4 warps, 1 thread per tile row, own D / A_hid / MMA mbarrier):
//     wait full[s] -> layer chain (A from TMEM, weights in smem, 3-term split,
//     bias via the ones slice) -> q / outputs -> arrive empty[s]
//  Tiles are taken in order: encoder e owns local tiles i = e (mod GE), MLP
//  group g owns i = g (mod GM), slot s = i mod S.  Gathers of tile i+1.. run
//  while MLP groups chain tiles i, i-1.
// ===========================================================================

// Per-phase cycle counters and the CTA-0 tile timeline (NRRS_DEBUG_TIMING on the
// host) exist only in builds with -DNRRS_KERNEL_TIMING: they cost registers.
#ifdef NRRS_KERNEL_TIMING
constexpr bool kTiming = true;
#else
constexpr bool kTiming = false;
#endif

// HALF: fp16 RRSNet (AID) grid tables.
template <int KIND, int GE, int GM, int P, int TPR, bool HALF>
__global__ void __launch_bounds__(ws::Cfg<GE, GM, P, TPR>::kThreads, 1) infer_ws_kernel(InferParams p) {
    using Cfg = ws::Cfg<GE, GM, P, TPR>;
    constexpr uint32_t kGT = Cfg::kGroupThreads;
    constexpr int S = Cfg::kSlots;
    constexpr int kNL = KIND == kKindNrrs ? 8 : 4;  // MMA layers per tile (NRRS: StatNet then RRSNet)
    unsigned long long g_start = 0, c_start = 0;
    if (kTiming && p.dbg && threadIdx.x == 0) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
        c_start = clock64();
    }
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem_w = smem_raw;
    ws::Side *side = reinterpret_cast<ws::Side *>(smem_raw + ((p.blob_bytes + 127u) & ~127u));
    ws::SmemTail *st = reinterpret_cast<ws::SmemTail *>(reinterpret_cast<uint8_t *>(side) + S * 128 * sizeof(ws::Side));
    const int tid = threadIdx.x, warp = tid >> 5;

    // ---- setup: weights -> smem, UMMA descriptors, barriers, TMEM (all 512 columns) ----
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(p.blob);
        uint4 *dst = reinterpret_cast<uint4 *>(smem_w);
        for (uint32_t i = tid; i < p.blob_bytes / 16u; i += Cfg::kThreads)
            dst[i] = __ldg(src + i);
    }
    if (tid == 0) {
        for (int net = 0; net < 2; ++net) {
            const NetDesc &nd = net == 0 ? p.nets.stat : p.nets.rrs;
            for (int l = 0; l < 4; ++l) {
                const LayerDesc &L = nd.layer[l];
                st->idesc_n[net][l] = make_idesc_f16(L.N);
                st->idesc_2n[net][l] = make_idesc_f16(2u * L.N);
                st->nslices[net][l] = (uint32_t)L.K / 16u;
                st->bias[net][l] = L.bias;
                const uint32_t sbo = (uint32_t)L.K * 16u;
                for (int k = 0; k < 2; ++k) {
                    st->wdesc[net][l][k] = make_smem_desc(smem_u32(smem_w + L.w_hi) + 256u * k, 128u, sbo);
                    st->wdesc_lo[net][l][k] =
                        make_smem_desc(smem_u32(smem_w + L.w_hi) + 256u * k + ((uint32_t)L.N / 8u) * sbo, 128u, sbo);
                }
            }
        }
        for (int q = 0; q < S; ++q) {
            mbar_init(&st->full[q], 256);
            mbar_init(&st->empty[q], kGT);
        }
        for (int q = 0; q < Cfg::kChains; ++q)
            mbar_init(&st->mma_bar[q], 1);
        fence_barrier_init();
    }
    if (warp == 0)
        tmem_alloc(&st->tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_trigger();  // K-B (PDL launch) may start on SMs this kernel leaves
    const uint32_t tmem_base = st->tmem_base;
    const uint32_t lane_base = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
    if (kTiming && p.dbg && tid == 0)
        p.dbg[blockIdx.x * 32 + 3] = clock64() - c_start;  // setup cycles

    const uint64_t n = p.n;
    const uint64_t num_tiles = (n + kTileM - 1) / kTileM;
    const uint64_t t_begin = num_tiles * blockIdx.x / gridDim.x;
    const uint64_t t_end = num_tiles * (blockIdx.x + 1) / gridDim.x;
    const uint32_t T = (uint32_t)(t_end - t_begin);
    Fx128 my_fx{0ull, 0ull};  // exact sum of q (fixed point)
    uint32_t my_nonfinite = 0, my_bc = 0;
    const bool depth1 = p.depth == 1u;

    if (tid < Cfg::kEncThreads) {
        // ============================== encoder ==============================
        const int e = tid >> 8;                 // encoder group
        const int r = tid & 127, half = (tid >> 7) & 1;
        const bool rec = kTiming && p.dbg && (tid & 255) == 0;
        unsigned long long c_empty = 0, c_enc = 0, c_st = 0, t0 = 0;
        for (uint32_t i = (uint32_t)e; i < T; i += GE) {
            const uint32_t s = i % S;
            if (rec) t0 = clock64();
            if (i >= (uint32_t)S)
            {
#if NRRS_ENC_ONE_POLLER
                // one warp polls the slot, the group's other warps block in bar.sync (no issue slots)
                if ((tid & 255) < 32)
                    mbar_wait_sleep(&st->empty[s], ((i / S) - 1u) & 1u, 1000u);
                named_bar_sync(1u + (uint32_t)GM + (uint32_t)e, 256u);
#else
                mbar_wait_sleep(&st->empty[s], ((i / S) - 1u) & 1u, 1000u);
#endif
            }
            if (rec) { const unsigned long long t1 = clock64(); c_empty += t1 - t0; t0 = t1; }
            const uint64_t j = (t_begin + i) * kTileM + r;
            const bool valid = j < n;
            float px = 0, py = 0, pz = 0, wx = 0, wy = 0, wz = 0, rough = 0;
            if (valid) {
                px = __ldg(p.p01 + 3 * j); py = __ldg(p.p01 + 3 * j + 1); pz = __ldg(p.p01 + 3 * j + 2);
                wx = __ldg(p.weight + 3 * j); wy = __ldg(p.weight + 3 * j + 1); wz = __ldg(p.weight + 3 * j + 2);
                rough = __ldg(p.roughness + j);
            }
            const bool active = valid && (p.gate ? (!depth1 && luminance(wx, wy, wz) > 0.0f) : true);
            auto load_ipix = [&](float &a, float &b, float &c) {
                a = b = c = 0.0f;
                if (!valid)
                    return;
                if (p.i_pixel) {
                    a = __ldg(p.i_pixel + 3 * j); b = __ldg(p.i_pixel + 3 * j + 1); c = __ldg(p.i_pixel + 3 * j + 2);
                } else {
                    const uint64_t px_idx = __ldg(p.pixel + j);
                    a = __ldg(p.i_acc + 3 * px_idx); b = __ldg(p.i_acc + 3 * px_idx + 1); c = __ldg(p.i_acc + 3 * px_idx + 2);
                }
            };
            float in16[16];
            float *g8 = in16, *t8 = in16 + 8;
            uint32_t bc = 0;
            if (kTiming && (p.ablate & 1u)) {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    g8[q] = px * (float)(q + 1) + py;
            } else if (KIND == kKindAid) {
                grid_encode4<HALF>(p.rrs_grid, p.grid_rrs, 4 * half, clamp01(px), clamp01(py), clamp01(pz), g8);
            } else {
                grid_encode4<false>(p.stat_grid, p.grid, 4 * half, clamp01(px), clamp01(py), clamp01(pz), g8);
            }
            ws::Side sd{};
            if (half == 0) {
                const float wox = valid ? __ldg(p.wo01 + 2 * j) : 0.0f;
                const float woy = valid ? __ldg(p.wo01 + 2 * j + 1) : 0.0f;
                one_blob_fast<4>(wox, t8);
                one_blob_fast<4>(woy, t8 + 4);
                sd.key = valid && KIND != kKindStats ? __ldg(p.path_key + j) : 0ull;
                sd.flags = (valid ? 1u : 0u) | (active ? 2u : 0u);
                if (KIND == kKindNrrs) {
                    float ipx, ipy, ipz;
                    load_ipix(ipx, ipy, ipz);
                    sd.ex[0] = box_cox_fast(wx, bc);
                    sd.ex[1] = box_cox_fast(wy, bc);
                    sd.ex[2] = box_cox_fast(wz, bc);
                    sd.ex[3] = box_cox_fast(mean3_fast(ipx, ipy, ipz), bc);
                    sd.ex[4] = remap_fast(rough);
                } else if (KIND == kKindAdrrs) {
                    float ipx, ipy, ipz;
                    load_ipix(ipx, ipy, ipz);
                    sd.ex[0] = wx;
                    sd.ex[1] = wy;
                    sd.ex[2] = wz;
                    sd.ex[3] = luminance(ipx, ipy, ipz);
                }
            } else if (KIND == kKindAid) {
                float ipx, ipy, ipz;
                load_ipix(ipx, ipy, ipz);
                t8[0] = box_cox_fast(wx, bc);
                t8[1] = box_cox_fast(wy, bc);
                t8[2] = box_cox_fast(wz, bc);
                t8[3] = box_cox_fast(mean3_fast(ipx, ipy, ipz), bc);
                one_blob_fast<4>(remap_fast(rough), t8 + 4);
            } else {
                one_blob_fast<8>(remap_fast(rough), t8);
            }
            if (!valid) {
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    in16[q] = 0.0f;
            }
            if (active)
                my_bc += bc;
            if (rec) { const unsigned long long t1 = clock64(); c_enc += t1 - t0; t0 = t1; }
            const uint32_t col = Cfg::kColSlots + 32u * s;
            uint32_t hw[8], lw[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                split2(in16[2 * q], in16[2 * q + 1], hw[q], lw[q]);
            tmem_st8(lane_base + col + 8u * half, hw);
            tmem_st8(lane_base + col + 16u + 8u * half, lw);
            if (half == 0)
                side[s * 128 + r] = sd;
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&st->full[s]);
            if (rec) c_st += clock64() - t0;
            if (kTiming && p.dbg && blockIdx.x == 0 && (tid & 255) == 0 && i < 1024)
                p.dbg[8192 + 4 * i] = clock64();  // timeline (CTA 0): tile i input ready
            if (kTiming && p.dbg && tid == 0) p.dbg[blockIdx.x * 32 + 18] = clock64();  // encoder 0: last full arrive
            if (kTiming && p.dbg && tid == 256) p.dbg[blockIdx.x * 32 + 19] = clock64();  // encoder 1: last full arrive
        }
        if (kTiming && p.dbg && tid == 0)
            p.dbg[blockIdx.x * 32 + 7] = clock64() - c_start;  // encoder group 0 loop end
        if (rec) {
            p.dbg[blockIdx.x * 32 + 4 * e + 0] = c_empty;
            p.dbg[blockIdx.x * 32 + 4 * e + 1] = c_enc;
            p.dbg[blockIdx.x * 32 + 4 * e + 2] = c_st;
        }
    } else {
        // ================================ MLP ================================
        // Group g runs P tile chains in lockstep, layer by layer: while chain c's
        // MMA is in flight the group drains the other chains' accumulators.
        const int mt = tid - Cfg::kEncThreads;
        const int g = mt / (int)kGT, gt = mt % (int)kGT, r = gt & 127, mh = gt >> 7;  // mh: column half (TPR 2)
        const bool issuer = gt == 0;
        const uint32_t bar_id = 1u + (uint32_t)g;
        uint32_t phases = 0;  // bit c: parity of chain c's mbarrier
        const bool rec = kTiming && p.dbg && issuer;
        unsigned long long c_wait = 0, c_epi = 0, t0 = 0;
        for (uint32_t base = 0; base < T; base += Cfg::kChains) {
            uint32_t tile[P], slot[P];
            bool live[P];
#pragma unroll
            for (int c = 0; c < P; ++c) {
                tile[c] = base + (uint32_t)(c * GM + g);
                live[c] = tile[c] < T;
                slot[c] = tile[c] % S;
            }
            if (!live[0])
                break;
            // layer 0 of every chain as soon as its input slot is full
            if (rec && g == 0) p.dbg[blockIdx.x * 32 + 16] = clock64() - 0;  // last tile: wait start
            if (rec && blockIdx.x == 0 && tile[0] < 1024) p.dbg[8192 + 4 * tile[0] + 1] = clock64();  // MLP tile start
            tc_fence_before();
            named_bar_sync(bar_id, kGT);
#pragma unroll
            for (int c = 0; c < P; ++c) {
                if (!live[c])
                    continue;
                if (issuer)  // only the MMA issuer needs the input slot; the group waits on the MMA
                    mbar_wait_sleep(&st->full[slot[c]], (tile[c] / S) & 1u, 1000u);
                if (rec && g == 0) p.dbg[blockIdx.x * 32 + 17] = clock64();  // last tile: full passed
                if (rec && blockIdx.x == 0 && tile[c] < 1024) p.dbg[8192 + 4 * tile[c] + 2] = clock64();
                if (issuer)
                    ws::ws_issue(st, KIND == kKindAid ? 1 : 0, 0, tmem_base, Cfg::kColSlots + 32u * slot[c],
                                 Cfg::kColD + ws::kDCols * (uint32_t)(g * P + c), &st->mma_bar[g * P + c]);
            }
#pragma unroll 1
            for (int l = 0; l < kNL; ++l) {  // layer l just issued for every live chain
#pragma unroll
                for (int c = 0; c < P; ++c) {
                    if (!live[c])
                        continue;
                    const int q = g * P + c;
                    const uint32_t col_d = Cfg::kColD + ws::kDCols * (uint32_t)q;
                    const uint32_t col_a = Cfg::kColSlots + 32u * slot[c];
                    if (rec) t0 = clock64();
#if NRRS_MMA_WAIT_HINT
                    mbar_wait_sleep(&st->mma_bar[q], (phases >> c) & 1u, NRRS_MMA_WAIT_HINT);
#else
                    mbar_wait(&st->mma_bar[q], (phases >> c) & 1u);
#endif
                    phases ^= 1u << c;
                    tc_fence_after();
                    if (rec) { const unsigned long long t1 = clock64(); c_wait += t1 - t0; t0 = t1; }
                    const int lyr = l & 3;
                    const bool head = lyr == 3;
                    const int net = (KIND == kKindAid || l >= 4) ? 1 : 0;
                    const uint32_t boff = st->bias[net][lyr];
                    const float *bias = boff == kNoBias ? nullptr : reinterpret_cast<const float *>(smem_w + boff);
                    if (!head) {
                        // z = D_hi + D_lo + bias -> leaky ReLU -> next A (hi/lo), 16 columns at a time
#pragma unroll
                        for (int hh = 0; hh < 2 / TPR; ++hh) {
                            const int h = TPR == 1 ? hh : mh;
                            float z[16];
                            ws::ws_load_sum16(lane_base, col_d, 32u, 16u * (uint32_t)h, bias, z);
#pragma unroll
                            for (int i = 0; i < 8; ++i) {  // leaky ReLU = cwiseMax(z, slope z)
                                const float2 t = upk2(fmul2(pk2(z[2 * i], z[2 * i + 1]), pk2(0.01f, 0.01f)));
                                z[2 * i] = fmaxf(z[2 * i], t.x);
                                z[2 * i + 1] = fmaxf(z[2 * i + 1], t.y);
                            }
                            ws::ws_store_a16(lane_base, col_a, h, z);
                        }
                        tmem_wait_st();
                        tc_fence_before();
                        named_bar_sync(bar_id, kGT);
                        if (issuer)
                            ws::ws_issue(st, net, lyr + 1, tmem_base, col_a, col_d, &st->mma_bar[q]);
                    } else if (mh != 0) {
                        // TPR 2, second column half: no head work; keep the group's barrier count
                        if (KIND == kKindNrrs && l == 3) {
                            tc_fence_before();
                            named_bar_sync(bar_id, kGT);
                        } else {
                            mbar_arrive(&st->empty[slot[c]]);
                        }
                    } else {
                        float y[16];
                        ws::ws_load_sum16(lane_base, col_d, 16u, 0u, bias, y);  // head: N = 16
                        mbar_wait(&st->full[slot[c]], (tile[c] / S) & 1u);  // sidecar visibility
                        const ws::Side sd = side[slot[c] * 128 + r];
                        const bool valid = sd.flags & 1u, active = (sd.flags >> 1) & 1u;
                        const uint64_t j = (t_begin + tile[c]) * kTileM + r;
                        if (KIND == kKindNrrs && l == 3) {
                            // stats -> build_nrrs_input (networks.cpp:137-147) -> RRSNet layer 0
                            float xin[16];
                            uint32_t bc = 0;
#pragma unroll
                            for (int k = 0; k < 6; ++k)
                                xin[k] = box_cox_fast(y[k], bc);
#pragma unroll
                            for (int k = 0; k < 5; ++k)
                                xin[6 + k] = sd.ex[k];
                            xin[11] = 1.0f;  // bias column of the RRSNet first layer
#pragma unroll
                            for (int k = 12; k < 16; ++k)
                                xin[k] = 0.0f;
                            if (!valid) {
#pragma unroll
                                for (int k = 0; k < 11; ++k)
                                    xin[k] = 0.0f;
                            }
                            if (active)
                                my_bc += bc;
                            uint32_t hw[8], lw[8];
#pragma unroll
                            for (int k = 0; k < 8; ++k)
                                split2(xin[2 * k], xin[2 * k + 1], hw[k], lw[k]);
                            tmem_st8(lane_base + col_a, hw);
                            tmem_st8(lane_base + col_a + 16u, lw);
                            tmem_wait_st();
                            tc_fence_before();
                            named_bar_sync(bar_id, kGT);
                            if (issuer)
                                ws::ws_issue(st, 1, 0, tmem_base, col_a, col_d, &st->mma_bar[q]);
                        } else {
                            float qv = 0.0f;
                            if (KIND == kKindStats) {
                                if (valid) {
#pragma unroll
                                    for (int k = 0; k < 6; ++k)
                                        p.stats_out[6 * j + k] = y[k];
                                }
                            } else if (KIND == kKindAdrrs) {
                                const float num = luminance(sd.ex[0] * y[0], sd.ex[1] * y[1], sd.ex[2] * y[2]);
                                const float qq = num / (sd.ex[3] + p.eps);
                                qv = qq < 0.05f ? 0.05f : (20.0f < qq ? 20.0f : qq);
                            } else {
                                qv = softplus_mod(y[0]);
                            }
                            if (kTiming && (p.ablate & 2u))
                                qv = sd.ex[0] + 1.0f;
                            if (KIND != kKindStats) {
                                uint32_t decided = active ? 1u : 0u;
                                if (p.gate) {
                                    if (valid && depth1)
                                        qv = 1.0f;
                                    if (!active && !depth1)
                                        qv = 0.0f;
                                    decided = valid && (depth1 || active) ? 1u : 0u;
                                    if (valid && (!isfinite(qv) || qv < 0.0f)) {  // sanitize (wavefront.cpp:381-385)
                                        qv = 0.0f;
                                        decided = 0;
                                        ++my_nonfinite;
                                    }
                                }
                                if (valid) {
                                    p.q_out[j] = qv;
                                    if (p.u_out)
                                        p.u_out[j] = rrs_uniform(p.mixed_seed, sd.key, p.depth);
                                    if (p.decided_out)
                                        p.decided_out[j] = (uint8_t)decided;
                                    fx_add_q(my_fx, qv);
                                }
                            }
                            mbar_arrive(&st->empty[slot[c]]);
                            if (rec && blockIdx.x == 0 && tile[c] < 1024) p.dbg[8192 + 4 * tile[c] + 3] = clock64();
                        }
                    }
                    if (rec) c_epi += clock64() - t0;
                }
            }
        }
        if (rec && g == 0)
            p.dbg[blockIdx.x * 32 + 14] = clock64();  // MLP group 0 loop end (clock64, minus start below)
        if (rec) {
            p.dbg[blockIdx.x * 32 + 8 + 2 * g + 0] = c_wait;
            p.dbg[blockIdx.x * 32 + 8 + 2 * g + 1] = c_epi;
        }
    }

    // ---- teardown + deterministic CTA reduction, then last-CTA-done ----
    tc_fence_before();
    __syncthreads();
    if (kTiming && p.dbg && tid == 0) {
        unsigned long long g_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
        p.dbg[blockIdx.x * 32 + 14] -= c_start;
        for (int q = 16; q < 20; ++q)
            p.dbg[blockIdx.x * 32 + q] -= c_start;
        p.dbg[blockIdx.x * 32 + 15] = clock64() - c_start;  // CTA end
        p.dbg[blockIdx.x * 32 + 12] = g_start;
        p.dbg[blockIdx.x * 32 + 13] = g_end;
    }
    if (warp == 0)
        tmem_dealloc(tmem_base, 512);
    if (KIND == kKindStats || p.parts == nullptr)
        return;
    ka_reduce_finish<Cfg::kThreads / 32>(p, st, my_fx, my_nonfinite, my_bc);
}

// ===========================================================================
// K-A, AID over level planes, no encoder warps: GM groups of 4 warps (one thread per tile
// row) each run a tile end to end -- load the row's 8 level planes and tail inputs, tail
// encodings, fp16 hi/lo layer-0 A into the group's own TMEM columns, then the 4-layer
// tcgen05 chain and the head -- so GM chains are in flight per SM instead of one per MLP
// group behind shared encoder groups.  TMEM: per group 32 accumulator + 32 A columns.
// ===========================================================================
template <int GM>
__global__ void __launch_bounds__(GM * 128, 1) infer_aid_fused_kernel(InferParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem_w = smem_raw;
    ws::SmemTail *st = reinterpret_cast<ws::SmemTail *>(smem_raw + ((p.blob_bytes + 127u) & ~127u));
    const int tid = threadIdx.x, warp = tid >> 5;
    constexpr int kThreads = GM * 128;
    static_assert(GM * 64 <= 512 && GM <= 8, "TMEM: 64 columns per group");
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(p.blob);
        uint4 *dst = reinterpret_cast<uint4 *>(smem_w);
        for (uint32_t i = tid; i < p.blob_bytes / 16u; i += kThreads)
            dst[i] = __ldg(src + i);
    }
    if (tid == 0) {
        const NetDesc &nd = p.nets.rrs;
        for (int l = 0; l < 4; ++l) {
            const LayerDesc &L = nd.layer[l];
            st->idesc_n[1][l] = make_idesc_f16(L.N);
            st->idesc_2n[1][l] = make_idesc_f16(2u * L.N);
            st->nslices[1][l] = (uint32_t)L.K / 16u;
            st->bias[1][l] = L.bias;
            const uint32_t sbo = (uint32_t)L.K * 16u;
            for (int k = 0; k < 2; ++k) {
                st->wdesc[1][l][k] = make_smem_desc(smem_u32(smem_w + L.w_hi) + 256u * k, 128u, sbo);
                st->wdesc_lo[1][l][k] =
                    make_smem_desc(smem_u32(smem_w + L.w_hi) + 256u * k + ((uint32_t)L.N / 8u) * sbo, 128u, sbo);
            }
        }
        for (int q = 0; q < GM; ++q) {
            mbar_init(&st->mma_bar[q], 1);
            mbar_init(&st->full[q], 1);
        }
        fence_barrier_init();
    }
    if (warp == 0)
        tmem_alloc(&st->tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_trigger();
    pdl_wait();  // the level planes of K-A0 (PDL launch: the prologue above overlapped its tail)
    const uint32_t tmem_base = st->tmem_base;
    const uint32_t lane_base = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
    const int g = tid >> 7, r = tid & 127;
    const bool issuer = r == 0;
    const uint32_t bar_id = 1u + (uint32_t)g;
    const uint32_t col_d = 64u * (uint32_t)g, col_a = col_d + 32u;

    const uint64_t n = p.n;
    const uint64_t num_tiles = (n + kTileM - 1) / kTileM;
    const uint64_t t_begin = num_tiles * blockIdx.x / gridDim.x;
    const uint64_t t_end = num_tiles * (blockIdx.x + 1) / gridDim.x;
    const uint32_t T = (uint32_t)(t_end - t_begin);
    Fx128 my_fx{0ull, 0ull};  // exact sum of q (fixed point)
    uint32_t my_nonfinite = 0, my_bc = 0;
    const bool depth1 = p.depth == 1u;
    const int levels = p.grid_rrs.levels;
    uint32_t phase = 0;

    // Row inputs of the group's NEXT tile are staged into its smem slot by TMA bulk copies
    // (issued right after the current tile's layer-0 MMA, so they land during the 4-layer
    // chain); a partial last tile, or unaligned inputs, load directly.
    uint8_t *in_s = smem_raw + aid_in_offset(p.blob_bytes) + (uint32_t)g * kAidInBytes;
    const bool in_bulk = p.in_bulk != 0u;
    const uint64_t full_tiles = n / kTileM;
    uint32_t in_phase = 0;
    auto issue_in = [&](uint64_t tile) {  // issuer only; the group has finished reading the slot
        const uint64_t j0 = tile * kTileM;
        const uint32_t ipx_bytes = p.i_pixel ? 12u * kTileM : 4u * kTileM;
        mbar_arrive_expect_tx(&st->full[g], (uint32_t)levels * 8u * kTileM + 12u * kTileM + 8u * kTileM +
                                                ipx_bytes + 4u * kTileM + 8u * kTileM);
        for (int q = 0; q < levels; ++q)
            bulk_g2s(in_s + kAidInPlane * q, p.feat + (uint64_t)q * p.feat_stride + j0, 8u * kTileM, &st->full[g]);
        bulk_g2s(in_s + kAidInWeight, p.weight + 3 * j0, 12u * kTileM, &st->full[g]);
        bulk_g2s(in_s + kAidInWo, p.wo01 + 2 * j0, 8u * kTileM, &st->full[g]);
        if (p.i_pixel)
            bulk_g2s(in_s + kAidInIpx, p.i_pixel + 3 * j0, ipx_bytes, &st->full[g]);
        else
            bulk_g2s(in_s + kAidInIpx, p.pixel + j0, ipx_bytes, &st->full[g]);
        bulk_g2s(in_s + kAidInRough, p.roughness + j0, 4u * kTileM, &st->full[g]);
        bulk_g2s(in_s + kAidInKey, p.path_key + j0, 8u * kTileM, &st->full[g]);
    };
    if (in_bulk && r == 32 && (uint32_t)g < T && t_begin + (uint32_t)g < full_tiles)
        issue_in(t_begin + (uint32_t)g);

    for (uint32_t i = (uint32_t)g; i < T; i += GM) {
        const uint64_t j = (t_begin + i) * kTileM + r;
        const bool valid = j < n;
        const bool staged = in_bulk && t_begin + i < full_tiles;
        // ---- row inputs: level planes + tail inputs ----
        float f[16];
        float wx = 0, wy = 0, wz = 0, wox = 0, woy = 0, ia = 0, ib = 0, ic = 0, rough = 0;
        uint64_t key = 0;
        if (staged) {
            mbar_wait(&st->full[g], in_phase);
            in_phase ^= 1u;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float2 v = make_float2(0.0f, 0.0f);
                if (q < levels)
                    v = reinterpret_cast<const float2 *>(in_s + kAidInPlane * q)[r];
                f[2 * q] = v.x;
                f[2 * q + 1] = v.y;
            }
            const float *w3 = reinterpret_cast<const float *>(in_s + kAidInWeight) + 3 * r;
            wx = w3[0]; wy = w3[1]; wz = w3[2];
            const float2 wo = reinterpret_cast<const float2 *>(in_s + kAidInWo)[r];
            wox = wo.x; woy = wo.y;
            if (p.i_pixel) {
                const float *i3 = reinterpret_cast<const float *>(in_s + kAidInIpx) + 3 * r;
                ia = i3[0]; ib = i3[1]; ic = i3[2];
            } else {
                const uint64_t px_idx = reinterpret_cast<const uint32_t *>(in_s + kAidInIpx)[r];
                ia = __ldg(p.i_acc + 3 * px_idx); ib = __ldg(p.i_acc + 3 * px_idx + 1); ic = __ldg(p.i_acc + 3 * px_idx + 2);
            }
            rough = reinterpret_cast<const float *>(in_s + kAidInRough)[r];
            key = reinterpret_cast<const uint64_t *>(in_s + kAidInKey)[r];
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float2 v = make_float2(0.0f, 0.0f);
                if (valid && q < levels)
                    v = __ldcs(p.feat + (uint64_t)q * p.feat_stride + j);
                f[2 * q] = v.x;
                f[2 * q + 1] = v.y;
            }
            if (valid) {
                wx = __ldg(p.weight + 3 * j); wy = __ldg(p.weight + 3 * j + 1); wz = __ldg(p.weight + 3 * j + 2);
                wox = __ldg(p.wo01 + 2 * j); woy = __ldg(p.wo01 + 2 * j + 1);
                if (p.i_pixel) {
                    ia = __ldg(p.i_pixel + 3 * j); ib = __ldg(p.i_pixel + 3 * j + 1); ic = __ldg(p.i_pixel + 3 * j + 2);
                } else {
                    const uint64_t px_idx = __ldg(p.pixel + j);
                    ia = __ldg(p.i_acc + 3 * px_idx); ib = __ldg(p.i_acc + 3 * px_idx + 1); ic = __ldg(p.i_acc + 3 * px_idx + 2);
                }
                rough = __ldg(p.roughness + j);
                key = __ldg(p.path_key + j);
            }
        }
        const bool active = valid && (p.gate ? (!depth1 && luminance(wx, wy, wz) > 0.0f) : true);
        // ---- layer-0 input (build_aid_tail, networks.cpp:149-157) in the packed K order ----
        uint32_t bc = 0;
        float x0[16], x1[16];  // K columns [0,16): grid 0-7 | tail 0-7; [16,32): grid 8-15 | tail 8-15
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            x0[q] = f[q];
            x1[q] = f[8 + q];
        }
        one_blob_fast<4>(wox, x0 + 8);
        one_blob_fast<4>(woy, x0 + 12);
        x1[8] = box_cox_fast(wx, bc);
        x1[9] = box_cox_fast(wy, bc);
        x1[10] = box_cox_fast(wz, bc);
        x1[11] = box_cox_fast(mean3_fast(ia, ib, ic), bc);
        one_blob_fast<4>(remap_fast(rough), x1 + 12);
        if (!valid) {
#pragma unroll
            for (int q = 0; q < 16; ++q)
                x0[q] = x1[q] = 0.0f;
        }
        if (active)
            my_bc += bc;
        // the group's previous tile finished reading D and A before the barrier below
        ws::ws_store_a16(lane_base, col_a, 0, x0);
        ws::ws_store_a16(lane_base, col_a, 1, x1);
        tmem_wait_st();
        tc_fence_before();
        named_bar_sync(bar_id, 128);
        if (issuer)
            ws::ws_issue(st, 1, 0, tmem_base, col_a, col_d, &st->mma_bar[g]);
        // every thread of the group has consumed its slot row (barrier above); a second warp
        // issues the copies so the MMA issuer's warp goes straight to the layer-0 wait
        if (r == 32 && in_bulk && i + GM < T && t_begin + i + GM < full_tiles) {
            fence_proxy_async_smem();
            issue_in(t_begin + i + GM);
        }
        // ---- 4-layer chain ----
#pragma unroll 1
        for (int l = 0; l < 4; ++l) {
#if NRRS_AID_MMA_HINT
            mbar_wait_sleep(&st->mma_bar[g], phase, NRRS_AID_MMA_HINT);
#else
            mbar_wait(&st->mma_bar[g], phase);
#endif
            phase ^= 1u;
            tc_fence_after();
            const uint32_t boff = st->bias[1][l];
            const float *bias = boff == kNoBias ? nullptr : reinterpret_cast<const float *>(smem_w + boff);
            if (l < 3) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float z[16];
                    ws::ws_load_sum16(lane_base, col_d, 32u, 16u * (uint32_t)h, bias, z);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {  // leaky ReLU = cwiseMax(z, slope z)
                        const float2 t = upk2(fmul2(pk2(z[2 * q], z[2 * q + 1]), pk2(0.01f, 0.01f)));
                        z[2 * q] = fmaxf(z[2 * q], t.x);
                        z[2 * q + 1] = fmaxf(z[2 * q + 1], t.y);
                    }
                    ws::ws_store_a16(lane_base, col_a, h, z);
                }
                tmem_wait_st();
                tc_fence_before();
                named_bar_sync(bar_id, 128);
                if (issuer)
                    ws::ws_issue(st, 1, l + 1, tmem_base, col_a, col_d, &st->mma_bar[g]);
            } else {
                const float y0 = ws::ws_load_head1(lane_base, col_d, bias);  // head: one output
                tc_fence_before();
                float qv = softplus_mod(y0);
                uint32_t decided = active ? 1u : 0u;
                if (p.gate) {
                    if (valid && depth1)
                        qv = 1.0f;
                    if (!active && !depth1)
                        qv = 0.0f;
                    decided = valid && (depth1 || active) ? 1u : 0u;
                    if (valid && (!isfinite(qv) || qv < 0.0f)) {  // sanitize (wavefront.cpp:381-385)
                        qv = 0.0f;
                        decided = 0;
                        ++my_nonfinite;
                    }
                }
                if (valid) {
                    p.q_out[j] = qv;
                    if (p.u_out)
                        p.u_out[j] = rrs_uniform(p.mixed_seed, key, p.depth);
                    if (p.decided_out)
                        p.decided_out[j] = (uint8_t)decided;
                    fx_add_q(my_fx, qv);
                }
            }
        }
    }

    // ---- teardown + deterministic CTA reduction, then last-CTA-done ----
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        tmem_dealloc(tmem_base, 512);
    if (p.parts == nullptr)
        return;
    ka_reduce_finish<kThreads / 32>(p, st, my_fx, my_nonfinite, my_bc);
}

// ===========================================================================
// K-A over fp32 feature planes for the StatNet-grid kinds (ADRRS-NN, stats, NRRS): the same
// self-contained-group shape as infer_aid_fused_kernel, fed by grid_level_kernel<true> (one
// (level, feature) table of the fp32 StatNet grid per CTA from shared memory) instead of L2 gathers.
// Layer-0 input: the 16 StatNet grid features + build_stat_tail (networks.cpp:131-135).  ADRRS-NN /
// stats end at the StatNet head (networks.cpp:252-264, rrs.hpp:56-61); NRRS continues with
// build_nrrs_input (networks.cpp:137-147) and the RRSNet chain (8 MMA layers per tile).
// ===========================================================================
template <int KIND>
__global__ void __launch_bounds__(8 * 128, 1) infer_stat_planes_kernel(InferParams p) {
    constexpr int GM = 8;
    constexpr int kNL = KIND == kKindNrrs ? 8 : 4;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem_w = smem_raw;
    ws::SmemTail *st = reinterpret_cast<ws::SmemTail *>(smem_raw + ((p.blob_bytes + 127u) & ~127u));
    const int tid = threadIdx.x, warp = tid >> 5;
    constexpr int kThreads = GM * 128;
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(p.blob);
        uint4 *dst = reinterpret_cast<uint4 *>(smem_w);
        for (uint32_t i = tid; i < p.blob_bytes / 16u; i += kThreads)
            dst[i] = __ldg(src + i);
    }
    if (tid == 0) {
        for (int net = 0; net < (KIND == kKindNrrs ? 2 : 1); ++net) {
            const NetDesc &nd = net == 0 ? p.nets.stat : p.nets.rrs;
            for (int l = 0; l < 4; ++l) {
                const LayerDesc &Ld = nd.layer[l];
                st->idesc_n[net][l] = make_idesc_f16(Ld.N);
                st->idesc_2n[net][l] = make_idesc_f16(2u * Ld.N);
                st->nslices[net][l] = (uint32_t)Ld.K / 16u;
                st->bias[net][l] = Ld.bias;
                const uint32_t sbo = (uint32_t)Ld.K * 16u;
                for (int kk = 0; kk < 2; ++kk) {
                    st->wdesc[net][l][kk] = make_smem_desc(smem_u32(smem_w + Ld.w_hi) + 256u * kk, 128u, sbo);
                    st->wdesc_lo[net][l][kk] = make_smem_desc(
                        smem_u32(smem_w + Ld.w_hi) + 256u * kk + ((uint32_t)Ld.N / 8u) * sbo, 128u, sbo);
                }
            }
        }
        for (int q = 0; q < GM; ++q) {
            mbar_init(&st->mma_bar[q], 1);
            mbar_init(&st->full[q], 1);
        }
        fence_barrier_init();
    }
    if (warp == 0)
        tmem_alloc(&st->tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_trigger();
    pdl_wait();  // the feature planes of grid_level_kernel<true>
    const uint32_t tmem_base = st->tmem_base;
    const uint32_t lane_base = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
    const int g = tid >> 7, r = tid & 127;
    const bool issuer = r == 0;
    const uint32_t bar_id = 1u + (uint32_t)g;
    const uint32_t col_d = 64u * (uint32_t)g, col_a = col_d + 32u;

    const uint64_t n = p.n;
    const uint64_t num_tiles = (n + kTileM - 1) / kTileM;
    const uint64_t t_begin = num_tiles * blockIdx.x / gridDim.x;
    const uint64_t t_end = num_tiles * (blockIdx.x + 1) / gridDim.x;
    const uint32_t T = (uint32_t)(t_end - t_begin);
    Fx128 my_fx{0ull, 0ull};  // exact sum of q (fixed point)
    uint32_t my_nonfinite = 0, my_bc = 0;
    const bool depth1 = p.depth == 1u;
    const int nfeat = 2 * p.grid.levels;  // fp32 planes: one per (level, feature)
    constexpr bool kNeedIpx = KIND != kKindStats;
    uint32_t phase = 0;
    uint8_t *in_s = smem_raw + aid_in_offset(p.blob_bytes) + (uint32_t)g * kAidInBytes;
    const bool in_bulk = p.in_bulk != 0u;
    const uint64_t full_tiles = n / kTileM;
    uint32_t in_phase = 0;
    const float *planes = reinterpret_cast<const float *>(p.feat);
    auto issue_in = [&](uint64_t tile) {
        const uint64_t j0 = tile * kTileM;
        const uint32_t ipx_bytes = !kNeedIpx ? 0u : (p.i_pixel ? 12u * kTileM : 4u * kTileM);
        mbar_arrive_expect_tx(&st->full[g], (uint32_t)nfeat * 4u * kTileM + 12u * kTileM + 8u * kTileM + ipx_bytes +
                                                4u * kTileM + 8u * kTileM);
        for (int q = 0; q < nfeat; ++q)
            bulk_g2s(in_s + 4u * kTileM * q, planes + (uint64_t)q * p.feat_stride + j0, 4u * kTileM, &st->full[g]);
        bulk_g2s(in_s + kAidInWeight, p.weight + 3 * j0, 12u * kTileM, &st->full[g]);
        bulk_g2s(in_s + kAidInWo, p.wo01 + 2 * j0, 8u * kTileM, &st->full[g]);
        if (kNeedIpx) {
            if (p.i_pixel)
                bulk_g2s(in_s + kAidInIpx, p.i_pixel + 3 * j0, ipx_bytes, &st->full[g]);
            else
                bulk_g2s(in_s + kAidInIpx, p.pixel + j0, ipx_bytes, &st->full[g]);
        }
        bulk_g2s(in_s + kAidInRough, p.roughness + j0, 4u * kTileM, &st->full[g]);
        bulk_g2s(in_s + kAidInKey, p.path_key + j0, 8u * kTileM, &st->full[g]);
    };
    if (in_bulk && r == 32 && (uint32_t)g < T && t_begin + (uint32_t)g < full_tiles)
        issue_in(t_begin + (uint32_t)g);

    for (uint32_t i = (uint32_t)g; i < T; i += GM) {
        const uint64_t j = (t_begin + i) * kTileM + r;
        const bool valid = j < n;
        const bool staged = in_bulk && t_begin + i < full_tiles;
        float f[16];
        float wx = 0, wy = 0, wz = 0, wox = 0, woy = 0, ia = 0, ib = 0, ic = 0, rough = 0;
        uint64_t key = 0;
        if (staged) {
            mbar_wait(&st->full[g], in_phase);
            in_phase ^= 1u;
#pragma unroll
            for (int q = 0; q < 16; ++q)
                f[q] = q < nfeat ? reinterpret_cast<const float *>(in_s + 4u * kTileM * q)[r] : 0.0f;
            const float *w3 = reinterpret_cast<const float *>(in_s + kAidInWeight) + 3 * r;
            wx = w3[0]; wy = w3[1]; wz = w3[2];
            const float2 wo = reinterpret_cast<const float2 *>(in_s + kAidInWo)[r];
            wox = wo.x; woy = wo.y;
            if (kNeedIpx) {
                if (p.i_pixel) {
                    const float *i3 = reinterpret_cast<const float *>(in_s + kAidInIpx) + 3 * r;
                    ia = i3[0]; ib = i3[1]; ic = i3[2];
                } else {
                    const uint64_t px_idx = reinterpret_cast<const uint32_t *>(in_s + kAidInIpx)[r];
                    ia = __ldg(p.i_acc + 3 * px_idx); ib = __ldg(p.i_acc + 3 * px_idx + 1); ic = __ldg(p.i_acc + 3 * px_idx + 2);
                }
            }
            rough = reinterpret_cast<const float *>(in_s + kAidInRough)[r];
            key = reinterpret_cast<const uint64_t *>(in_s + kAidInKey)[r];
        } else {
#pragma unroll
            for (int q = 0; q < 16; ++q)
                f[q] = valid && q < nfeat ? __ldcs(planes + (uint64_t)q * p.feat_stride + j) : 0.0f;
            if (valid) {
                wx = __ldg(p.weight + 3 * j); wy = __ldg(p.weight + 3 * j + 1); wz = __ldg(p.weight + 3 * j + 2);
                wox = __ldg(p.wo01 + 2 * j); woy = __ldg(p.wo01 + 2 * j + 1);
                if (kNeedIpx) {
                    if (p.i_pixel) {
                        ia = __ldg(p.i_pixel + 3 * j); ib = __ldg(p.i_pixel + 3 * j + 1); ic = __ldg(p.i_pixel + 3 * j + 2);
                    } else {
                        const uint64_t px_idx = __ldg(p.pixel + j);
                        ia = __ldg(p.i_acc + 3 * px_idx); ib = __ldg(p.i_acc + 3 * px_idx + 1); ic = __ldg(p.i_acc + 3 * px_idx + 2);
                    }
                }
                rough = __ldg(p.roughness + j);
                key = KIND != kKindStats ? __ldg(p.path_key + j) : 0ull;
            }
        }
        const bool active = valid && (p.gate ? (!depth1 && luminance(wx, wy, wz) > 0.0f) : true);
        // ---- layer-0 input: encode_stat_inputs (networks.cpp:206-217) in the packed K order ----
        float x0[16], x1[16];  // [0,16): grid 0-7 | ob4(wo.x), ob4(wo.y); [16,32): grid 8-15 | ob8(remap(r))
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            x0[q] = f[q];
            x1[q] = f[8 + q];
        }
        one_blob_fast<4>(wox, x0 + 8);
        one_blob_fast<4>(woy, x0 + 12);
        one_blob_fast<8>(remap_fast(rough), x1 + 8);
        if (!valid) {
#pragma unroll
            for (int q = 0; q < 16; ++q)
                x0[q] = x1[q] = 0.0f;
        }
        ws::ws_store_a16(lane_base, col_a, 0, x0);
        ws::ws_store_a16(lane_base, col_a, 1, x1);
        tmem_wait_st();
        tc_fence_before();
        named_bar_sync(bar_id, 128);
        if (issuer)
            ws::ws_issue(st, 0, 0, tmem_base, col_a, col_d, &st->mma_bar[g]);
        if (r == 32 && in_bulk && i + GM < T && t_begin + i + GM < full_tiles) {
            fence_proxy_async_smem();
            issue_in(t_begin + i + GM);
        }
        // ---- MMA chain: StatNet (layers 0-3), then for NRRS the RRSNet (4-7) ----
#pragma unroll 1
        for (int l = 0; l < kNL; ++l) {
            mbar_wait(&st->mma_bar[g], phase);
            phase ^= 1u;
            tc_fence_after();
            const int lyr = l & 3;
            const int net = l >= 4 ? 1 : 0;
            const uint32_t boff = st->bias[net][lyr];
            const float *bias = boff == kNoBias ? nullptr : reinterpret_cast<const float *>(smem_w + boff);
            if (lyr < 3) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float z[16];
                    ws::ws_load_sum16(lane_base, col_d, 32u, 16u * (uint32_t)h, bias, z);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {  // leaky ReLU = cwiseMax(z, slope z)
                        const float2 t = upk2(fmul2(pk2(z[2 * q], z[2 * q + 1]), pk2(0.01f, 0.01f)));
                        z[2 * q] = fmaxf(z[2 * q], t.x);
                        z[2 * q + 1] = fmaxf(z[2 * q + 1], t.y);
                    }
                    ws::ws_store_a16(lane_base, col_a, h, z);
                }
                tmem_wait_st();
                tc_fence_before();
                named_bar_sync(bar_id, 128);
                if (issuer)
                    ws::ws_issue(st, net, lyr + 1, tmem_base, col_a, col_d, &st->mma_bar[g]);
            } else if (KIND == kKindNrrs && l == 3) {
                // stats -> build_nrrs_input (networks.cpp:137-147) -> RRSNet layer 0
                float y[16];
                ws::ws_load_sum16(lane_base, col_d, 16u, 0u, bias, y);
                uint32_t bc = 0;
                float xin[16];
#pragma unroll
                for (int q = 0; q < 6; ++q)
                    xin[q] = box_cox_fast(y[q], bc);
                xin[6] = box_cox_fast(wx, bc);
                xin[7] = box_cox_fast(wy, bc);
                xin[8] = box_cox_fast(wz, bc);
                xin[9] = box_cox_fast(mean3_fast(ia, ib, ic), bc);
                xin[10] = remap_fast(rough);
                xin[11] = 1.0f;  // bias column of the RRSNet first layer
#pragma unroll
                for (int q = 12; q < 16; ++q)
                    xin[q] = 0.0f;
                if (!valid) {
#pragma unroll
                    for (int q = 0; q < 11; ++q)
                        xin[q] = 0.0f;
                }
                if (active)
                    my_bc += bc;
                uint32_t hw[8], lw[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    split2(xin[2 * q], xin[2 * q + 1], hw[q], lw[q]);
                tmem_st8(lane_base + col_a, hw);
                tmem_st8(lane_base + col_a + 16u, lw);
                tmem_wait_st();
                tc_fence_before();
                named_bar_sync(bar_id, 128);
                if (issuer)
                    ws::ws_issue(st, 1, 0, tmem_base, col_a, col_d, &st->mma_bar[g]);
            } else {
                float qv = 0.0f;
                if (KIND == kKindStats) {
                    float y[16];
                    ws::ws_load_sum16(lane_base, col_d, 16u, 0u, bias, y);
                    tc_fence_before();
                    if (valid) {
#pragma unroll
                        for (int q = 0; q < 6; ++q)
                            p.stats_out[6 * j + q] = y[q];
                    }
                    continue;
                } else if (KIND == kKindAdrrs) {
                    float y[16];
                    ws::ws_load_sum16(lane_base, col_d, 16u, 0u, bias, y);
                    const float num = luminance(wx * y[0], wy * y[1], wz * y[2]);
                    const float qq = num / (luminance(ia, ib, ic) + p.eps);
                    qv = qq < 0.05f ? 0.05f : (20.0f < qq ? 20.0f : qq);
                } else {
                    qv = softplus_mod(ws::ws_load_head1(lane_base, col_d, bias));
                }
                tc_fence_before();
                uint32_t decided = active ? 1u : 0u;
                if (p.gate) {
                    if (valid && depth1)
                        qv = 1.0f;
                    if (!active && !depth1)
                        qv = 0.0f;
                    decided = valid && (depth1 || active) ? 1u : 0u;
                    if (valid && (!isfinite(qv) || qv < 0.0f)) {  // sanitize (wavefront.cpp:381-385)
                        qv = 0.0f;
                        decided = 0;
                        ++my_nonfinite;
                    }
                }
                if (valid) {
                    p.q_out[j] = qv;
                    if (p.u_out)
                        p.u_out[j] = rrs_uniform(p.mixed_seed, key, p.depth);
                    if (p.decided_out)
                        p.decided_out[j] = (uint8_t)decided;
                    fx_add_q(my_fx, qv);
                }
            }
        }
    }

    // ---- teardown + deterministic CTA reduction, then last-CTA-done ----
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        tmem_dealloc(tmem_base, 512);
    if (KIND == kKindStats || p.parts == nullptr)
        return;
    ka_reduce_finish<kThreads / 32>(p, st, my_fx, my_nonfinite, my_bc);
}

static bool aligned16(const void *q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; }

template <int GM>
static cudaError_t launch_aid_fused(const InferParams &p_in, int num_sms, cudaStream_t stream, uint32_t *grid_out) {
    InferParams p = p_in;
    // TMA-staged row inputs need 16-byte aligned field bases and plane stride (whole tiles are
    // 16-byte multiples); otherwise every tile loads directly.
    const size_t smem_direct = ((p.blob_bytes + 127u) & ~127u) + sizeof(ws::SmemTail) + 64;
    const size_t smem_staged = (size_t)aid_in_offset(p.blob_bytes) + (size_t)GM * kAidInBytes;
    p.in_bulk = 0;
#ifndef NRRS_AID_NO_PREFETCH
    if (smem_staged <= 227u * 1024u && p.grid_rrs.levels <= 8 && (p.feat_stride & 1u) == 0 && aligned16(p.feat) &&
        aligned16(p.weight) && aligned16(p.wo01) && aligned16(p.roughness) && aligned16(p.path_key) &&
        (p.i_pixel ? aligned16(p.i_pixel) : (p.pixel != nullptr && aligned16(p.pixel))))
        p.in_bulk = 1;
#endif
    const size_t smem = p.in_bulk ? smem_staged : smem_direct;
    cudaError_t e = cudaFuncSetAttribute(infer_aid_fused_kernel<GM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess)
        return e;
    const uint64_t tiles = (p.n + kTileM - 1) / kTileM;
    uint64_t grid = (uint64_t)num_sms;
    if (grid > tiles)
        grid = tiles;
    if (grid < 1)
        grid = 1;
    *grid_out = (uint32_t)grid;
    return launch_maybe_pdl(infer_aid_fused_kernel<GM>, (uint32_t)grid, GM * 128, smem, stream, p);
}

template <int KIND>
static cudaError_t launch_stat_planes(const InferParams &p_in, int num_sms, cudaStream_t stream, uint32_t *grid_out) {
    InferParams p = p_in;
    const size_t smem_direct = ((p.blob_bytes + 127u) & ~127u) + sizeof(ws::SmemTail) + 64;
    const size_t smem_staged = (size_t)aid_in_offset(p.blob_bytes) + (size_t)8 * kAidInBytes;
    p.in_bulk = 0;
    const bool ipx_ok = KIND == kKindStats || (p.i_pixel ? aligned16(p.i_pixel) : (p.pixel != nullptr && aligned16(p.pixel)));
    if (smem_staged <= 227u * 1024u && p.grid.levels <= 8 && (p.feat_stride & 3u) == 0 && aligned16(p.feat) &&
        aligned16(p.weight) && aligned16(p.wo01) && aligned16(p.roughness) && aligned16(p.path_key) && ipx_ok)
        p.in_bulk = 1;
    const size_t smem = p.in_bulk ? smem_staged : smem_direct;
    cudaError_t e = cudaFuncSetAttribute(infer_stat_planes_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess)
        return e;
    const uint64_t tiles = (p.n + kTileM - 1) / kTileM;
    uint64_t grid = (uint64_t)num_sms;
    if (grid > tiles)
        grid = tiles;
    if (grid < 1)
        grid = 1;
    *grid_out = (uint32_t)grid;
    return launch_maybe_pdl(infer_stat_planes_kernel<KIND>, (uint32_t)grid, 8 * 128, smem, stream, p);
}

template <int KIND, int GE, int GM, int P, int TPR, bool HALF>
static cudaError_t launch_ws(const InferParams &p, int num_sms, cudaStream_t stream, uint32_t *grid_out) {
    using Cfg = ws::Cfg<GE, GM, P, TPR>;
    const size_t smem = ((p.blob_bytes + 127u) & ~127u) + Cfg::kSlots * 128 * sizeof(ws::Side) +
                        sizeof(ws::SmemTail) + 64;
    cudaError_t e = cudaFuncSetAttribute(infer_ws_kernel<KIND, GE, GM, P, TPR, HALF>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
#ifdef NRRS_CARVEOUT
    // smallest shared-memory carveout that fits: the rest of the 256 KB stays L1 for the grid levels
    e = cudaFuncSetAttribute(infer_ws_kernel<KIND, GE, GM, P, TPR, HALF>,
                             cudaFuncAttributePreferredSharedMemoryCarveout, NRRS_CARVEOUT);
    if (e != cudaSuccess)
        return e;
#endif
    const uint64_t tiles = (p.n + kTileM - 1) / kTileM;
    uint64_t grid = (uint64_t)num_sms;
    if (grid > tiles)
        grid = tiles;
    if (grid < 1)
        grid = 1;
    *grid_out = (uint32_t)grid;
    infer_ws_kernel<KIND, GE, GM, P, TPR, HALF><<<(uint32_t)grid, Cfg::kThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

// ===========================================================================
// Two-pass large-tile compaction (round 1's K-C form), kept for the 72-byte PathState records of
// trace_frame (compact2_kernel<18, 1>; the stage's slot records use compact3_kernel).  A tile is
// NRRS_BSUBS (default 4) sub-tiles of 512 threads x 4 items = 8,192 records.  Pass 1 keeps the
// flags in shared memory; one warp-parallel look-back gives the tile's exclusive prefix; pass 2
// re-scans sub-tile by sub-tile and writes the kept records with coalesced stores.
// ===========================================================================
constexpr int kBT = 512;            // threads
#ifndef NRRS_BSUBS
#define NRRS_BSUBS 4
#endif
constexpr int kBSubs = NRRS_BSUBS;  // sub-tiles per CTA tile (sweep 8/4/2/1: DESIGN.md section 6)

template <int NT>
__device__ __forceinline__ uint32_t block_scan_excl(uint32_t v, uint32_t *warp_tot, uint32_t &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o)
            inc += t;
    }
    __syncthreads();  // warp_tot reuse across calls
    if (lane == 31)
        warp_tot[warp] = inc;
    __syncthreads();
    uint32_t before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        const uint32_t t = warp_tot[w];
        if (w < warp)
            before += t;
        all += t;
    }
    total = all;
    return before + inc - v;
}

template <int W, int IPT>
__global__ void __launch_bounds__(kBT) compact2_kernel(CompactParams p) {
    constexpr int kSub = kBT * IPT;
    constexpr int kTile = kSub * kBSubs;
    extern __shared__ __align__(16) uint8_t csm[];
    uint32_t *stage = reinterpret_cast<uint32_t *>(csm);              // kSub * W words
    uint8_t *masks = csm + (size_t)kSub * W * 4;                      // kBSubs * kBT bytes
    uint32_t *warp_tot = reinterpret_cast<uint32_t *>(masks + kBSubs * kBT);
    unsigned long long *prefix = reinterpret_cast<unsigned long long *>(warp_tot + kBT / 32 + 2);
    uint32_t *tile_s = reinterpret_cast<uint32_t *>(prefix + 1);
    const int tid = threadIdx.x;
    if (tid == 0)
        tile_s[0] = claim_tile_epoch(p.sync, tile_s + 1);
    __syncthreads();
    const uint32_t tile = tile_s[0], epoch = tile_s[1];
    const uint64_t tbase = (uint64_t)tile * kTile;
    uint64_t count = p.count;
    if (p.count_in) {
        const uint64_t c = *p.count_in;
        count = c < count ? c : count;
    }
    // pass 1: flags -> per-thread masks, tile count
    uint32_t my_cnt = 0;
#pragma unroll
    for (int sub = 0; sub < kBSubs; ++sub) {
        const uint64_t first = tbase + (uint64_t)sub * kSub + (uint64_t)tid * IPT;
        uint32_t m = 0;
        if (IPT == 4 && first + 4 <= count && (reinterpret_cast<uintptr_t>(p.used + first) & 3u) == 0) {
            const uint32_t w4 = __ldcs(reinterpret_cast<const unsigned int *>(p.used + first));
#pragma unroll
            for (int i = 0; i < 4; ++i)
                m |= ((w4 >> (8 * i)) & 0xffu) ? (1u << i) : 0u;
        } else {
#pragma unroll
            for (int i = 0; i < IPT; ++i)
                if (first + i < count && p.used[first + i])
                    m |= 1u << i;
        }
        masks[sub * kBT + tid] = (uint8_t)m;
        my_cnt += __popc(m);
    }
    const uint32_t *in = reinterpret_cast<const uint32_t *>(p.in);
    // slot records (W = 2): every sub-tile's records are requested now, so their HBM round trip
    // overlaps the block scan and the look-back instead of following it sub-tile by sub-tile
    constexpr bool kVec = W == 2 && IPT == 4;
    constexpr int kPre = kVec ? kBSubs : 1;
    uint4 pre[kPre][2];
    const bool vec_ok = kVec && (reinterpret_cast<uintptr_t>(in) & 15u) == 0;
    if (kVec) {
#pragma unroll
        for (int sub = 0; sub < kPre; ++sub) {
            const uint64_t first = tbase + (uint64_t)sub * kSub + (uint64_t)tid * IPT;
            if (vec_ok && first + 4 <= count && masks[sub * kBT + tid]) {
                const uint4 *in4 = reinterpret_cast<const uint4 *>(in + first * 2);
                pre[sub][0] = __ldcs(in4);
                pre[sub][1] = __ldcs(in4 + 1);
            }
        }
    }
    uint32_t agg = 0;
    block_scan_excl<kBT>(my_cnt, warp_tot, agg);
    if (tid < 32) {
        const uint64_t ex = lookback_warp(p.tile_state, tile, agg, epoch);
        if (tid == 0)
            *prefix = ex;
    }
    __syncthreads();
    uint64_t out_base = *prefix;
    // pass 2: stage kept records of each sub-tile in smem, write them coalesced
#pragma unroll
    for (int sub = 0; sub < kBSubs; ++sub) {
        const uint64_t first = tbase + (uint64_t)sub * kSub + (uint64_t)tid * IPT;
        const uint32_t m = masks[sub * kBT + tid];
        uint32_t sagg = 0;
        uint32_t pos = block_scan_excl<kBT>(__popc(m), warp_tot, sagg);
        if (kVec && vec_ok && m && first + 4 <= count) {
            // 4 slot records = 32 contiguous bytes, loaded above as two 16-byte requests
            const uint4 a = pre[kVec ? sub : 0][0], b = pre[kVec ? sub : 0][1];
            const uint2 rec[4] = {make_uint2(a.x, a.y), make_uint2(a.z, a.w), make_uint2(b.x, b.y),
                                  make_uint2(b.z, b.w)};
            uint2 *st2 = reinterpret_cast<uint2 *>(stage);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (m & (1u << i))
                    st2[pos++] = rec[i];
        } else {
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                if (m & (1u << i)) {
#pragma unroll
                    for (int w = 0; w < W; ++w)
                        stage[pos * W + w] = __ldcs(in + (first + i) * W + w);
                    ++pos;
                }
            }
        }
        __syncthreads();
        if (W == 2) {
            uint2 *out2 = reinterpret_cast<uint2 *>(p.out) + out_base;
            const uint2 *st2 = reinterpret_cast<const uint2 *>(stage);
            for (uint32_t r = tid; r < sagg; r += kBT)
                __stcs(out2 + r, st2[r]);
        } else {
            uint32_t *out = reinterpret_cast<uint32_t *>(p.out) + out_base * W;
            for (uint32_t w = tid; w < sagg * W; w += kBT)
                __stcs(out + w, stage[w]);
        }
        out_base += sagg;
        __syncthreads();
    }
    if (tile == p.num_tiles - 1 && tid == 0)
        *p.count_out = (uint32_t)(*prefix + agg);
    if (tid == 0)
        finish_launch(p.sync, p.tile_state, p.state_cap, epoch);
}

// ===========================================================================
// K-B / K-C, register-resident single-pass versions (round 2).
//
// A tile is up to 32 warps x 512 items; the launcher sizes it so the whole batch is ONE wave of
// <= one tile per SM (2,073,600 vertices: 145 tiles of 14,336), larger batches use 16,384-item
// tiles in several waves.  Items are warp-striped so every vector access is a fully coalesced
// 512-byte warp request: lane l of warp w holds items w * 512 + 128 i + 4 l + e (group i, element
// e).  One pass: all loads in flight at once, counts, 4 warp scans + one block reduction, the
// tile's exclusive prefix (single wave: the sum of every predecessor's published aggregate, one
// L2 round trip; several waves: the warp-parallel decoupled look-back), then the outputs.  A
// warp's slot records of one item group are contiguous in the queue, so they are staged in the
// warp's shared-memory buffer and leave as full 256-byte warp stores.  Index arithmetic is 32-bit
// (n < 2^32 and the capacity is a u32; positions are tile-relative).
// ===========================================================================
template <int SRC>  // 0: counts from (q, u) with normalization; 1: counts given (plan_spawns)
__global__ void __launch_bounds__(kD3T, 1) decide3_kernel(DecideParams p) {
    __shared__ Scan3Smem sm;
    extern __shared__ uint4 kq[];  // [group i][thread]: the thread's counts, parked between scan and writes
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_trigger();
    // the factor kernel's q / u / rank sums -- and a previous decide launch on this stream must be
    // done before this launch claims tiles from the shared LaunchSync (back-to-back stage calls)
    pdl_wait();
    if (tid == 0)
        sm.tile = claim_tile_epoch(p.sync, &sm.epoch);
    __syncthreads();
    const uint32_t tile = sm.tile, epoch = sm.epoch;
    stamp(p.dbg, tile, 0);
    // this tile's items end at min(n, (tile + 1) * tile_items): warps past a short tile idle
    const uint32_t n = min((uint32_t)p.n, (tile + 1u) * p.tile_items);
    const uint32_t wbase = tile * p.tile_items + (uint32_t)warp * kD3Warp + 4u * (uint32_t)lane;

    bool apply = false;
    float scale = 1.0f;
    if (SRC == 0) {
        double sum = 0.0;
        if (p.mbox) {  // sharded mailbox mode: every rank's sum of this depth from the own mailbox
            __shared__ double s_sum;
            if (tid == 0) {
                Fx128 t{0ull, 0ull};  // the ranks' exact sums add exactly: F equals the one-rank F bit for bit
                mbox_wait(p.mbox, 0, [&](int r, unsigned long long lo, unsigned long long hi) {
                    fx_add(t, Fx128{lo, hi});
                    if (tile == 0)
                        p.mbox->sums_seen[r] = fx_to_double(Fx128{lo, hi});
                });
                s_sum = fx_to_double(t);
            }
            __syncthreads();
            sum = s_sum;
        } else if (p.rank_sums_fx) {  // exact rank sums: F equals the one-rank F bit for bit
            Fx128 t{0ull, 0ull};
            for (int r = 0; r < p.nranks; ++r)
                fx_add(t, Fx128{p.rank_sums_fx[2 * r], p.rank_sums_fx[2 * r + 1]});
            sum = fx_to_double(t);
        } else {
            for (int r = 0; r < p.nranks; ++r)
                sum += p.rank_sums[r];
        }
        if (sum > 0.0) {
            const double f = __ddiv_rn((double)p.n_pixels, sum);  // F = Npx / sum (rrs.cpp:17)
            if (f < 1.0) {
                apply = true;
                scale = __double2float_rn(f);  // s = float(F)  (rrs.cpp:19)
            }
            if (tile == 0 && tid == 0 && p.res)
                p.res->f_norm = f;
        } else if (tile == 0 && tid == 0 && p.res) {
            p.res->f_norm = 1.0;
        }
    }
    // items of this thread that exist, per group
    uint32_t nv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t first = wbase + 128u * (uint32_t)i;
        nv[i] = first >= n ? 0u : (n - first < 4u ? n - first : 4u);
    }
    // ---- load every item of this thread (all requests in flight together) ----
    uint32_t gs[4];
    bool bad = false;
    if (SRC == 0) {
        float4 q4[4], u4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t first = wbase + 128u * (uint32_t)i;
            if (nv[i] == 4u) {
                q4[i] = __ldcs(reinterpret_cast<const float4 *>(p.q + first));
                u4[i] = __ldcs(reinterpret_cast<const float4 *>(p.u + first));
            } else {
                float qq[4], uu[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    qq[e] = (uint32_t)e < nv[i] ? p.q[first + e] : 0.0f;
                    uu[e] = (uint32_t)e < nv[i] ? p.u[first + e] : 1.0f;
                }
                q4[i] = make_float4(qq[0], qq[1], qq[2], qq[3]);
                u4[i] = make_float4(uu[0], uu[1], uu[2], uu[3]);
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t first = wbase + 128u * (uint32_t)i;
            const float q[4] = {q4[i].x, q4[i].y, q4[i].z, q4[i].w};
            const float u[4] = {u4[i].x, u4[i].y, u4[i].z, u4[i].w};
            float qn[4], qr[4];
            uint32_t k[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                qn[e] = apply ? __fmul_rn(q[e], scale) : q[e];  // q *= float(F)  (rrs.cpp:18-21)
                qr[e] = __fmul_rn(qn[e], p.gain);               // q_real = q * gain (wavefront.cpp:396)
                k[e] = stochastic_round(qr[e], u[e]);           // (rrs.cpp:35-45); padding has q = 0, u = 1
            }
            if (nv[i] == 4u) {
                __stcs(reinterpret_cast<float4 *>(p.q_norm + first), make_float4(qn[0], qn[1], qn[2], qn[3]));
                __stcs(reinterpret_cast<float4 *>(p.q_real + first), make_float4(qr[0], qr[1], qr[2], qr[3]));
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if ((uint32_t)e < nv[i]) {
                        p.q_norm[first + e] = qn[e];
                        p.q_real[first + e] = qr[e];
                    }
            }
            gs[i] = k[0] + k[1] + k[2] + k[3];
            kq[i * kD3T + tid] = make_uint4(k[0], k[1], k[2], k[3]);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t first = wbase + 128u * (uint32_t)i;
            uint32_t k[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int32_t c = (uint32_t)e < nv[i] ? p.counts_in[first + e] : 0;
                bad |= c < 0;
                k[e] = c < 0 ? 0u : (uint32_t)c;
            }
            gs[i] = k[0] + k[1] + k[2] + k[3];
            kq[i * kD3T + tid] = make_uint4(k[0], k[1], k[2], k[3]);
        }
        if (bad)
            atomicOr(p.err_flag, 1u);
    }
    stamp(p.dbg, tile, 1);
    // ---- tile scan + prefix ----
    uint32_t excl[4], agg = 0;
    scan4_positions(gs, sm, excl, agg);
    stamp(p.dbg, tile, 2);
    if (warp == 0) {
        const uint64_t ex = tile_prefix(p.tile_state, tile, agg, epoch, p.single_wave != 0u, p.dbg);
        if (lane == 0)
            sm.prefix = ex;
    }
    __syncthreads();
    const uint64_t P = sm.prefix;
    const uint64_t cap = p.capacity;
    stamp(p.dbg, tile, 3);
    // room left in the queue at this tile's first record (positions below are tile-relative)
    const uint32_t room = P < cap ? (uint32_t)min(cap - P, (uint64_t)0xFFFFFFFFu) : 0u;
    const bool vec_out = ((reinterpret_cast<uintptr_t>(p.offset) | reinterpret_cast<uintptr_t>(p.k_out)) & 15u) == 0;
    uint2 *slots = reinterpret_cast<uint2 *>(p.slots) + P;
    uint2 *wbuf = reinterpret_cast<uint2 *>(kq + 4 * kD3T) + warp * kD3Stage;
    // ---- slot records (wavefront.cpp:421-425, :436) and offsets (:148).  A warp's records of one
    // item group are contiguous in the queue and in (item, child) order, so they are staged
    // unclipped at their group-relative position and the capacity clip is a truncation of the
    // copy-out; counts above 4 or groups beyond the staging buffer take the general loop. ----
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t first = wbase + 128u * (uint32_t)i;
        const uint32_t gbase = __shfl_sync(0xffffffffu, excl[i], 0);
        const uint32_t gtot = __shfl_sync(0xffffffffu, excl[i] + gs[i], 31) - gbase;
        const uint4 k4 = kq[i * kD3T + tid];
        const uint32_t kk[4] = {k4.x, k4.y, k4.z, k4.w};
        if (p.slots) {
            const bool big = __any_sync(0xffffffffu, (k4.x | k4.y | k4.z | k4.w) > 4u) || gtot > (uint32_t)kD3Stage;
            uint32_t rel = excl[i] - gbase;
            if (!big) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t j = first + (uint32_t)e + p.parent_base;
#pragma unroll
                    for (uint32_t c = 0; c < 4u; ++c)
                        if (c < kk[e])
                            wbuf[rel + c] = make_uint2(j, c);
                    rel += kk[e];
                }
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t j = first + (uint32_t)e + p.parent_base;
                    const uint32_t pos = excl[i] + (rel - (excl[i] - gbase));  // tile-relative
                    const uint32_t kept = pos < room ? min(kk[e], room - pos) : 0u;
                    for (uint32_t c = 0; c < kept; ++c) {
                        if (rel + c < (uint32_t)kD3Stage) {
                            wbuf[rel + c] = make_uint2(j, c);
                        } else {
                            NRRS_CHECK(P + pos + c < cap, "slot record (direct)", P + pos + c, cap);
                            __stcs(slots + pos + c, make_uint2(j, c));
                        }
                    }
                    rel += kk[e];
                }
            }
            __syncwarp();
            const uint32_t groom = gbase < room ? room - gbase : 0u;
            uint32_t nw = gtot < groom ? gtot : groom;
            nw = nw < (uint32_t)kD3Stage ? nw : (uint32_t)kD3Stage;
            for (uint32_t r = (uint32_t)lane; r < nw; r += 32u) {
                NRRS_CHECK(P + gbase + r < cap, "slot record (staged)", P + gbase + r, cap);
                __stcs(slots + gbase + r, wbuf[r]);
            }
            __syncwarp();
        }
        if (p.offset || p.k_out) {
            uint32_t off[4];
            uint64_t cum = P + excl[i];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                off[e] = (uint32_t)(cum < cap ? cum : cap);  // min(cum, capacity)
                cum += kk[e];
            }
            NRRS_CHECK(nv[i] == 0u || first + nv[i] <= n, "offset / k index", first + nv[i], n);
            if (nv[i] == 4u && vec_out) {
                if (p.offset)
                    *reinterpret_cast<uint4 *>(p.offset + first) = make_uint4(off[0], off[1], off[2], off[3]);
                if (p.k_out)
                    *reinterpret_cast<int4 *>(p.k_out + first) =
                        make_int4((int)kk[0], (int)kk[1], (int)kk[2], (int)kk[3]);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if ((uint32_t)e < nv[i]) {
                        if (p.offset)
                            p.offset[first + e] = off[e];
                        if (p.k_out)
                            p.k_out[first + e] = (int32_t)kk[e];
                    }
            }
        }
    }
    if (tile == p.num_tiles - 1 && tid == 0) {
        const uint64_t total = P + agg;
        if (p.total_out)
            *p.total_out = total;
        if (p.mbox)  // this rank's realized total to every rank (the clip kernel waits on all of them)
            mbox_publish(p.mbox, 1, total);
        if (p.res) {
            const uint64_t spawned = total < cap ? total : cap;
            p.res->total = total;
            p.res->spawned = (uint32_t)spawned;
            p.res->dropped = total - spawned;
            p.res->overflow = total > spawned ? 1u : 0u;
        }
    }
#ifdef NRRS_KERNEL_TIMING
    __syncthreads();
    stamp(p.dbg, tile, 4);
#endif
    if (tid == 0)
        finish_launch(p.sync, p.tile_state, p.state_cap, epoch);
}

// Order-preserving compaction of 8-byte records (slot records, surface pairs) by a used mask
// (wavefront.cpp:488-497), same tile shape as decide3: 16 records and their mask bytes per
// thread in registers, one prefix per tile, kept records staged per warp and written in order.
__global__ void __launch_bounds__(kD3T, 1) compact3_kernel(CompactParams p) {
    __shared__ Scan3Smem sm;
    __shared__ uint2 cbuf[kD3T / 32 * 128];  // per-warp staging of one item group's kept records
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_wait();  // the records and count of the producing kernel (and any earlier compaction)
    if (tid == 0)
        sm.tile = claim_tile_epoch(p.sync, &sm.epoch);
    __syncthreads();
    const uint32_t tile = sm.tile, epoch = sm.epoch;
    stamp(p.dbg, tile, 0);
    uint64_t count64 = p.count;
    if (p.count_in) {
        const uint64_t c = *p.count_in;
        count64 = c < count64 ? c : count64;
    }
    const uint32_t count = min((uint32_t)count64, (tile + 1u) * p.tile_items);
    const uint32_t wbase = tile * p.tile_items + (uint32_t)warp * kD3Warp + 4u * (uint32_t)lane;
    const uint2 *in = reinterpret_cast<const uint2 *>(p.in);
    const bool vec = (reinterpret_cast<uintptr_t>(p.in) & 15u) == 0 && (reinterpret_cast<uintptr_t>(p.used) & 3u) == 0;
    uint32_t m[4];
    uint2 rec[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t first = wbase + 128u * (uint32_t)i;
        const uint32_t nvi = first >= count ? 0u : (count - first < 4u ? count - first : 4u);
        m[i] = 0;
        if (vec && nvi == 4u) {
            const uint32_t w4 = __ldcs(reinterpret_cast<const unsigned int *>(p.used + first));
            const uint4 a = __ldcs(reinterpret_cast<const uint4 *>(in + first));
            const uint4 b = __ldcs(reinterpret_cast<const uint4 *>(in + first) + 1);
            rec[4 * i] = make_uint2(a.x, a.y);
            rec[4 * i + 1] = make_uint2(a.z, a.w);
            rec[4 * i + 2] = make_uint2(b.x, b.y);
            rec[4 * i + 3] = make_uint2(b.z, b.w);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                m[i] |= ((w4 >> (8 * e)) & 0xffu) ? (1u << e) : 0u;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                rec[4 * i + e] = make_uint2(0u, 0u);
                if ((uint32_t)e < nvi && p.used[first + e]) {
                    m[i] |= 1u << e;
                    rec[4 * i + e] = __ldcs(in + first + e);
                }
            }
        }
    }
    uint32_t gs[4], excl[4], agg = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        gs[i] = __popc(m[i]);
    stamp(p.dbg, tile, 1);
    scan4_positions(gs, sm, excl, agg);
    stamp(p.dbg, tile, 2);
    if (warp == 0) {
        const uint64_t ex = tile_prefix(p.tile_state, tile, agg, epoch, p.single_wave != 0u, p.dbg);
        if (lane == 0)
            sm.prefix = ex;
    }
    __syncthreads();
    stamp(p.dbg, tile, 3);
    // a warp's kept records of one item group (<= 128) are contiguous in the output: stage them
    // in the warp's buffer and write them as full warp stores
    uint2 *out = reinterpret_cast<uint2 *>(p.out) + sm.prefix;
    uint2 *wbuf = cbuf + warp * 128;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t gbase = __shfl_sync(0xffffffffu, excl[i], 0);
        const uint32_t gtot = __shfl_sync(0xffffffffu, excl[i] + gs[i], 31) - gbase;
        uint32_t pos = excl[i] - gbase;
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (m[i] & (1u << e))
                wbuf[pos++] = rec[4 * i + e];
        __syncwarp();
        for (uint32_t r = (uint32_t)lane; r < gtot; r += 32u) {
            NRRS_CHECK(sm.prefix + gbase + r < p.count, "compacted record", sm.prefix + gbase + r, p.count);
            __stcs(out + gbase + r, wbuf[r]);
        }
        __syncwarp();
    }
    if (tile == p.num_tiles - 1 && tid == 0)
        *p.count_out = (uint32_t)(sm.prefix + agg);
#ifdef NRRS_KERNEL_TIMING
    __syncthreads();
    stamp(p.dbg, tile, 4);
#endif
    if (tid == 0)
        finish_launch(p.sync, p.tile_state, p.state_cap, epoch);
}

// ===========================================================================
// granular helpers: normalize_factors / realize_counts
// ===========================================================================
__global__ void __launch_bounds__(256) sum_check_kernel(const float *q, uint64_t n, double *parts,
                                                        uint32_t *counter, uint32_t *err, double *sum_out) {
    // the stage's exact fixed-point sum (Fx128), so normalize_factors here and inside the stage agree
    __shared__ Fx128 ws[8];
    __shared__ uint32_t is_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t begin = n * blockIdx.x / gridDim.x, end = n * (blockIdx.x + 1) / gridDim.x;
    Fx128 s{0ull, 0ull};
    uint32_t bad = 0;
    for (uint64_t i = begin + tid; i < end; i += 256) {
        const float v = q[i];
        if (!(v >= 0.0f) || !isfinite(v))
            bad = 1;
        else
            fx_add_q(s, v);
    }
    s = fx_warp_sum(s);
    if (__any_sync(0xffffffffu, bad) && lane == 0)
        atomicOr(err, 1u);
    if (lane == 0)
        ws[warp] = s;
    __syncthreads();
    if (tid == 0) {
        Fx128 t{0ull, 0ull};
        for (int w = 0; w < 8; ++w)
            fx_add(t, ws[w]);
        reinterpret_cast<Fx128 *>(parts)[blockIdx.x] = t;
        __threadfence();
        is_last = atomicAdd(counter, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (!is_last)
        return;
    __threadfence();
    Fx128 t{0ull, 0ull};
    for (uint32_t b = tid; b < gridDim.x; b += 256) {
        const unsigned long long *pp = reinterpret_cast<const unsigned long long *>(parts) + 2 * b;
        fx_add(t, Fx128{__ldcg(pp), __ldcg(pp + 1)});
    }
    t = fx_warp_sum(t);
    if (lane == 0)
        ws[warp] = t;
    __syncthreads();
    if (tid == 0) {
        Fx128 tot{0ull, 0ull};
        for (int w = 0; w < 8; ++w)
            fx_add(tot, ws[w]);
        *sum_out = fx_to_double(tot);
        *counter = 0;
    }
}

// Per-frame ADRRS divisor input (wavefront.cpp:238-243): sum over pixels of the
// f32 luminance of i_acc (left-to-right, no contraction, core.hpp:24-26), in f64,
// per-CTA fixed tree then last-CTA-done reduction in CTA order.
__global__ void __launch_bounds__(256) lum_sum_kernel(const float *i_acc, uint64_t n, double *parts,
                                                      uint32_t *counter, double *sum_out) {
    __shared__ double ws[8];
    __shared__ uint32_t is_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t begin = n * blockIdx.x / gridDim.x, end = n * (blockIdx.x + 1) / gridDim.x;
    double s = 0.0;
    for (uint64_t i = begin + tid; i < end; i += 256)
        s += (double)luminance(i_acc[3 * i], i_acc[3 * i + 1], i_acc[3 * i + 2]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0)
        ws[warp] = s;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w)
            t += ws[w];
        parts[blockIdx.x] = t;
        __threadfence();
        is_last = atomicAdd(counter, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (!is_last)
        return;
    __threadfence();
    if (tid == 0) {
        double t = 0.0;
        for (uint32_t b = 0; b < gridDim.x; ++b)
            t += __ldcg(parts + b);
        *sum_out = t;
        *counter = 0;
    }
}

cudaError_t launch_lum_sum(const float *i_acc, uint64_t n, double *parts, uint32_t *counter, double *sum_out,
                           uint32_t grid, cudaStream_t stream) {
    lum_sum_kernel<<<grid, 256, 0, stream>>>(i_acc, n, parts, counter, sum_out);
    return cudaGetLastError();
}

__global__ void scale_kernel(float *q, uint64_t n, const double *sum, uint64_t n_pixels, const uint32_t *err,
                             double *f_out) {
    if (*err)
        return;
    const double s = *sum;
    if (!(s > 0.0)) {
        if (blockIdx.x == 0 && threadIdx.x == 0)
            *f_out = 1.0;
        return;
    }
    const double f = __ddiv_rn((double)n_pixels, s);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        *f_out = f;
    if (!(f < 1.0))
        return;
    const float sc = __double2float_rn(f);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        q[i] = __fmul_rn(q[i], sc);
}

__global__ void realize_kernel(const float *q, const float *u, int32_t *counts, uint64_t n, uint32_t *err,
                               unsigned long long *total) {
    uint64_t local = 0;
    uint32_t bad = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float v = q[i];
        if (!(v >= 0.0f) || !isfinite(v)) {
            bad = 1;
            counts[i] = 0;
            continue;
        }
        const uint32_t k = stochastic_round(v, u[i]);
        counts[i] = (int32_t)k;
        local += k;
    }
    if (bad)
        atomicOr(err, 1u);
    if (local)
        atomicAdd(total, (unsigned long long)local);
}

// ===========================================================================
// launch wrappers (called from the C ABI layer)
// ===========================================================================
size_t infer_smem_bytes(int kind, const InferParams &p) {
    return kind == kKindHeuristic ? 0 : p.blob_bytes;
}

// Pipeline shape: 2 encoder groups, 3 MLP groups with one tile chain each, 1 thread per row (the
// tuned default; the sweep over other shapes is recorded in DESIGN.md section 3a).
#ifndef NRRS_WS_GE
#define NRRS_WS_GE 2  // fused-gather K-A for NRRS: encoder groups
#endif
#ifndef NRRS_WS_GM
#define NRRS_WS_GM 3  // fused-gather K-A: MLP groups
#endif
#ifndef NRRS_WS4_GE
#define NRRS_WS4_GE 3  // fused-gather K-A for the 4-layer kinds (ADRRS-NN, stats, AID with fp32 tables)
#endif
#ifndef NRRS_WS4_GM
#define NRRS_WS4_GM 2
#endif
#ifndef NRRS_AID_FUSED
#define NRRS_AID_FUSED 8  // K-A over level planes as NRRS_AID_FUSED self-contained groups
#endif
#ifndef NRRS_AID_MMA_HINT
#define NRRS_AID_MMA_HINT 0  // ns suspend hint of the AID K-A MMA-completion wait (0: plain try_wait loop)
#endif
template <int KIND>
static cudaError_t launch_ws_cfg(const InferParams &p, int num_sms, cudaStream_t stream, uint32_t *grid_out) {
    if constexpr (KIND == kKindAid) {
        if (p.rrs_half && p.feat) {
            // K-A0 (level-sliced smem encode) then K-A reading the level planes
            GridLevelParams gp{};
            gp.p01 = p.p01;
            gp.n = p.n;
            gp.table = p.rrs_grid;
            gp.g = p.grid_rrs;
            gp.feat = p.feat;
            gp.feat_stride = p.feat_stride;
            cudaError_t e = launch_grid_levels(gp, num_sms, stream);
            if (e != cudaSuccess)
                return e;
            return launch_aid_fused<NRRS_AID_FUSED>(p, num_sms, stream, grid_out);
        }
        if (p.rrs_half)
            return launch_ws<KIND, NRRS_WS4_GE, NRRS_WS4_GM, 1, 1, true>(p, num_sms, stream, grid_out);
    }
    if constexpr (KIND == kKindAdrrs || KIND == kKindStats || KIND == kKindNrrs) {
        if (p.feat && p.stat_fm) {
            // fp32 StatNet grid from shared memory, one (level, feature) table per CTA, then K-A over
            // the feature planes
            GridLevelParams gp{};
            gp.p01 = p.p01;
            gp.n = p.n;
            gp.table = p.stat_fm;
            gp.g = p.grid;
            gp.feat = p.feat;
            gp.feat_stride = p.feat_stride;
            gp.f32 = 1;
            cudaError_t e = launch_grid_levels(gp, num_sms, stream);
            if (e != cudaSuccess)
                return e;
            return launch_stat_planes<KIND>(p, num_sms, stream, grid_out);
        }
    }
    // NRRS chains 8 MMA layers per tile (StatNet then RRSNet): 2 encoder + 3 MLP groups; the 4-layer
    // kinds are gather-bound and run 3 encoder + 2 MLP groups (ADRRS-NN 0.397 -> 0.377 ms)
    if constexpr (KIND == kKindNrrs)
        return launch_ws<KIND, NRRS_WS_GE, NRRS_WS_GM, 1, 1, false>(p, num_sms, stream, grid_out);
    else
        return launch_ws<KIND, NRRS_WS4_GE, NRRS_WS4_GM, 1, 1, false>(p, num_sms, stream, grid_out);
}

cudaError_t launch_infer(int kind, const InferParams &p, int num_sms, cudaStream_t stream, uint32_t *grid_out) {
    switch (kind) {
    case kKindAdrrs: return launch_ws_cfg<kKindAdrrs>(p, num_sms, stream, grid_out);
    case kKindNrrs: return launch_ws_cfg<kKindNrrs>(p, num_sms, stream, grid_out);
    case kKindAid: return launch_ws_cfg<kKindAid>(p, num_sms, stream, grid_out);
    case kKindStats: return launch_ws_cfg<kKindStats>(p, num_sms, stream, grid_out);
    default: break;
    }
    int occ = 1;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, infer_kernel, kInferThreads, 0);
    if (e != cudaSuccess)
        return e;
    uint64_t grid = (uint64_t)num_sms * (uint64_t)(occ < 1 ? 1 : occ);
    const uint64_t blocks = (p.n + kInferThreads - 1) / kInferThreads;
    if (grid > blocks)
        grid = blocks;
    if (grid < 1)
        grid = 1;
    *grid_out = (uint32_t)grid;
    infer_kernel<<<(uint32_t)grid, kInferThreads, 0, stream>>>(p);
    return cudaGetLastError();
}

uint32_t infer_max_grid(int num_sms) { return (uint32_t)num_sms * 16u; }

// Tile shape of decide3 / compact3: batches up to num_sms full tiles run as one wave with the
// items spread evenly over the SMs (512-item warp granularity); larger ones use full tiles.  Small
// batches keep at least kD3MinItems per tile: the warps of a CTA run side by side, while every
// extra tile lengthens the look-back and adds a CTA launch (C1: 8 tiles of 16 warps, not 128 of 1).
#ifndef NRRS_D3_MIN_ITEMS
#define NRRS_D3_MIN_ITEMS 8192
#endif
constexpr uint64_t kD3MinItems = NRRS_D3_MIN_ITEMS;
static void scan_tile_shape(uint64_t n, int num_sms, uint32_t *items, uint32_t *tiles, uint32_t *single) {
    const uint64_t sms = num_sms < 1 ? 1 : (uint64_t)num_sms;
    if (n <= sms * (uint64_t)kD3Tile && sms <= 256) {
        uint64_t per = (n + sms - 1) / sms;
        if (per < kD3MinItems)
            per = kD3MinItems;
        per = (per + kD3Warp - 1) / kD3Warp * kD3Warp;
        if (per == 0)
            per = kD3Warp;
        *items = (uint32_t)per;
        *tiles = (uint32_t)((n + per - 1) / per);
        *single = 1u;
    } else {
        *items = (uint32_t)kD3Tile;
        *tiles = (uint32_t)((n + kD3Tile - 1) / kD3Tile);
        *single = 0u;
    }
}

uint32_t decide_tiles(uint64_t n) {
    // state entries: full tiles (several waves), or <= 256 padded single-wave tiles
    const uint64_t full = (n + kD3Tile - 1) / kD3Tile, one_wave = 256u * kStatePad;
    return (uint32_t)(full > one_wave ? full : one_wave);
}

cudaError_t launch_decide(int src, DecideParams p, int num_sms, cudaStream_t stream) {
    if (p.n == 0)
        return cudaSuccess;
    scan_tile_shape(p.n, num_sms, &p.tile_items, &p.num_tiles, &p.single_wave);
    const int smem = 4 * kD3T * (int)sizeof(uint4) + (kD3T / 32) * kD3Stage * (int)sizeof(uint2);
    cudaError_t e;
    if (src == 0) {
        e = cudaFuncSetAttribute(decide3_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess)
            e = launch_maybe_pdl(decide3_kernel<0>, p.num_tiles, kD3T, smem, stream, p);
    } else {
        e = cudaFuncSetAttribute(decide3_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess)
            decide3_kernel<1><<<p.num_tiles, kD3T, smem, stream>>>(p);
    }
    if (e != cudaSuccess)
        return e;
    return cudaGetLastError();
}

template <int W, int IPT>
static size_t compact2_smem() {
    return (size_t)kBT * IPT * W * 4 + kBSubs * kBT + (kBT / 32 + 2) * 4 + 16 + 16;
}

uint32_t compact_tiles(uint64_t count, uint32_t words) {
    if (words == 2)
        return decide_tiles(count);
    const uint64_t tile = (uint64_t)kBT * 1 * kBSubs;
    return (uint32_t)((count + tile - 1) / tile);
}

cudaError_t launch_compact(uint32_t words, CompactParams p, int num_sms, cudaStream_t stream) {
    if (p.count == 0)
        return cudaSuccess;
    if (words == 2) {
        scan_tile_shape(p.count, num_sms, &p.tile_items, &p.num_tiles, &p.single_wave);
        const cudaError_t ce = launch_maybe_pdl(compact3_kernel, p.num_tiles, kD3T, 0, stream, p);
        if (ce != cudaSuccess)
            return ce;
    } else if (words == 18) {
        p.num_tiles = compact_tiles(p.count, words);
        const size_t smem = compact2_smem<18, 1>();
        cudaFuncSetAttribute(compact2_kernel<18, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        compact2_kernel<18, 1><<<p.num_tiles, kBT, smem, stream>>>(p);
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// Device-side table copies for nrrs_gpu_set_weights_dev (the layout set_weights builds on the host,
// see GridDev): copy 0 = the reference layout; for hashed levels copy t stores entry e at
// pair_pos(e, t) (when 2^(t+1) <= T); for dense levels copy 1 is shifted by one entry.  dst is
// zeroed by the caller; half: fp16 entries.
__global__ void grid_copies_kernel(const float2 *src, void *dst, uint32_t levels, uint32_t T, uint32_t copies,
                                   uint32_t dense_mask, int half) {
    const uint64_t per_copy = (uint64_t)levels * T, total = per_copy * copies;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = (uint32_t)(i / per_copy);
        const uint64_t rem = i % per_copy;
        const uint32_t l = (uint32_t)(rem / T), e = (uint32_t)(rem % T);
        const float2 *lv = src + (uint64_t)l * T;
        uint64_t pos;
        float2 v;
        if (t == 0) {
            pos = e;
            v = lv[e];
        } else if ((dense_mask >> l) & 1u) {
            if (t != 1 || e + 1 >= T)
                continue;
            pos = e;
            v = lv[e + 1];
        } else if ((2ull << t) <= T) {
            pos = pair_pos(e, t);
            v = lv[e];
        } else {
            continue;
        }
        const uint64_t o = (uint64_t)t * per_copy + (uint64_t)l * T + pos;
        if (half)
            reinterpret_cast<__half2 *>(dst)[o] = __floats2half2_rn(v.x, v.y);
        else
            reinterpret_cast<float2 *>(dst)[o] = v;
    }
}

__global__ void max_abs_kernel(const float *x, uint64_t n, unsigned int *out_bits) {
    float m = 0.0f;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float a = fabsf(x[i]);
        m = (a > m || a != a) ? (a != a ? __int_as_float(0x7f800000) : a) : m;  // NaN counts as +inf
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0)
        atomicMax(out_bits, __float_as_uint(m));  // non-negative floats order like their bits
}

// Feature-major copy [level][feature][T] of a [level][T][feature] fp32 grid (grid_level_kernel<true>).
__global__ void feature_major_kernel(const float2 *src, float *dst, uint32_t levels, uint32_t T) {
    const uint64_t total = (uint64_t)levels * T;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t l = i / T, e = i % T;
        const float2 v = src[i];
        dst[(2 * l) * T + e] = v.x;
        dst[(2 * l + 1) * T + e] = v.y;
    }
}

cudaError_t launch_feature_major(const float *src, float *dst, uint32_t levels, uint32_t T, cudaStream_t stream) {
    feature_major_kernel<<<512, 256, 0, stream>>>(reinterpret_cast<const float2 *>(src), dst, levels, T);
    return cudaGetLastError();
}

cudaError_t launch_grid_copies(const float *src, void *dst, uint32_t levels, uint32_t T, uint32_t copies,
                               uint32_t dense_mask, bool half, cudaStream_t stream) {
    grid_copies_kernel<<<1024, 256, 0, stream>>>(reinterpret_cast<const float2 *>(src), dst, levels, T, copies,
                                                 dense_mask, half ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_max_abs(const float *x, uint64_t n, unsigned int *out_bits, cudaStream_t stream) {
    max_abs_kernel<<<256, 256, 0, stream>>>(x, n, out_bits);
    return cudaGetLastError();
}

cudaError_t launch_sum_check(const float *q, uint64_t n, double *parts, uint32_t *counter, uint32_t *err,
                             double *sum_out, uint32_t grid, cudaStream_t stream) {
    sum_check_kernel<<<grid, 256, 0, stream>>>(q, n, parts, counter, err, sum_out);
    return cudaGetLastError();
}

cudaError_t launch_scale(float *q, uint64_t n, const double *sum, uint64_t n_pixels, const uint32_t *err,
                         double *f_out, int num_sms, cudaStream_t stream) {
    scale_kernel<<<num_sms * 4, 256, 0, stream>>>(q, n, sum, n_pixels, err, f_out);
    return cudaGetLastError();
}

cudaError_t launch_realize(const float *q, const float *u, int32_t *counts, uint64_t n, uint32_t *err,
                           unsigned long long *total, int num_sms, cudaStream_t stream) {
    realize_kernel<<<num_sms * 4, 256, 0, stream>>>(q, u, counts, n, err, total);
    return cudaGetLastError();
}

}  // namespace nrrs
