// nrrs_ka.cuh -- device pieces shared by the K-A / K-B / K-C kernels (nrrs_kernels.cu) and the
// fused AID stage kernel (nrrs_fused.cu): the fp16 hi/lo split, tolerance-path encodings, the
// shared-memory hash-grid level encode, the tcgen05 layer issue / epilogue helpers, the AID
// input-slot layout, and the register-resident scan / tile-prefix helpers.
#pragma once

#include "nrrs_device.cuh"
#include "nrrs_internal.h"

namespace nrrs {

constexpr int kTileM = 128;           // vertices per MMA tile (UMMA M)

// fp32 -> fp16 hi/lo split of two values (x = hi + lo to ~22 bits).  The
// residual is produced NEGATED, l = f16(hi - x): sm_100's mixed-precision subtract (f16 operand
// minus f32, one FHADD per element) replaces unpacking hi to fp32 plus an fp32x2 subtract, and
// hi - x is exact in fp32 either way.  Every MMA that consumes the lo operand sets the
// instruction descriptor's negate-A bit (kIdescNegA), so the products are bit-identical.
#ifndef NRRS_NEG_LO
#define NRRS_NEG_LO 1
#endif
constexpr bool kNegLo = NRRS_NEG_LO != 0;
constexpr uint32_t kIdescNegA = kNegLo ? (1u << 13) : 0u;  // tcgen05 instruction descriptor: negate A
__device__ __forceinline__ void split2(float v0, float v1, uint32_t &h, uint32_t &l) {
    const __half2 hh = __float22half2_rn(make_float2(v0, v1));
    h = *reinterpret_cast<const uint32_t *>(&hh);
    if (kNegLo) {
        float r0, r1;
        asm("{\n\t.reg .f16 a, b;\n\tmov.b32 {a, b}, %2;\n\t"
            "sub.rn.f32.f16 %0, a, %3;\n\tsub.rn.f32.f16 %1, b, %4;\n\t}"
            : "=f"(r0), "=f"(r1)
            : "r"(h), "f"(v0), "f"(v1));
        const __half2 ll = __float22half2_rn(make_float2(r0, r1));
        l = *reinterpret_cast<const uint32_t *>(&ll);
    } else {
        const float2 b = __half22float2(hh);
        const __half2 ll = __float22half2_rn(upk2(fsub2(pk2(v0, v1), pk2(b.x, b.y))));
        l = *reinterpret_cast<const uint32_t *>(&ll);
    }
}


// one_blob_encode (encodings.hpp:31-44), tolerance path: exp(-d^2 / (2 sigma^2)) as one
// flush-to-zero ex2 per bin with log2(e) folded into the constant, approximate reciprocal.
template <int BINS>
__device__ __forceinline__ void one_blob_fast(float x, float *out) {
    constexpr float k = -(float)(BINS * BINS) * 0.5f * 1.4426950408889634f;
    float sum = 0.0f;
#pragma unroll
    for (int i = 0; i < BINS; ++i) {
        const float d = x - ((float)i + 0.5f) / (float)BINS;
        out[i] = ex2_ftz(d * d * k);
        sum += out[i];
    }
    const float inv = rcp_ftz(sum);
#pragma unroll
    for (int i = 0; i < BINS; ++i)
        out[i] *= inv;
}

__device__ __forceinline__ float remap_fast(float a) { return 1.0f - ex2_ftz(a * -1.4426950408889634f); }


// (a ^ b) & c in one LOP3.
__device__ __forceinline__ uint32_t lop3_xor_and(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Per-level constants of K-A0 (uniform over the CTA).
struct LevelConsts {
    uint32_t res, nn, m4;  // resolution, res + 1, (T - 1) * 4
    float resf;
    bool dense;
    uint32_t doff4[8];     // dense corner offsets * 4
};

// One level of HashGrid::encode for one point from the shared-memory table
// (hashgrid.cpp:38-82): cell and weights per axis, 8 corner entries (byte offsets
// idx * 4: the hash is computed on pre-scaled terms, ((a ^ b) & m) * 4 =
// (4a ^ 4b) & 4m), weights w = wx * (wy * wz) as x-pairs, (f0, f1) accumulated as
// one fp32x2 FMA per corner.
__device__ __forceinline__ float2 level_encode(const uint8_t *tab, const LevelConsts &c, float px, float py,
                                               float pz) {
    const float fx = __saturatef(px) * c.resf, fy = __saturatef(py) * c.resf, fz = __saturatef(pz) * c.resf;
    const uint32_t cx = min((uint32_t)fx, c.res - 1u);
    const uint32_t cy = min((uint32_t)fy, c.res - 1u);
    const uint32_t cz = min((uint32_t)fz, c.res - 1u);
    const float tx = fx - (float)cx, ty = fy - (float)cy, tz = fz - (float)cz;
    const uint64_t wxp = pk2(1.0f - tx, tx);
    const float wy[2] = {1.0f - ty, ty}, wz[2] = {1.0f - tz, tz};
    uint32_t idx4[8];
    if (c.dense) {
        const uint32_t b4 = ((cx * c.nn + cy) * c.nn + cz) * 4u;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            idx4[k] = b4 + c.doff4[k];
    } else {
        const uint32_t hx0 = cx * 4u, hx1 = hx0 + 4u;
        const uint32_t hy0 = cy * (2654435761u * 4u), hy1 = hy0 + 2654435761u * 4u;
        const uint32_t hz0 = cz * (805459861u * 4u), hz1 = hz0 + 805459861u * 4u;
        const uint32_t hyz[4] = {hy0 ^ hz0, hy1 ^ hz0, hy0 ^ hz1, hy1 ^ hz1};
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // (hx ^ hyz) & m as one LOP3 each (nvcc splits it into two)
            idx4[2 * q] = lop3_xor_and(hx0, hyz[q], c.m4);
            idx4[2 * q + 1] = lop3_xor_and(hx1, hyz[q], c.m4);
        }
    }
    uint32_t raw[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        NRRS_CHECK(idx4[k] <= c.m4 || (c.dense && idx4[k] < c.nn * c.nn * c.nn * 4u), "level table index", idx4[k], c.m4);
        raw[k] = *reinterpret_cast<const uint32_t *>(tab + idx4[k]);
    }
    uint64_t acc[2] = {pk2(0.0f, 0.0f), pk2(0.0f, 0.0f)};  // oz = 0 / 1 (two short FMA chains)
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // corners (0, oy, oz), (1, oy, oz); q = oy + 2 oz
        const float2 w = upk2(fmul2(wxp, pk2(wy[q & 1] * wz[q >> 1], wy[q & 1] * wz[q >> 1])));
        const float2 v0 = __half22float2(*reinterpret_cast<const __half2 *>(&raw[2 * q]));
        const float2 v1 = __half22float2(*reinterpret_cast<const __half2 *>(&raw[2 * q + 1]));
        acc[q >> 1] = ffma2(pk2(w.x, w.x), pk2(v0.x, v0.y), acc[q >> 1]);
        acc[q >> 1] = ffma2(pk2(w.y, w.y), pk2(v1.x, v1.y), acc[q >> 1]);
    }
    return upk2(fadd2(acc[0], acc[1]));
}

// One feature of one level from a shared-memory fp32 table (the StatNet grid's feature-major copy):
// the same cell, weights and corner indices as level_encode, 8 scalar loads and FMAs.
__device__ __forceinline__ float level_encode_f32(const uint8_t *tab, const LevelConsts &c, float px, float py,
                                                  float pz) {
    const float fx = __saturatef(px) * c.resf, fy = __saturatef(py) * c.resf, fz = __saturatef(pz) * c.resf;
    const uint32_t cx = min((uint32_t)fx, c.res - 1u);
    const uint32_t cy = min((uint32_t)fy, c.res - 1u);
    const uint32_t cz = min((uint32_t)fz, c.res - 1u);
    const float tx = fx - (float)cx, ty = fy - (float)cy, tz = fz - (float)cz;
    const float wx[2] = {1.0f - tx, tx}, wy[2] = {1.0f - ty, ty}, wz[2] = {1.0f - tz, tz};
    uint32_t idx4[8];
    if (c.dense) {
        const uint32_t b4 = ((cx * c.nn + cy) * c.nn + cz) * 4u;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            idx4[k] = b4 + c.doff4[k];
    } else {
        const uint32_t hx0 = cx * 4u, hx1 = hx0 + 4u;
        const uint32_t hy0 = cy * (2654435761u * 4u), hy1 = hy0 + 2654435761u * 4u;
        const uint32_t hz0 = cz * (805459861u * 4u), hz1 = hz0 + 805459861u * 4u;
        const uint32_t hyz[4] = {hy0 ^ hz0, hy1 ^ hz0, hy0 ^ hz1, hy1 ^ hz1};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            idx4[2 * q] = lop3_xor_and(hx0, hyz[q], c.m4);
            idx4[2 * q + 1] = lop3_xor_and(hx1, hyz[q], c.m4);
        }
    }
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        NRRS_CHECK(idx4[k] <= c.m4 || (c.dense && idx4[k] < c.nn * c.nn * c.nn * 4u), "f32 level table index", idx4[k], c.m4);
        v[k] = *reinterpret_cast<const float *>(tab + idx4[k]);
    }
    float a0 = 0.0f, a1 = 0.0f;  // oz = 0 / 1 (two short FMA chains)
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // corners (0, oy, oz), (1, oy, oz); q = oy + 2 oz
        const float wyz = wy[q & 1] * wz[q >> 1];
        float &acc = (q >> 1) ? a1 : a0;
        acc = fmaf(wx[0] * wyz, v[2 * q], acc);
        acc = fmaf(wx[1] * wyz, v[2 * q + 1], acc);
    }
    return a0 + a1;
}


// The launch's exact sum of q -> the call's running total (chunked host paths add their chunks in
// any order with the same bits), written back to res->sum_fx; returns it as double.
__device__ __forceinline__ double fx_finish(const InferParams &p, Fx128 launch_total) {
    if (p.accumulate)
        fx_add(launch_total, Fx128{p.res->sum_fx[0], p.res->sum_fx[1]});
    p.res->sum_fx[0] = launch_total.lo;
    p.res->sum_fx[1] = launch_total.hi;
    return fx_to_double(launch_total);
}

namespace ws {

struct Side {        // 32 B per tile row
    uint64_t key;
    uint32_t flags;  // bit0 valid, bit1 active
    float ex[5];     // NRRS: bc(t_x)x3, bc(mean I), remap(r); ADRRS: w x3, lum(I)
};

// TMEM (512 columns, 1 CTA / SM): one 64-column fp32 accumulator per MLP chain,
// [64c, 64c + 64): columns [0, N) collect A_hi*W_hi + A_lo*W_hi and [N, 2N)
// collect A_hi*W_lo (one N = 2N instruction covers both weight halves); then a
// ring of tile slots [kColSlots + 32s, +32) holding the layer-0 input
// (hi 16 | lo 16 packed fp16x2 columns), reused as the hidden-layer A.
// NRRS_MMA3 = 1: three N-wide MMAs per K16 slice accumulate A_hi*W_hi + A_lo*W_hi +
// A_hi*W_lo into ONE 32-column accumulator (same tensor work as the N = 2N form; the
// epilogue reads half the TMEM columns and skips the hi + lo add).
#ifndef NRRS_MMA_WAIT_HINT
#define NRRS_MMA_WAIT_HINT 0  // ns suspend hint of the MLP groups' MMA-completion wait (0: plain try_wait loop)
#endif
#ifndef NRRS_MMA3
#define NRRS_MMA3 1
#endif
constexpr bool kMma3 = NRRS_MMA3 != 0;
constexpr uint32_t kDCols = kMma3 ? 32u : 64u;

template <int GE, int GM, int P, int TPR>
struct Cfg {
    static constexpr int kGroupThreads = 128 * TPR;  // MLP threads per group (TPR threads per tile row)
    static constexpr int kEncThreads = GE * 256;
    static constexpr int kMlpThreads = GM * kGroupThreads;
    static constexpr int kThreads = kEncThreads + kMlpThreads;
    static constexpr int kChains = GM * P;
    static constexpr uint32_t kColD = 0;
    static constexpr uint32_t kColSlots = kDCols * kChains;
    static constexpr int kSlotsRaw = (512 - (int)kColSlots) / 32;
    static constexpr int kSlots = kSlotsRaw > 16 ? 16 : kSlotsRaw;
    static_assert(kSlots >= GE + kChains, "TMEM slot ring too small");
};

struct SmemTail {
    uint64_t full[16];
    uint64_t empty[16];
    uint64_t mma_bar[8];
    uint64_t wdesc[2][4][2];   // UMMA smem descriptor of [W_hi ; W_lo] per K16 slice (W_hi alone = first N rows)
    uint64_t wdesc_lo[2][4][2];  // W_lo alone (rows N .. 2N)
    uint32_t idesc_n[2][4];    // N = layer width
    uint32_t idesc_2n[2][4];   // N = 2 x layer width (both weight halves)
    uint32_t nslices[2][4];
    uint32_t bias[2][4];       // smem byte offset of the fp32 bias, or kNoBias (folded into W)
    uint32_t tmem_base;
    uint32_t is_last;
    Fx128 red_fx[32];
    uint32_t red_nf[32];
    uint32_t red_bc[32];
};

// Elected issue of one layer, 2 MMAs per K16 slice, commit to the chain's mbarrier:
//   D[:, 0:2N]  (+)= A_hi x [W_hi | W_lo]    (N = 2N: hi*W_hi and hi*W_lo side by side)
//   D[:, 0:N]    += A_lo x W_hi
// The epilogue adds the two column halves (3-term split).
// Caller has synchronized the group.
__device__ __forceinline__ void ws_issue(const SmemTail *st, int net, int layer, uint32_t tmem_base,
                                         uint32_t col_a, uint32_t col_d, uint64_t *bar) {
    tc_fence_after();
    const uint32_t i2 = st->idesc_2n[net][layer], i1 = st->idesc_n[net][layer];
    const uint32_t ns = st->nslices[net][layer];
    const uint32_t d = tmem_base + col_d;
#pragma unroll
    for (uint32_t k = 0; k < 2; ++k) {
        if (k >= ns)
            break;
        const uint64_t w = st->wdesc[net][layer][k];
        const uint32_t ah = tmem_base + col_a + 8u * k, al = ah + 16u;
        if (kMma3) {
            mma_f16_ts(d, ah, w, i1, k > 0 ? 1u : 0u);
            mma_f16_ts(d, al, w, i1 | kIdescNegA, 1u);  // A_lo holds -lo (split2)
            mma_f16_ts(d, ah, st->wdesc_lo[net][layer][k], i1, 1u);
        } else {
            mma_f16_ts(d, ah, w, i2, k > 0 ? 1u : 0u);
            mma_f16_ts(d, al, w, i1 | kIdescNegA, 1u);
        }
    }
    mma_commit(bar);
}

// 16 fp32 values (K columns [16h, 16h + 16) of the next A) -> 8 hi + 8 lo packed
// fp16x2 TMEM columns of this thread's lane.
__device__ __forceinline__ void ws_store_a16(uint32_t lane_base, uint32_t col_a, int h, const float (&x)[16]) {
    uint32_t hw[8], lw[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
        split2(x[2 * e], x[2 * e + 1], hw[e], lw[e]);
    tmem_st8(lane_base + col_a + 8u * (uint32_t)h, hw);
    tmem_st8(lane_base + col_a + 16u + 8u * (uint32_t)h, lw);
}

// 16 accumulator columns [c0, c0 + 16) of this lane: D_hi + D_lo (+ bias), fp32
// (element order of the scalar form; the adds run as fp32x2 pairs).
__device__ __forceinline__ void ws_load_sum16(uint32_t lane_base, uint32_t col_d, uint32_t n, uint32_t c0,
                                              const float *bias, float (&z)[16]) {
    float lo[16];
    if (kMma3)
        tmem_ld16(lane_base + col_d + c0, z);
    else
        tmem_ld16x2(lane_base + col_d + c0, lane_base + col_d + n + c0, z, lo);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        uint64_t v = pk2(z[2 * i], z[2 * i + 1]);
        if (!kMma3)
            v = fadd2(v, pk2(lo[2 * i], lo[2 * i + 1]));
        if (bias) {  // 16-byte bias loads (the blob keeps every bias 64-byte aligned)
            const float4 b4 = reinterpret_cast<const float4 *>(bias + c0)[i >> 1];
            v = fadd2(v, (i & 1) ? pk2(b4.z, b4.w) : pk2(b4.x, b4.y));
        }
        const float2 f = upk2(v);
        z[2 * i] = f.x;
        z[2 * i + 1] = f.y;
    }
}

// Head output y[0] only (RRSNet has one output; the N = 16 accumulator's other columns are
// padding): one TMEM column instead of sixteen.
__device__ __forceinline__ float ws_load_head1(uint32_t lane_base, uint32_t col_d, const float *bias) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(lane_base + col_d));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const float y = __uint_as_float(r);
    return bias ? y + bias[0] : y;
}

}  // namespace ws

// Per-group input slot of infer_aid_fused_kernel (one 128-row tile, field-major so each
// thread's row reads are bank-conflict free): 8 level planes (float2), weight (3 f32),
// wo01 (2 f32), i_pixel (3 f32; or the u32 pixel index), roughness, path_key.
constexpr uint32_t kAidInPlane = 8u * kTileM;
constexpr uint32_t kAidInWeight = 8u * kAidInPlane;
constexpr uint32_t kAidInWo = kAidInWeight + 12u * kTileM;
constexpr uint32_t kAidInIpx = kAidInWo + 8u * kTileM;
constexpr uint32_t kAidInRough = kAidInIpx + 12u * kTileM;
constexpr uint32_t kAidInKey = kAidInRough + 4u * kTileM;
constexpr uint32_t kAidInBytes = kAidInKey + 8u * kTileM;
static_assert(kAidInBytes % 128u == 0, "slot alignment");
__host__ __device__ constexpr uint32_t aid_in_offset(uint32_t blob_bytes) {
    return ((blob_bytes + 127u) & ~127u) + (((uint32_t)sizeof(ws::SmemTail) + 127u) & ~127u);
}


constexpr int kD3T = 1024;            // threads
constexpr int kD3Tile = kD3T * 16;    // items per full tile
constexpr int kD3Warp = 512;          // items per warp
constexpr int kD3Stage = 256;         // staged slot records per warp and item group (2 KB)

__device__ __forceinline__ void stamp(unsigned long long *dbg, uint32_t tile, int k) {
#ifdef NRRS_KERNEL_TIMING
    if (dbg && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        dbg[tile * 8 + k] = t;
    }
#endif
}

struct Scan3Smem {
    uint32_t warp_tot[kD3T / 32];
    unsigned long long prefix;
    uint32_t tile, epoch;
};

// Tile-relative exclusive position of this lane's first item of each group (items in (warp, i,
// lane, e) order) from the per-group lane sums s[i]; the tile total in `agg`.
__device__ __forceinline__ void scan4_positions(const uint32_t (&s)[4], Scan3Smem &sm, uint32_t (&excl)[4],
                                                uint32_t &agg) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t run = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t inc = s[i];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o)
                inc += t;
        }
        excl[i] = run + inc - s[i];
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0)
        sm.warp_tot[warp] = run;
    __syncthreads();
    const uint32_t t = lane < (int)(blockDim.x >> 5) ? sm.warp_tot[lane] : 0u;
    uint32_t before = lane < warp ? t : 0u, all = t;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        before += __shfl_xor_sync(0xffffffffu, before, o);
        all += __shfl_xor_sync(0xffffffffu, all, o);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
        excl[i] += before;
    agg = all;
}

// Exclusive prefix of `tile` (warp 0, every lane gets it).  single_wave: every tile of the launch
// is resident, so the prefix is the sum of all predecessors' aggregates, read at once; each tile's
// state word sits on its own 128-byte line (kStatePad) so the ~N^2 / 2 polls spread over N L2
// lines instead of hammering a few.
constexpr uint32_t kStatePad = 16;
__device__ __forceinline__ uint64_t tile_prefix(uint64_t *state, uint32_t tile, uint64_t agg, uint32_t epoch,
                                                bool single_wave, unsigned long long *dbg = nullptr) {
    NRRS_CHECK(!single_wave || tile < 256u, "single-wave tile", tile, 256u);
    if (!single_wave)
        return lookback_warp(state, tile, agg, epoch);
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t tag = (uint64_t)(epoch & 0x3FFFu) << 48;
    if (lane == 0)
        st_relaxed_u64(&state[tile * kStatePad], kFlagAgg | tag | agg);
    // up to 8 predecessors per lane (single wave: <= 256 tiles), requested together
    const uint32_t ep = epoch & 0x3FFFu;
    uint64_t st[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const uint32_t t = lane + 32u * (uint32_t)r;
        st[r] = t < tile ? ld_relaxed_u64(&state[t * kStatePad]) : 0ull;
    }
    uint64_t v = 0;
    uint32_t polls = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const uint32_t t = lane + 32u * (uint32_t)r;
        if (t < tile) {
            while ((st[r] >> 62) == 0 || ((st[r] >> 48) & 0x3FFFu) != ep) {
                st[r] = ld_relaxed_u64(&state[t * kStatePad]);
                ++polls;
            }
            v += st[r] & kValueMask;
        }
    }
#ifdef NRRS_KERNEL_TIMING
    polls = __reduce_max_sync(0xffffffffu, polls);
    if (dbg && lane == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        dbg[tile * 8 + 5] = t1;
        dbg[tile * 8 + 6] = polls + 1;
    }
#else
    (void)polls;
#endif
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}


}  // namespace nrrs
