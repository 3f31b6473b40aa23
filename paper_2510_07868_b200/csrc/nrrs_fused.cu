// nrrs_fused.cu -- the AID-NRRS stage as ONE persistent kernel (K-F) on sm_100a.
//
// One CTA per SM, all CTAs co-resident (cooperative launch).  Each CTA plays three roles at once
// on disjoint warps, then all of its warps run the decision tail:
//
//   producers (15 warps)  HashGrid::encode of ONE level (hashgrid.cpp:38-82) from that level's
//                         fp16 table staged in shared memory (CTA b serves level b % L), for the
//                         tiles of a round of consumer CTAs; features go to an L2-resident ring
//                         of level planes (3 rounds deep), so they never reach HBM.
//   loader (1 warp)       waits for a round's planes (global produced-counter, acquire), TMA
//                         bulk-copies each MLP group's next tile (8 plane segments + row inputs)
//                         into the group's shared-memory slot, and hands ring slots back
//                         (consumed-counter) once the copies landed.
//   MLP groups (4 x 4 warps) build_aid_tail (networks.cpp:149-157) + the 4-layer RRSNet on
//                         tcgen05 (mlp.cpp:52-72; 3-term fp16 split, A in TMEM) + softplus,
//                         sanitize, Mix-Depth gate (wavefront.cpp:363-389) and the RrsRound
//                         uniform (wavefront.cpp:397-399); q and u are parked in TMEM columns.
//   decision tail         grid barrier on the per-CTA double partials of q (fixed order, so
//                         every CTA derives the same F = Npx / sum, rrs.cpp:8-24), then each CTA
//                         normalizes, applies the gain and rounds its own contiguous tile range
//                         straight out of TMEM (rrs.cpp:35-45), takes its exclusive prefix as the
//                         sum of its predecessors' published counts, and writes q_norm, q_real,
//                         the offsets and the (parent, child) slot records with the capacity clip
//                         (wavefront.cpp:141-154, :421-425).  q and u never leave the chip.
//
// Tile ownership: CTA b owns tiles [b * tpc, (b + 1) * tpc) (a contiguous vertex range, so its
// decision scan is local); in round r its MLP group m takes local tile r * GM + m.  The producer
// of level l with index q (of nq CTAs serving l) encodes, each round, the round's tiles of
// consumer CTAs [G q / nq, G (q + 1) / nq).
#include "nrrs_device.cuh"
#include "nrrs_internal.h"
#include "nrrs_ka.cuh"

#include <cuda_runtime.h>

namespace nrrs {
namespace fused {

// Warp roles.  The issue arbiter prefers higher warp ids, so the MLP groups (the latency-bound
// tile chains) take the top warps and the producers (plenty of independent gathers) fill in.
constexpr int kGM = 4;                       // MLP groups (4 warps each): warps 16..31
constexpr int kThreads = 1024;
constexpr int kMlpWarp0 = 32 - 4 * kGM;      // 16
constexpr int kLoaderWarp = kMlpWarp0 - 1;   // 15
constexpr int kProdThreads = kLoaderWarp * 32;  // warps 0..14: 480 producer threads
constexpr int kRoundSlots = 3;               // ring depth in rounds
constexpr uint32_t kParkCol = 64u * kGM;     // first TMEM column of the parked (q, u) pairs
constexpr uint32_t kMaxParkTiles = (512u - kParkCol) / 2u;  // 128 tiles per CTA
constexpr int kProdPer = 3;                  // vertices per producer thread in flight
constexpr int kStage = 256;                  // staged slot records per warp
constexpr uint32_t kPad = 32;                // u32 words between counters (128-byte lines)

struct Smem {  // after the weight blob
    ws::SmemTail st;
    uint64_t full[kGM];       // loader -> group: the tile's inputs landed
    uint64_t slot_free[kGM];  // group -> loader: the group has consumed its input slot
    uint64_t table_bar;
    Fx128 red_fx[32];
    uint32_t red_nf[32], red_bc[32];
    uint32_t cta_total;
    unsigned long long prefix;
    double sum_all;
    uint32_t gen1;
};

__host__ __device__ constexpr uint32_t smem_offset_tail(uint32_t blob_bytes) { return (blob_bytes + 127u) & ~127u; }
__host__ __device__ constexpr uint32_t smem_offset_slots(uint32_t blob_bytes) {
    return smem_offset_tail(blob_bytes) + (((uint32_t)sizeof(Smem) + 127u) & ~127u);
}
__host__ __device__ constexpr uint32_t smem_offset_table(uint32_t blob_bytes) {
    return smem_offset_slots(blob_bytes) + (uint32_t)kGM * kAidInBytes;
}

__device__ __forceinline__ void tmem_st2(uint32_t taddr, float a, float b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(__float_as_uint(a)),
                 "r"(__float_as_uint(b))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, float &a, float &b) {
    uint32_t x, y;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    a = __uint_as_float(x);
    b = __uint_as_float(y);
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(uint32_t *p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// Relaxed polls (an acquire load at gpu scope invalidates the SM's L1 on every poll), then one
// acquire fence once the count is reached.
__device__ __forceinline__ void spin_until_geq(const uint32_t *p, uint32_t target) {
    while (ld_relaxed_u32(p) < target)
        __nanosleep(64);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Grid-wide barrier over co-resident CTAs (thread 0 arrives; the generation word is monotone
// across launches, the count self-resets).  Returns the new generation (unique per barrier).
__device__ __forceinline__ uint32_t grid_sync(uint32_t *count, uint32_t *gen, uint32_t ctas, uint32_t *gen_out_smem) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t g = ld_relaxed_u32(gen);
        __threadfence();
        if (atomicAdd(count, 1u) == ctas - 1u) {
            *count = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (ld_relaxed_u32(gen) == g)
                __nanosleep(32);
        }
        __threadfence();
        *gen_out_smem = g + 1u;
    }
    __syncthreads();
    return *gen_out_smem;
}

}  // namespace fused

using namespace fused;

__global__ void __launch_bounds__(kThreads, 1) aid_stage_kernel(AidStageParams P) {
    const InferParams &p = P.f;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem_w = smem_raw;
    Smem &S = *reinterpret_cast<Smem *>(smem_raw + smem_offset_tail(p.blob_bytes));
    ws::SmemTail *st = &S.st;
    uint8_t *slots_s = smem_raw + smem_offset_slots(p.blob_bytes);
    uint8_t *tab_s = smem_raw + smem_offset_table(p.blob_bytes);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t G = gridDim.x, b = blockIdx.x;
    const GridDev &gd = p.grid_rrs;
    const uint32_t L = (uint32_t)gd.levels;
    const uint64_t n = p.n;
    const uint32_t num_tiles = (uint32_t)((n + kTileM - 1) / kTileM);
    const uint32_t tpc = P.tpc, rounds = P.rounds;
    const uint32_t t0 = b * tpc;
    const uint32_t my_tiles = t0 >= num_tiles ? 0u : (num_tiles - t0 < tpc ? num_tiles - t0 : tpc);
    // level served by this CTA's producers
    const uint32_t lvl = b % L, pq = b / L, pnq = (G - lvl + L - 1) / L;
    const uint32_t c_lo = G * pq / pnq, c_hi = G * (pq + 1) / pnq;  // consumer CTAs served
    const uint32_t lres = (uint32_t)gd.base_resolution << lvl, lnn = lres + 1u;
    const bool ldense = (gd.dense_mask >> lvl) & 1u;
    const uint32_t tab_bytes = ldense ? ((lnn * lnn * lnn * 4u + 15u) & ~15u) : gd.table_size * 4u;

    // ---- setup: weights, descriptors, barriers, TMEM, this CTA's level table ----
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(p.blob);
        uint4 *dst = reinterpret_cast<uint4 *>(smem_w);
        for (uint32_t i = tid; i < p.blob_bytes / 16u; i += kThreads)
            dst[i] = __ldg(src + i);
    }
    if (tid == 0) {
        const NetDesc &nd = p.nets.rrs;
        for (int l = 0; l < 4; ++l) {
            const LayerDesc &Ld = nd.layer[l];
            st->idesc_n[1][l] = make_idesc_f16(Ld.N);
            st->idesc_2n[1][l] = make_idesc_f16(2u * Ld.N);
            st->nslices[1][l] = (uint32_t)Ld.K / 16u;
            st->bias[1][l] = Ld.bias;
            const uint32_t sbo = (uint32_t)Ld.K * 16u;
            for (int k = 0; k < 2; ++k) {
                st->wdesc[1][l][k] = make_smem_desc(smem_u32(smem_w + Ld.w_hi) + 256u * k, 128u, sbo);
                st->wdesc_lo[1][l][k] =
                    make_smem_desc(smem_u32(smem_w + Ld.w_hi) + 256u * k + ((uint32_t)Ld.N / 8u) * sbo, 128u, sbo);
            }
        }
        for (int m = 0; m < kGM; ++m) {
            mbar_init(&st->mma_bar[m], 1);
            mbar_init(&S.full[m], 1);
            mbar_init(&S.slot_free[m], 1);
        }
        mbar_init(&S.table_bar, 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(&S.table_bar, tab_bytes);
        const uint8_t *src = reinterpret_cast<const uint8_t *>(p.rrs_grid) + (uint64_t)lvl * gd.table_size * 4u;
        for (uint32_t off = 0; off < tab_bytes; off += 32768u)
            bulk_g2s(tab_s + off, src + off, tab_bytes - off < 32768u ? tab_bytes - off : 32768u, &S.table_bar);
    }
    if (warp == 0)
        tmem_alloc(&st->tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = st->tmem_base;

#ifdef NRRS_KERNEL_TIMING
        if (P.dbg && tid == 0) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            P.dbg[b * 8 + 0] = tt;
        }
#endif
    const uint32_t lane_base = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t *produced = P.sync + 2u * kPad;                      // [kRoundSlots] padded
    uint32_t *consumed = produced + (uint32_t)kRoundSlots * kPad;  // [kRoundSlots] padded
    const uint32_t ring_round = L * G * (uint32_t)kGM * kTileM;   // float2 per ring slot
    Fx128 my_fx{0ull, 0ull};  // exact sum of q (fixed point)
    uint32_t my_nonfinite = 0, my_bc = 0;

    if (warp < kLoaderWarp) {
        // ================================ producers ================================
        const uint32_t pt = (uint32_t)tid;
        LevelConsts c;
        c.res = lres;
        c.nn = lnn;
        c.m4 = (gd.table_size - 1u) * 4u;
        c.resf = (float)lres;
        c.dense = ldense;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            c.doff4[k] = (((k & 1) * lnn + ((k >> 1) & 1)) * lnn + (k >> 2)) * 4u;
        const uint32_t items = (c_hi - c_lo) * (uint32_t)kGM * kTileM;  // vertex slots per round
        mbar_wait(&S.table_bar, 0);
        for (uint32_t r = 0; r < rounds; ++r) {
            const uint32_t slot = r % kRoundSlots;
            if (r >= (uint32_t)kRoundSlots) {  // ring slot reuse: every CTA's loader released round r - 3
                if (pt == 0)
                    spin_until_geq(consumed + slot * kPad, G * (r / kRoundSlots));
                named_bar_sync(1, kProdThreads);
            }
            float2 *ring = P.ring + (uint64_t)slot * ring_round + ((uint64_t)lvl * G + c_lo) * kGM * kTileM;
            // item i -> consumer CTA c_lo + i / (GM*128), group m, row
            auto vertex_of = [&](uint32_t i, uint64_t &v) -> bool {
                const uint32_t cb = c_lo + i / (kGM * kTileM), rem = i % (kGM * kTileM);
                const uint32_t tl = r * kGM + rem / kTileM;  // consumer-local tile
                const uint32_t t = cb * tpc + tl;
                v = (uint64_t)t * kTileM + rem % kTileM;
                return tl < tpc && t < num_tiles && v < n;
            };
            float pv[kProdPer][3];
            auto load = [&](uint32_t i0) {
#pragma unroll
                for (int u = 0; u < kProdPer; ++u) {
                    const uint32_t i = i0 + (uint32_t)u * kProdThreads;
                    uint64_t v;
                    if (i < items && vertex_of(i, v)) {
                        const float *g3 = p.p01 + 3 * v;
                        pv[u][0] = __ldg(g3);
                        pv[u][1] = __ldg(g3 + 1);
                        pv[u][2] = __ldg(g3 + 2);
                    } else {
                        pv[u][0] = pv[u][1] = pv[u][2] = 0.0f;
                    }
                }
            };
            load(pt);
            for (uint32_t i0 = pt; i0 < items; i0 += kProdPer * kProdThreads) {
                float cur[kProdPer][3];
#pragma unroll
                for (int u = 0; u < kProdPer; ++u) {
                    cur[u][0] = pv[u][0];
                    cur[u][1] = pv[u][1];
                    cur[u][2] = pv[u][2];
                }
                if (i0 + kProdPer * kProdThreads < items)
                    load(i0 + kProdPer * kProdThreads);
                float2 f[kProdPer];
#pragma unroll
                for (int u = 0; u < kProdPer; ++u)
                    f[u] = level_encode(tab_s, c, cur[u][0], cur[u][1], cur[u][2]);
#pragma unroll
                for (int u = 0; u < kProdPer; ++u) {
                    const uint32_t i = i0 + (uint32_t)u * kProdThreads;
                    if (i < items)
                        ring[i] = f[u];  // [consumer CTA c_lo + ...][group][row] of this level
                }
            }
            // the barrier orders every producer thread's plane stores before thread 0's release
            named_bar_sync(1, kProdThreads);
            if (pt == 0)
                red_release_add(produced + slot * kPad, 1u);
        }

#ifdef NRRS_KERNEL_TIMING
        if (P.dbg && pt == 0) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            P.dbg[b * 8 + 1] = tt;
        }
#endif
    } else if (warp == kLoaderWarp) {
        // ================================= loader =================================
        if (lane == 0) {
            const bool bulk_in = p.in_bulk != 0u;
            uint32_t full_phase = 0;  // bit m: parity of full[m]'s next phase
            uint32_t free_phase = 0;  // bit m: parity of slot_free[m]'s next phase
            for (uint32_t r = 0; r < rounds; ++r) {
                const uint32_t slot = r % kRoundSlots;
                spin_until_geq(produced + slot * kPad, G * (r / kRoundSlots + 1u));
                fence_proxy_async_global();
                const float2 *ring = P.ring + (uint64_t)slot * ring_round;
                uint32_t issued = 0;
                for (int m = 0; m < kGM; ++m) {
                    const uint32_t tl = r * kGM + (uint32_t)m;
                    if (tl >= my_tiles)
                        continue;
                    if (r > 0) {  // the group has moved its previous tile into TMEM
                        mbar_wait(&S.slot_free[m], (free_phase >> m) & 1u);
                        free_phase ^= 1u << m;
                    }
                    const uint64_t tile = t0 + tl, j0 = tile * kTileM;
                    const bool inputs = bulk_in && j0 + kTileM <= n;
                    uint8_t *in_s = slots_s + (uint32_t)m * kAidInBytes;
                    const uint32_t ipx_bytes = p.i_pixel ? 12u * kTileM : 4u * kTileM;
                    uint32_t bytes = L * 8u * kTileM;
                    if (inputs)
                        bytes += 12u * kTileM + 8u * kTileM + ipx_bytes + 4u * kTileM + 8u * kTileM;
                    mbar_arrive_expect_tx(&S.full[m], bytes);
                    for (uint32_t l = 0; l < L; ++l)
                        bulk_g2s(in_s + kAidInPlane * l,
                                 ring + ((uint64_t)l * G + b) * kGM * kTileM + (uint32_t)m * kTileM, 8u * kTileM,
                                 &S.full[m]);
                    if (inputs) {
                        bulk_g2s(in_s + kAidInWeight, p.weight + 3 * j0, 12u * kTileM, &S.full[m]);
                        bulk_g2s(in_s + kAidInWo, p.wo01 + 2 * j0, 8u * kTileM, &S.full[m]);
                        if (p.i_pixel)
                            bulk_g2s(in_s + kAidInIpx, p.i_pixel + 3 * j0, ipx_bytes, &S.full[m]);
                        else
                            bulk_g2s(in_s + kAidInIpx, p.pixel + j0, ipx_bytes, &S.full[m]);
                        bulk_g2s(in_s + kAidInRough, p.roughness + j0, 4u * kTileM, &S.full[m]);
                        bulk_g2s(in_s + kAidInKey, p.path_key + j0, 8u * kTileM, &S.full[m]);
                    }
                    issued |= 1u << m;
                }
                // the ring slot is free again once this round's copies have landed
                for (int m = 0; m < kGM; ++m)
                    if (issued & (1u << m)) {
                        mbar_wait(&S.full[m], (full_phase >> m) & 1u);
                        full_phase ^= 1u << m;
                    }
                red_release_add(consumed + slot * kPad, 1u);
            }

#ifdef NRRS_KERNEL_TIMING
        if (P.dbg && true) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            P.dbg[b * 8 + 2] = tt;
        }
#endif
        }
        __syncwarp();
    } else {
        // =============================== MLP groups ===============================
        const int g = (warp - kMlpWarp0) >> 2, r = tid & 127;
        const bool issuer = r == 0;
        const uint32_t bar_id = 2u + (uint32_t)g;
        const uint32_t col_d = 64u * (uint32_t)g, col_a = col_d + 32u;
        const bool depth1 = p.depth == 1u;
        uint8_t *in_s = slots_s + (uint32_t)g * kAidInBytes;
        uint32_t phase = 0, in_phase = 0;
        for (uint32_t rr = 0; rr < rounds; ++rr) {
            const uint32_t tl = rr * kGM + (uint32_t)g;
            if (tl >= my_tiles)
                break;
            const uint64_t tile = t0 + tl;
            const uint64_t j = tile * kTileM + r;
            const bool valid = j < n;
            const bool staged = p.in_bulk != 0u && tile * kTileM + kTileM <= n;
            mbar_wait_sleep(&S.full[g], in_phase, 20000u);  // parked, not polling: producers need the issue slots
            in_phase ^= 1u;
            // ---- row inputs: level planes (smem) + tail inputs ----
            float f[16];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                float2 v = make_float2(0.0f, 0.0f);
                if (q < (int)L)
                    v = reinterpret_cast<const float2 *>(in_s + kAidInPlane * q)[r];
                f[2 * q] = v.x;
                f[2 * q + 1] = v.y;
            }
            float wx = 0, wy = 0, wz = 0, wox = 0, woy = 0, ia = 0, ib = 0, ic = 0, rough = 0;
            uint64_t key = 0;
            if (staged) {
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
            } else if (valid) {
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
            ws::ws_store_a16(lane_base, col_a, 0, x0);
            ws::ws_store_a16(lane_base, col_a, 1, x1);
            tmem_wait_st();
            tc_fence_before();
            named_bar_sync(bar_id, 128);
            if (issuer)
                ws::ws_issue(st, 1, 0, tmem_base, col_a, col_d, &st->mma_bar[g]);
            if (r == 32)  // every row of the slot has been read (barrier above): hand it back
                mbar_arrive(&S.slot_free[g]);
            // ---- 4-layer chain ----
#pragma unroll 1
            for (int l = 0; l < 4; ++l) {
                mbar_wait_sleep(&st->mma_bar[g], phase, 20000u);
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
                    float uv = 1.0f;  // padding rows: q = 0, u = 1 -> count 0
                    if (valid) {
                        uv = rrs_uniform(p.mixed_seed, key, p.depth);
                        if (p.q_out)
                            p.q_out[j] = qv;
                        if (p.u_out)
                            p.u_out[j] = uv;
                        if (p.decided_out)
                            p.decided_out[j] = (uint8_t)decided;
                        fx_add_q(my_fx, qv);
                    } else {
                        qv = 0.0f;
                    }
                    if (P.park_tmem)
                        tmem_st2(lane_base + kParkCol + 2u * tl, qv, uv);
                    tc_fence_before();
                }
            }
        }

#ifdef NRRS_KERNEL_TIMING
        if (P.dbg && tid == 0) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            P.dbg[b * 8 + 3] = tt;
        }
#endif
        tmem_wait_st();
    }

    // ======================= decision tail (all warps) =======================
    // CTA partials of q (fixed tree over the threads), then the grid barrier
    {
        const Fx128 sv = fx_warp_sum(my_fx);
        const uint32_t nf = __reduce_add_sync(0xffffffffu, my_nonfinite);
        const uint32_t bcs = __reduce_add_sync(0xffffffffu, my_bc);
        if (lane == 0) {
            S.red_fx[warp] = sv;
            S.red_nf[warp] = nf;
            S.red_bc[warp] = bcs;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        Fx128 cs{0ull, 0ull};
        uint32_t cn = 0, cb = 0;
        for (int w = 0; w < 32; ++w) {
            fx_add(cs, S.red_fx[w]);
            cn += S.red_nf[w];
            cb += S.red_bc[w];
        }
        reinterpret_cast<Fx128 *>(p.parts)[b] = cs;
        p.part_counts[2 * b] = cn;
        p.part_counts[2 * b + 1] = cb;
    }
    grid_sync(P.sync, P.sync + kPad, G, &S.gen1);
    const uint32_t gen1 = S.gen1;

#ifdef NRRS_KERNEL_TIMING
        if (P.dbg && tid == 0) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            P.dbg[b * 8 + 4] = tt;
        }
#endif
    if (b == 0 && tid == 32) {  // every role of every CTA is past the ring: reset its counters
        for (int s = 0; s < kRoundSlots; ++s) {
            produced[s * kPad] = 0u;
            consumed[s * kPad] = 0u;
        }
    }
    // sum of q over the whole batch in CTA order (identical on every CTA)
    if (warp == 0) {
        Fx128 fx{0ull, 0ull};  // exact, so every CTA (and K-A0 + K-A + K-B) gets the same bits
        uint32_t nf = 0, bcs = 0;
        for (uint32_t c = lane; c < G; c += 32) {
            const unsigned long long *pp = reinterpret_cast<const unsigned long long *>(p.parts) + 2 * c;
            fx_add(fx, Fx128{__ldcg(pp), __ldcg(pp + 1)});
            nf += __ldcg(p.part_counts + 2 * c);
            bcs += __ldcg(p.part_counts + 2 * c + 1);
        }
        fx = fx_warp_sum(fx);
        const double sv = fx_to_double(fx);
        nf = __reduce_add_sync(0xffffffffu, nf);
        bcs = __reduce_add_sync(0xffffffffu, bcs);
        if (lane == 0) {
            S.sum_all = sv;
            if (b == 0) {
                *p.sum_out = sv;
                p.res->sum_q = sv;
                p.res->sum_fx[0] = fx.lo;
                p.res->sum_fx[1] = fx.hi;
                p.res->nonfinite = nf;
                p.res->box_cox_clamps = bcs;
            }
        }
    }
    __syncthreads();
    const double sum = S.sum_all;
    bool apply = false;
    float scale = 1.0f;
    if (sum > 0.0) {
        const double F = __ddiv_rn((double)P.n_pixels, sum);  // F = Npx / sum (rrs.cpp:17)
        if (F < 1.0) {
            apply = true;
            scale = __double2float_rn(F);  // s = float(F) (rrs.cpp:19)
        }
        if (b == 0 && tid == 0)
            p.res->f_norm = F;
    } else if (b == 0 && tid == 0) {
        p.res->f_norm = 1.0;
    }
    const float gain = P.gain;
    // one 32-vertex chunk = rows [32 qd, 32 qd + 32) of tile tl: the lanes of warp quadrant qd
    const uint32_t qd = (uint32_t)(warp & 3), wsub = (uint32_t)(warp >> 2);  // 8 warps per quadrant
    auto load_qu = [&](uint32_t tl, float &q, float &u) {
        const uint64_t v = (uint64_t)(t0 + tl) * kTileM + 32u * qd + (uint32_t)lane;
        if (P.park_tmem) {
            tmem_ld2(lane_base + kParkCol + 2u * tl, q, u);
        } else if (v < n) {
            q = __ldcg(p.q_out + v);
            u = __ldcg(p.u_out + v);
        } else {
            q = 0.0f;
            u = 1.0f;
        }
    };
    auto count_of = [&](float q, float u, float &qn, float &qr) -> uint32_t {
        qn = apply ? __fmul_rn(q, scale) : q;  // q *= float(F) (rrs.cpp:18-21)
        qr = __fmul_rn(qn, gain);              // q_real = q * gain (wavefront.cpp:396)
        return stochastic_round(qr, u);        // (rrs.cpp:35-45)
    };
    // the level table is done (every producer passed the barrier): its smem holds the per-warp
    // slot staging buffers (64 KB) and the 32-vertex chunk counts / bases (<= 16K chunks)
    uint2 *wbuf = reinterpret_cast<uint2 *>(tab_s) + (uint32_t)warp * kStage;
    uint32_t *chunk = reinterpret_cast<uint32_t *>(tab_s + 32u * kStage * sizeof(uint2));
    // pass A: chunk counts
    for (uint32_t tl = wsub; tl < my_tiles; tl += 8u) {
        float q, u, qn, qr;
        load_qu(tl, q, u);
        const uint32_t k = count_of(q, u, qn, qr);
        const uint32_t s = __reduce_add_sync(0xffffffffu, k);
        if (lane == 0)
            chunk[4u * tl + qd] = s;
    }
    __syncthreads();
#ifdef NRRS_KERNEL_TIMING
    if (P.dbg && tid == 0) {
        unsigned long long tt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
        P.dbg[b * 8 + 6] = tt;
    }
#endif
    if (warp == 0) {  // exclusive scan over the CTA's chunks in vertex order
        const uint32_t nch = 4u * my_tiles;
        const uint32_t per = (nch + 31u) / 32u, c0 = (uint32_t)lane * per;
        uint32_t s = 0;
        for (uint32_t c = c0; c < c0 + per && c < nch; ++c)
            s += chunk[c];
        uint32_t inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o)
                inc += t;
        }
        uint32_t run = inc - s;
        for (uint32_t c = c0; c < c0 + per && c < nch; ++c) {
            const uint32_t v = chunk[c];
            chunk[c] = run;
            run += v;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
        // exclusive prefix of this CTA: its predecessors' published totals (all CTAs resident)
        const uint64_t word = ((uint64_t)gen1 << 32) | total;
        if (lane == 0)
            st_relaxed_u64(P.state + (uint64_t)b * kStatePad, word);
        uint64_t pre = 0;
        uint64_t sv[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const uint32_t c = (uint32_t)lane + 32u * (uint32_t)i;
            sv[i] = c < b ? ld_relaxed_u64(P.state + (uint64_t)c * kStatePad) : 0ull;
        }
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const uint32_t c = (uint32_t)lane + 32u * (uint32_t)i;
            if (c < b) {
                while ((uint32_t)(sv[i] >> 32) != gen1)
                    sv[i] = ld_relaxed_u64(P.state + (uint64_t)c * kStatePad);
                pre += sv[i] & 0xFFFFFFFFull;
            }
        }
        for (uint32_t c = (uint32_t)lane + 160u; c < b; c += 32u) {  // G > 160 (not on B200)
            uint64_t w;
            while (((w = ld_relaxed_u64(P.state + (uint64_t)c * kStatePad)) >> 32) != gen1) {
            }
            pre += w & 0xFFFFFFFFull;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            pre += __shfl_xor_sync(0xffffffffu, pre, o);
        if (lane == 0) {
            S.prefix = pre;
            S.cta_total = total;
            if (b == G - 1) {
                const uint64_t all = pre + total, cap = P.capacity;
                const uint64_t spawned = all < cap ? all : cap;
                if (P.total_out)
                    *P.total_out = all;
                p.res->total = all;
                p.res->spawned = (uint32_t)spawned;
                p.res->dropped = all - spawned;
                p.res->overflow = all > spawned ? 1u : 0u;
            }
        }
    }
    __syncthreads();
#ifdef NRRS_KERNEL_TIMING
    if (P.dbg && tid == 0) {
        unsigned long long tt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
        P.dbg[b * 8 + 7] = tt;
    }
#endif
    // pass B: outputs (wavefront.cpp:148, :421-425, :436)
    const uint64_t Pfx = S.prefix, cap = P.capacity;
    for (uint32_t tl = wsub; tl < my_tiles; tl += 8u) {
        float q, u, qn, qr;
        load_qu(tl, q, u);
        const uint32_t k = count_of(q, u, qn, qr);
        uint32_t inc = k;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o)
                inc += t;
        }
        const uint32_t cbase = chunk[4u * tl + qd];  // CTA-relative first position of the chunk
        const uint32_t gtot = __shfl_sync(0xffffffffu, inc, 31);
        const uint64_t cum = Pfx + cbase + inc - k;
        const uint64_t v = (uint64_t)(t0 + tl) * kTileM + 32u * qd + (uint32_t)lane;
        if (v < n) {
            P.q_norm[v] = qn;
            P.q_real[v] = qr;
            if (P.offset)
                P.offset[v] = (uint32_t)(cum < cap ? cum : cap);  // min(cum, capacity)
            if (P.k_out)
                P.k_out[v] = (int32_t)k;
        }
        if (P.slots) {
            const uint64_t gb = Pfx + cbase;  // the chunk's first slot
            const uint32_t kept = cum < cap ? (uint32_t)min((uint64_t)k, cap - cum) : 0u;
            const uint32_t rel = inc - k;
            const uint32_t jj = (uint32_t)v + P.parent_base;
            uint2 *slots = reinterpret_cast<uint2 *>(P.slots);
            for (uint32_t c = 0; c < kept; ++c) {
                if (rel + c < (uint32_t)kStage)
                    wbuf[rel + c] = make_uint2(jj, c);
                else
                    slots[cum + c] = make_uint2(jj, c);
            }
            __syncwarp();
            const uint64_t room = gb < cap ? cap - gb : 0;
            uint32_t nw = (uint64_t)gtot < room ? gtot : (uint32_t)room;
            nw = nw < (uint32_t)kStage ? nw : (uint32_t)kStage;
            for (uint32_t i = (uint32_t)lane; i < nw; i += 32u)
                __stcs(slots + gb + i, wbuf[i]);
            __syncwarp();
        }
    }

#ifdef NRRS_KERNEL_TIMING
        if (P.dbg && tid == 0) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            P.dbg[b * 8 + 5] = tt;
        }
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        tmem_dealloc(tmem_base, 512);
}

// ---------------------------------------------------------------------------
size_t aid_stage_smem_bytes(uint32_t blob_bytes, uint32_t table_size) {
    return (size_t)smem_offset_table(blob_bytes) + (size_t)table_size * 4u;
}

uint32_t aid_stage_ring_floats2(uint32_t levels, uint32_t ctas) {
    return (uint32_t)kRoundSlots * levels * ctas * (uint32_t)kGM * kTileM;
}

uint32_t aid_stage_sync_words() { return (2u + 2u * kRoundSlots) * kPad; }

// Grid / round shape of the fused stage for n vertices on num_sms SMs; false if the fused kernel
// does not apply (too few tiles for one producer per level, or more tiles per CTA than TMEM parks
// while the q / u scratch is absent).
bool aid_stage_shape(uint64_t n, int num_sms, uint32_t levels, uint32_t *ctas, uint32_t *tpc, uint32_t *rounds,
                     uint32_t *park) {
    const uint64_t tiles = (n + kTileM - 1) / kTileM;
    uint64_t G = (uint64_t)num_sms;
    if (G > tiles)
        G = tiles;
    if (G < levels || levels > 8 || G > 160)
        return false;
    const uint64_t per = (tiles + G - 1) / G;
    G = (tiles + per - 1) / per;  // every CTA owns at least one tile
    if (G < levels)
        return false;
    *ctas = (uint32_t)G;
    *tpc = (uint32_t)per;
    *rounds = (uint32_t)((per + kGM - 1) / kGM);
    *park = per <= kMaxParkTiles ? 1u : 0u;
    return per * 4u <= 16384u;  // chunk table in the freed level-table smem
}

cudaError_t launch_aid_stage(const AidStageParams &p, uint32_t ctas, cudaStream_t stream) {
    const size_t smem = aid_stage_smem_bytes(p.f.blob_bytes, p.f.grid_rrs.table_size);
    cudaError_t e = cudaFuncSetAttribute(aid_stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, aid_stage_kernel, p);
}

}  // namespace nrrs
