// nrrs_device.cuh -- device building blocks of the sm_100a NRRS stage.
//
// Bit-exactness contract: every expression that feeds an
// integer decision (luminance gate, normalization scale, gain, stochastic
// rounding) uses explicit round-to-nearest intrinsics so nvcc cannot contract
// it into an FMA; the network chain (tolerance 1e-3) may contract freely.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>

#include "nrrs_internal.h"

namespace nrrs {

// Bounds-checked diagnostics build (NRRS_BOUNDS_CHECK; compute-sanitizer is not available on the
// GPU pool): every checked index is tested on the device and a violation prints and traps, so the
// GPU suite run against this build fails loudly on an out-of-range access.  Compiles to nothing
// otherwise.
#ifdef NRRS_BOUNDS_CHECK
#define NRRS_CHECK(cond, what, a, b)                                                                        \
    do {                                                                                                    \
        if (!(cond)) {                                                                                      \
            printf("NRRS_CHECK failed: %s (%llu vs %llu) block %d thread %d\n", what, (unsigned long long)(a), \
                   (unsigned long long)(b), (int)blockIdx.x, (int)threadIdx.x);                             \
            __trap();                                                                                       \
        }                                                                                                   \
    } while (0)
#else
#define NRRS_CHECK(cond, what, a, b) \
    do {                             \
    } while (0)
#endif

// ---------------------------------------------------------------------------
// Counter-based RNG: SplitMix64 keyed PCG32 (reference rng.hpp:8-82).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix_bits(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ uint32_t pcg_output(uint64_t old) {
    const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    const uint32_t rot = (uint32_t)(old >> 59u);
    return __funnelshift_r(xs, xs, rot);  // rotate right
}

// path_stream(seed, key, depth, Draw::RrsRound).next_float()  (wavefront.cpp:397-399).
// The stream constructor advances twice (rng.hpp:37-41); the third output is u.
__device__ __forceinline__ float rrs_uniform(uint64_t mixed_seed, uint64_t key, uint32_t depth) {
    constexpr uint64_t kMul = 6364136223846793005ull;
    const uint64_t seq = mix_bits(key ^ mix_bits(((uint64_t)depth << 8) ^ 0x55ull));
    const uint64_t inc = (seq << 1u) | 1u;
    uint64_t state = inc;            // 0 * kMul + inc
    state = state + mixed_seed;      // m_state += mix_bits(seed)
    state = state * kMul + inc;      // second constructor step
    const uint32_t out = pcg_output(state);
    return __fmul_rn((float)(out >> 8), 0x1p-24f);
}

// ---------------------------------------------------------------------------
// Encodings (encodings.hpp:21-88, core.hpp:24-26)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float luminance(float x, float y, float z) {
    return __fadd_rn(__fadd_rn(__fmul_rn(0.2126f, x), __fmul_rn(0.7152f, y)), __fmul_rn(0.0722f, z));
}

__device__ __forceinline__ float clamp01(float v) { return v < 0.0f ? 0.0f : (1.0f < v ? 1.0f : v); }

template <int BINS>
__device__ __forceinline__ void one_blob(float x, float *out) {
    constexpr float sigma = 1.0f / (float)BINS;
    constexpr float inv_two_sigma2 = 1.0f / (2.0f * sigma * sigma);
    float sum = 0.0f;
#pragma unroll
    for (int i = 0; i < BINS; ++i) {
        const float c = ((float)i + 0.5f) / (float)BINS;
        const float d = x - c;
        out[i] = expf(-d * d * inv_two_sigma2);
        sum += out[i];
    }
    const float inv = 1.0f / sum;
#pragma unroll
    for (int i = 0; i < BINS; ++i)
        out[i] *= inv;
}

// box_cox with lambda = 0.5; negative inputs clamp to 0 and are counted.
__device__ __forceinline__ float box_cox(float x, uint32_t &clamps) {
    if (x < 0.0f) {
        ++clamps;
        x = 0.0f;
    }
    return (sqrtf(x) - 1.0f) * 2.0f;
}

__device__ __forceinline__ float roughness_remap(float a) { return 1.0f - expf(-a); }

__device__ __forceinline__ float softplus_mod(float x) {
    if (x < 0.0f)
        return log1pf(expf(x));
    return 0.5f * x + 0.6931471805599453f;
}

__device__ __forceinline__ float mean3(float x, float y, float z) { return (x + (y + z)) / 3.0f; }

// Tolerance-path forms of the encodings (the network inputs; q within 1e-3): single MUFU
// ops with flush-to-zero instead of the IEEE / denormal-safe sequences.  The clamp count of
// box_cox (an integer output) is the exact predicate.
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sqrt_ftz(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float box_cox_fast(float x, uint32_t &clamps) {
    if (x < 0.0f) {
        ++clamps;
        x = 0.0f;
    }
    return (sqrt_ftz(x) - 1.0f) * 2.0f;
}
__device__ __forceinline__ float mean3_fast(float x, float y, float z) { return (x + (y + z)) * (1.0f / 3.0f); }

// stochastic_round (encodings.hpp:21-27) on a sanitized q >= 0.
__device__ __forceinline__ uint32_t stochastic_round(float q, float u) {
    const float fl = floorf(q);
    const float r = __fsub_rn(q, fl);
    return (uint32_t)fl + (u < r ? 1u : 0u);
}

// ---------------------------------------------------------------------------
// tcgen05 / TMEM / mbarrier wrappers (inline PTX, sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t addr = smem_u32(bar);
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
    }
}

// Programmatic dependent launch: the dependent grid may start (its prologue overlapping this
// grid's tail) once every CTA here triggered or exited; pdl_wait() in the dependent blocks until
// this grid completed and its memory is visible.  Both are no-ops outside a PDL launch.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Named barrier over `count` threads (id 1..15; 0 is __syncthreads).
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// try_wait with a suspend-time hint (ns): for long waits, parks the thread
// instead of re-polling so it does not steal issue slots from working warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t hint_ns) {
    uint32_t done = 0;
    const uint32_t addr = smem_u32(bar);
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity), "r"(hint_ns)
            : "memory");
    }
}

// Busy-poll variant (mbarrier.test_wait never suspends the thread).
__device__ __forceinline__ void mbar_spin(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t addr = smem_u32(bar);
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Arrive on `bar` and add `bytes` to its expected transaction count.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// TMA bulk copy global -> shared (1-D, bytes % 16 == 0), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Packed fp32x2 helpers (FMUL2 / FFMA2; a pair {w, w} folds into a broadcast operand).
__device__ __forceinline__ uint64_t pk2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 upk2(uint64_t r) {
    float2 o;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
    return o;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Warp-wide: allocate `ncols` TMEM columns, base address written to *dst (smem).
__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// UMMA shared-memory matrix descriptor, K-major, SWIZZLE_NONE canonical layout
// ((8,m),(8 elems,k)) : 8x16B core matrices; lbo = byte stride between the two
// 16-byte K chunks of one K16 slice, sbo = byte stride between 8-row groups.
__device__ __forceinline__ uint64_t make_smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // version = 1 (sm_100)
    // base_offset = 0, lbo_mode = 0, layout_type = 0 (SWIZZLE_NONE)
    return d;
}

// Instruction descriptor: kind::f16, A = B = F16, D = F32, both K-major, M = 128.
__host__ __device__ constexpr uint32_t make_idesc_f16(uint32_t n) {
    return (1u << 4)              // c_format = F32
           | (0u << 7)            // a_format = F16
           | (0u << 10)           // b_format = F16
           | ((n >> 3) << 17)     // N >> 3
           | ((128u >> 4) << 24); // M >> 4
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]  (A from tensor memory, K-major, fp16 pairs per column)
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Each thread writes 8 consecutive 32-bit TMEM columns of its lane.
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i)
        v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i)
        v[i] = __uint_as_float(r[i]);
}

// Two 16-column loads (e.g. the hi and lo halves of a split accumulator), one wait.
__device__ __forceinline__ void tmem_ld16x2(uint32_t ta, uint32_t tb, float (&va)[16], float (&vb)[16]) {
    uint32_t r[16], s[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15])
        : "r"(ta));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]), "=r"(s[7]),
          "=r"(s[8]), "=r"(s[9]), "=r"(s[10]), "=r"(s[11]), "=r"(s[12]), "=r"(s[13]), "=r"(s[14]),
          "=r"(s[15])
        : "r"(tb));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        va[i] = __uint_as_float(r[i]);
        vb[i] = __uint_as_float(s[i]);
    }
}

// ---------------------------------------------------------------------------
// Decoupled look-back tile state: [63:62] flag (1 = aggregate, 2 = inclusive
// prefix), [61:48] launch epoch, [47:0] value.  Entries written by an earlier
// launch carry another epoch and read as "not yet published", so the state
// array never needs a memset between launches (LaunchSync clears it when the
// 14-bit epoch wraps).
// ---------------------------------------------------------------------------
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPrefix = 2ull << 62;
constexpr uint64_t kValueMask = (1ull << 48) - 1;

__device__ __forceinline__ void st_release_u64(uint64_t *p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Relaxed (no fence) forms: a published aggregate carries its value in the same word, so readers
// need no ordering against the publisher's other stores -- and a release would first wait for
// every store the CTA has in flight.
__device__ __forceinline__ void st_relaxed_u64(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// ---- peer mailbox (MboxDev): system-scope stores into peer memory, polls of the own mailbox ----
constexpr unsigned long long kMboxTimeoutNs = 10ull * 1000 * 1000 * 1000;  // a missing rank: error, not a hang

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// One thread: the rank's value of `kind` into its line of every rank's mailbox, value before the
// generation (st.release.sys orders it), generation = the rank's next counter value.
__device__ __forceinline__ void mbox_publish(const MboxDev *m, int kind, unsigned long long value,
                                             unsigned long long value2 = 0ull) {
    const uint32_t g = m->gen[kind] + 1u;
    m->gen[kind] = g;
    for (int r = 0; r < m->nranks; ++r) {
        unsigned long long *line = m->peer[r] + ((size_t)kind * kMboxMaxRanks + m->rank) * kMboxLineWords;
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(line + 1), "l"(value) : "memory");
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(line + 2), "l"(value2) : "memory");
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(line), "l"((unsigned long long)g) : "memory");
    }
}

// One thread: waits until every rank's line of `kind` in this rank's mailbox carries this rank's
// current generation of `kind` (its own publish of the same step already advanced it), then hands
// the values to f(rank, value, value2) in rank order.  Returns false (and raises m->err) after
// kMboxTimeoutNs.
template <typename F>
__device__ __forceinline__ bool mbox_wait(const MboxDev *m, int kind, F &&f) {
    const uint32_t g = m->gen[kind];
    const unsigned long long *mine = m->peer[m->rank] + (size_t)kind * kMboxMaxRanks * kMboxLineWords;
    const unsigned long long t0 = globaltimer_ns();
    bool ok = true;
    for (int r = 0; r < m->nranks; ++r) {
        const unsigned long long *line = mine + (size_t)r * kMboxLineWords;
        for (;;) {
            unsigned long long w;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(w) : "l"(line) : "memory");
            if ((int32_t)((uint32_t)w - g) >= 0)
                break;
            if (globaltimer_ns() - t0 > kMboxTimeoutNs) {
                atomicExch(m->err, 1u);
                ok = false;
                break;
            }
            __nanosleep(100);
        }
        unsigned long long v, v2;
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(line + 1) : "memory");
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v2) : "l"(line + 2) : "memory");
        f(r, v, v2);
    }
    return ok;
}

// ---- exact sum of the sanitized factors (normalize_factors' sum, rrs.cpp:8-24) ----
// q >= 0 accumulated as a 128-bit integer in units of 2^-40 (the high word counts 2^24).  Integer
// addition is associative, so the sum's bits do not depend on the grid, the SM count, the kernel or
// the chunking of the host paths; it is converted to double once.  A factor below 2^24 costs one
// rounded conversion (q * 2^40 < 2^64); larger ones are split at 2^24.  Terms are rounded to the
// 2^-40 grid (|error| <= 2^-41 each, ~1e-12 relative at the sums where F < 1 applies).
struct Fx128 {
    unsigned long long lo, hi;
};
__device__ __forceinline__ void fx_add(Fx128 &a, const Fx128 &b) {
    a.lo += b.lo;
    a.hi += b.hi + (a.lo < b.lo ? 1ull : 0ull);
}
__device__ __forceinline__ void fx_add_q(Fx128 &a, float q) {
    if (q < 16777216.0f) {
        fx_add(a, Fx128{__float2ull_rn(q * 1099511627776.0f), 0ull});  // q * 2^40 (exact scaling)
    } else {
        const float qh = truncf(q * 5.9604644775390625e-08f);  // floor(q / 2^24), exact
        const float ql = fmaf(qh, -16777216.0f, q);           // q - qh * 2^24, exact
        fx_add(a, Fx128{__float2ull_rn(ql * 1099511627776.0f), __float2ull_rz(qh)});
    }
}
__device__ __forceinline__ Fx128 fx_warp_sum(Fx128 a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const Fx128 b{__shfl_xor_sync(0xffffffffu, a.lo, o), __shfl_xor_sync(0xffffffffu, a.hi, o)};
        fx_add(a, b);
    }
    return a;
}
__device__ __forceinline__ double fx_to_double(const Fx128 &a) {
    return (double)a.hi * 16777216.0 + (double)a.lo * 9.094947017729282e-13;  // hi * 2^24 + lo * 2^-40
}

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Single-thread look-back: returns the exclusive prefix of `tile` and publishes
// its inclusive prefix.  Tiles are claimed in launch order (dynamic tile id),
// so predecessors always make progress.
__device__ __forceinline__ uint64_t lookback_exclusive(uint64_t *state, uint32_t tile, uint64_t aggregate,
                                                       uint32_t epoch) {
    const uint64_t tag = (uint64_t)(epoch & 0x3FFFu) << 48;
    if (tile == 0) {
        st_release_u64(&state[0], kFlagPrefix | tag | aggregate);
        return 0;
    }
    st_release_u64(&state[tile], kFlagAgg | tag | aggregate);
    uint64_t excl = 0;
    int32_t t = (int32_t)tile - 1;
    while (t >= 0) {
        uint64_t s;
        do {
            s = ld_acquire_u64(&state[t]);
        } while ((s >> 62) == 0 || ((s >> 48) & 0x3FFFu) != (epoch & 0x3FFFu));
        excl += s & kValueMask;
        if ((s >> 62) == 2)
            break;
        --t;
    }
    st_release_u64(&state[tile], kFlagPrefix | tag | (excl + aggregate));
    return excl;
}

// Warp-parallel look-back (all 32 lanes of one warp call it): each round reads
// the 32 preceding tile states at once, sums aggregates up to the nearest
// inclusive prefix.  Returns the exclusive prefix on every lane; lane 0
// publishes the tile's inclusive prefix.
__device__ __forceinline__ uint64_t lookback_warp(uint64_t *state, uint32_t tile, uint64_t aggregate,
                                                  uint32_t epoch) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t tag = (uint64_t)(epoch & 0x3FFFu) << 48;
    if (tile == 0) {
        if (lane == 0)
            st_release_u64(&state[0], kFlagPrefix | tag | aggregate);
        return 0;
    }
    if (lane == 0)
        st_release_u64(&state[tile], kFlagAgg | tag | aggregate);
    uint64_t excl = 0;
    int64_t window_end = (int64_t)tile - 1;  // lane i inspects tile window_end - i
    while (true) {
        const int64_t t = window_end - (int64_t)lane;
        uint64_t s;
        if (t >= 0) {
            do {
                s = ld_acquire_u64(&state[t]);
            } while ((s >> 62) == 0 || ((s >> 48) & 0x3FFFu) != (epoch & 0x3FFFu));
        } else {
            s = kFlagPrefix;  // virtual prefix 0 before tile 0
        }
        const uint32_t is_prefix = (uint32_t)((s >> 62) == 2);
        const uint32_t pmask = __ballot_sync(0xffffffffu, is_prefix);
        uint64_t v = s & kValueMask;
        if (pmask) {
            const uint32_t first = __ffs(pmask) - 1;  // nearest prefix
            if (lane > first)
                v = 0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (pmask)
            break;
        window_end -= 32;
    }
    if (lane == 0)
        st_release_u64(&state[tile], kFlagPrefix | tag | (excl + aggregate));
    return excl;
}

// Claims the next tile in launch order; the CTA that claims the last tile
// resets the counter for the next launch (no claims can follow it).
// Per-kernel launch bookkeeping, kept on the device so a stage captured in a
// CUDA graph replays correctly: claim = [63:32] launch epoch | [31:0] tiles
// claimed.  One atomic hands a CTA both its tile (launch order) and the epoch
// that tags its look-back states; the last CTA to finish resets the count,
// advances the epoch and, when the 14-bit tag wraps, clears the state array.
__device__ __forceinline__ uint32_t claim_tile_epoch(LaunchSync *s, uint32_t *epoch) {
    const unsigned long long v = atomicAdd(&s->claim, 1ull);
    *epoch = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

// Thread 0 of every CTA, after the CTA's last look-back access.
__device__ __forceinline__ void finish_launch(LaunchSync *s, uint64_t *state, uint32_t state_cap, uint32_t epoch) {
    __threadfence();
    if (atomicAdd(&s->done, 1u) != gridDim.x - 1)
        return;
    __threadfence();
    uint32_t next = epoch + 1u;
    if ((next & 0x3FFFu) == 0u) {  // tag wrap: no stale state may carry a reusable tag
        for (uint32_t i = 0; i < state_cap; ++i)
            state[i] = 0ull;
        next += 1u;
    }
    s->done = 0u;
    __threadfence();
    atomicExch(&s->claim, (unsigned long long)next << 32);
}

}  // namespace nrrs
