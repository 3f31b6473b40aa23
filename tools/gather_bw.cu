// Microbenchmark: scattered 8-byte gathers from a 256 KB..2 MB table (L2/L1 resident) vs
// shared-memory gathers.  Reports gathers per cycle per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/gather_bw.cu -o tools/gather_bw.bin
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

template <int ILP>
__global__ void gmem_gather(const float2 *__restrict__ t, uint32_t mask, int iters, float *out) {
    uint32_t s = hash(blockIdx.x * blockDim.x + threadIdx.x);
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float2 v[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k) { s = hash(s + k); v[k] = __ldg(t + (s & mask)); }
#pragma unroll
        for (int k = 0; k < ILP; ++k) acc += v[k].x + v[k].y;
    }
    if (acc == 12345.f) out[0] = acc;
}

template <int ILP>
__global__ void gmem_gather4(const float4 *__restrict__ t, uint32_t mask, int iters, float *out) {
    uint32_t s = hash(blockIdx.x * blockDim.x + threadIdx.x);
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float4 v[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k) { s = hash(s + k); v[k] = __ldg(t + (s & mask)); }
#pragma unroll
        for (int k = 0; k < ILP; ++k) acc += v[k].x + v[k].w;
    }
    if (acc == 12345.f) out[0] = acc;
}

template <int ILP>
__global__ void smem_gather(int entries, int iters, float *out) {
    extern __shared__ float2 tab[];
    for (int i = threadIdx.x; i < entries; i += blockDim.x) tab[i] = make_float2(i, i);
    __syncthreads();
    uint32_t s = hash(blockIdx.x * blockDim.x + threadIdx.x);
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float2 v[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k) { s = hash(s + k); v[k] = tab[s % entries]; }
#pragma unroll
        for (int k = 0; k < ILP; ++k) acc += v[k].x + v[k].y;
    }
    if (acc == 12345.f) out[0] = acc;
}

// Random 4-byte (half2) / 8-byte loads from a 2^15-entry shared-memory table (the K-A0
// level table), cheap LCG indices so the loads, not the index math, bind.
template <typename T, int ILP>
__global__ void smem_gather_pow2(uint32_t mask, int iters, float *out) {
    extern __shared__ __align__(16) uint8_t raw2[];
    T *tab2 = reinterpret_cast<T *>(raw2);
    for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) tab2[i] = T{};
    __syncthreads();
    uint32_t s[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) s[k] = hash(blockIdx.x * blockDim.x * ILP + threadIdx.x * ILP + k);
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            s[k] = s[k] * 1664525u + 1013904223u;
            const T v = tab2[(s[k] >> 9) & mask];
            acc ^= *reinterpret_cast<const uint32_t *>(&v);
        }
    }
    if (acc == 12345u) out[0] = (float)acc;
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float2 *t; float *o; cudaMalloc(&t, 64 << 20); cudaMalloc(&o, 4);
    cudaMemset(t, 0, 64 << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 256;
    for (int log2n : {12, 15, 18, 21}) {
        for (int warps : {16, 64}) {
            const int blocks = sms * 2, threads = warps * 16;
            gmem_gather<8><<<blocks, threads>>>(t, (1u << log2n) - 1, iters, o);
            cudaEventRecord(a);
            gmem_gather<8><<<blocks, threads>>>(t, (1u << log2n) - 1, iters, o);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double loads = (double)blocks * threads * iters * 8;
            double cyc = ms * 1e-3 * clk * 1e3;  // clk in kHz
            printf("gmem table %5d KB warps/SM %2d: %.2f G gathers/s, %.2f gathers/cycle/SM\n",
                   (8 << log2n) >> 10, warps, loads / ms / 1e6, loads / cyc / sms);
        }
    }
    for (int log2n : {17, 20}) {
        for (int warps : {16, 32, 64}) {
            const int blocks = sms * 2, threads = warps * 16;
            gmem_gather4<8><<<blocks, threads>>>((const float4 *)t, (1u << log2n) - 1, iters, o);
            cudaEventRecord(a);
            gmem_gather4<8><<<blocks, threads>>>((const float4 *)t, (1u << log2n) - 1, iters, o);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double loads = (double)blocks * threads * iters * 8;
            double cyc = ms * 1e-3 * clk * 1e3;
            printf("gmem float4 table %5d KB warps/SM %2d: %.2f G gathers/s, %.2f gathers/cycle/SM\n",
                   (16 << log2n) >> 10, warps, loads / ms / 1e6, loads / cyc / sms);
        }
    }
    cudaFuncSetAttribute(smem_gather<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int entries : {4913, 16384}) {
        const int blocks = sms, threads = 1024;
        smem_gather<8><<<blocks, threads, entries * 8>>>(entries, iters, o);
        cudaEventRecord(a);
        smem_gather<8><<<blocks, threads, entries * 8>>>(entries, iters, o);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double loads = (double)blocks * threads * iters * 8;
        double cyc = ms * 1e-3 * clk * 1e3;
        printf("smem table %5d entries: %.2f G gathers/s, %.2f gathers/cycle/SM\n", entries, loads / ms / 1e6,
               loads / cyc / sms);
    }
    cudaFuncSetAttribute(smem_gather_pow2<uint32_t, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(smem_gather_pow2<uint2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int width : {4, 8}) {
        for (int warps : {16, 32}) {
            const int blocks = sms, threads = warps * 32;
            const uint32_t entries = width == 4 ? 32768u : 16384u;  // 128 KB either way
            auto run = [&] {
                if (width == 4)
                    smem_gather_pow2<uint32_t, 8><<<blocks, threads, entries * 4>>>(entries - 1, iters, o);
                else
                    smem_gather_pow2<uint2, 8><<<blocks, threads, entries * 8>>>(entries - 1, iters, o);
            };
            run();
            cudaEventRecord(a);
            run();
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double loads = (double)blocks * threads * iters * 8;
            double cyc = ms * 1e-3 * clk * 1e3;
            printf("smem %d-byte random loads, 128 KB table, warps/SM %2d: %.2f G loads/s, %.2f loads/cycle/SM\n",
                   width, warps, loads / ms / 1e6, loads / cyc / sms);
        }
    }
    printf("status %s (clock %d MHz)\n", cudaGetErrorString(cudaDeviceSynchronize()), clk / 1000);
    return 0;
}
