// Microbenchmark: latency of a dependent tcgen05.mma (+commit +mbarrier wait) round trip
// on one CTA, M=128 N=32 K=16 kind::f16, A from TMEM (TS) or smem (SS).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_07868_b200/csrc tools/mma_latency.cu -o /tmp/mma_latency
#include "nrrs_device.cuh"
#include <cstdio>
using namespace nrrs;

__global__ void bench(int mode, int nmma, int iters, unsigned long long *out) {
    __shared__ __align__(1024) uint8_t smem[16384];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3C003C00u;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (threadIdx.x < 32) tmem_alloc(&tbase, 128);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tbase;
    const uint32_t idesc = make_idesc_f16(32);
    uint32_t phase = 0;
    unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            for (int k = 0; k < nmma; ++k) {
                const uint64_t b = make_smem_desc(smem_u32(smem) + 8192, 128, 256);
                if (mode == 0) {
                    mma_f16_ts(tb, tb + 64 + 8 * (k & 1), b, idesc, k > 0);
                } else {
                    const uint64_t a = make_smem_desc(smem_u32(smem), 128, 256);
                    mma_f16(tb, a, b, idesc, k > 0);
                }
            }
            mma_commit(&bar);
            mbar_wait(&bar, phase);
            phase ^= 1;
            tc_fence_after();
        }
        out[mode * 16 + nmma] = (clock64() - t0) / iters;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tb, 128);
}

int main() {
    unsigned long long *d, h[32] = {0};
    cudaMalloc(&d, sizeof h);
    cudaMemset(d, 0, sizeof h);
    for (int mode = 0; mode < 2; ++mode)
        for (int n : {1, 2, 4, 8})
            bench<<<1, 128>>>(mode, n, 2000, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("status %s\n", cudaGetErrorString(e));
    for (int mode = 0; mode < 2; ++mode)
        for (int n : {1, 2, 4, 8})
            printf("%s nmma=%d: %llu cycles per dependent round trip\n", mode ? "SS" : "TS", n, h[mode * 16 + n]);
    return 0;
}
