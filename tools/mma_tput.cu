// Microbenchmark: tcgen05.mma kind::f16 M=128 K=16 cost vs N, dependent (same D) vs
// independent (distinct D) chains of 8 MMAs, A from TMEM.
#include "nrrs_device.cuh"
#include <cstdio>
using namespace nrrs;

__device__ __forceinline__ uint32_t idesc_n(uint32_t n) { return make_idesc_f16(n); }

__global__ void bench(int n, int indep, int iters, unsigned long long *out) {
    __shared__ __align__(1024) uint8_t smem[16384];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3C003C00u;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tbase;
    const uint32_t idesc = idesc_n(n);
    uint32_t phase = 0;
    const uint64_t b = make_smem_desc(smem_u32(smem), 128, 256);
    unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            for (int k = 0; k < 8; ++k) {
                const uint32_t d = indep ? tb + (uint32_t)((k * n) % 448) : tb;
                mma_f16_ts(d, tb + 448 + 8 * (k & 1), b, idesc, indep ? 0u : (k > 0));
            }
            mma_commit(&bar);
            mbar_wait(&bar, phase);
            phase ^= 1;
            tc_fence_after();
        }
        out[0] = (clock64() - t0) / iters;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tb, 512);
}

int main() {
    unsigned long long *d, h;
    cudaMalloc(&d, 8);
    for (int n : {16, 32, 64, 128, 256})
        for (int indep : {0, 1}) {
            if (indep && n > 56) { if (n != 64) continue; }
            bench<<<1, 128>>>(n, indep, 2000, d);
            cudaDeviceSynchronize();
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("N=%3d %s: %llu cycles per 8-MMA round trip\n", n, indep ? "independent D" : "same D     ", h);
        }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
