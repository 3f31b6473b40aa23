#include <cub/cub.cuh>
#include <cstdio>
int main() {
    const int n = 2332800;
    uint2 *in, *out; unsigned char *flags; int *nsel; void *tmp = nullptr; size_t tb = 0;
    cudaMalloc(&in, n * 8); cudaMalloc(&out, n * 8); cudaMalloc(&flags, n); cudaMalloc(&nsel, 4);
    unsigned char *h = (unsigned char *)malloc(n);
    for (int i = 0; i < n; ++i) h[i] = ((i * 2654435761u) >> 7) % 10 != 0;
    cudaMemcpy(flags, h, n, cudaMemcpyHostToDevice);
    cub::DeviceSelect::Flagged(tmp, tb, in, flags, out, nsel, n);
    cudaMalloc(&tmp, tb);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 5; ++w) cub::DeviceSelect::Flagged(tmp, tb, in, flags, out, nsel, n);
    float best = 1e9;
    for (int r = 0; r < 20; ++r) {
        cudaEventRecord(a);
        cub::DeviceSelect::Flagged(tmp, tb, in, flags, out, nsel, n);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
    }
    // scan of 2.07M u32 (K-B's look-back part)
    unsigned *ci, *co; cudaMalloc(&ci, n * 4); cudaMalloc(&co, n * 4);
    void *t2 = nullptr; size_t tb2 = 0;
    cub::DeviceScan::ExclusiveSum(t2, tb2, ci, co, 2073600); cudaMalloc(&t2, tb2);
    float best2 = 1e9;
    for (int r = 0; r < 20; ++r) {
        cudaEventRecord(a);
        cub::DeviceScan::ExclusiveSum(t2, tb2, ci, co, 2073600);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); best2 = ms < best2 ? ms : best2;
    }
    printf("cub select flagged %d x 8B: %.1f us; cub exclusive scan 2073600 u32: %.1f us\n", n, best * 1e3, best2 * 1e3);
    return 0;
}
