// tma_burst_bench.cu — dev microbenchmark: N back-to-back bulk copies (one mbarrier
// each), wait for all; is the per-SM bulk-copy engine serialising copies?
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2007_13988_b200/csrc/tc_ptx.cuh"

using namespace icg;

__global__ void __launch_bounds__(32, 1) burst(const uint8_t* src, int bytes, int n, int reps, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar[16];
    if (threadIdx.x != 0) return;
    for (int i = 0; i < n; ++i) ptx::mbar_init(&bar[i], 1);
    ptx::fence_mbar_init();
    unsigned long long best = ~0ull, first_done = 0;
    for (int r = 0; r < reps; ++r) {
        unsigned long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
            ptx::mbar_arrive_expect_tx(&bar[i], bytes);
            ptx::bulk_g2s(smem + (size_t)i * bytes, src + ((size_t)(r * n + i) % 64) * bytes, bytes, &bar[i]);
        }
        ptx::mbar_wait(&bar[0], r & 1);
        unsigned long long t1 = clock64();
        for (int i = 1; i < n; ++i) ptx::mbar_wait(&bar[i], r & 1);
        unsigned long long t2 = clock64();
        if (t2 - t0 < best) {
            best = t2 - t0;
            first_done = t1 - t0;
        }
    }
    out[0] = best;
    out[1] = first_done;
}

int main() {
    uint8_t* src;
    cudaMalloc(&src, 64 << 20);
    cudaMemset(src, 1, 64 << 20);
    unsigned long long* out;
    cudaMallocManaged(&out, 64);
    cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int bytes : {4096, 16384, 32768})
        for (int n : {1, 2, 4, 6}) {
            if ((size_t)bytes * n > 196 * 1024) continue;
            burst<<<1, 32, bytes * n>>>(src, bytes, n, 20, out);
            cudaDeviceSynchronize();
            printf("bytes %6d x %d copies: all done %6llu cyc, first done %6llu cyc\n", bytes, n, out[0], out[1]);
        }
    return 0;
}
