// tma_stream_bench.cu — dev microbenchmark: per-SM bulk-copy streaming rate when
// every SM streams the same L2-resident weight set through an S-stage ring
// (the k_mlp_pair / k_lp access pattern), no compute.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_stream_bench.cu -o tma_stream_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2007_13988_b200/csrc/tc_ptx.cuh"

using namespace icg;

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(ptx::smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_try_hint(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(ptx::smem_u32(bar)), "r"(parity), "r"(20)
        : "memory");
    return ok != 0;
}
__device__ int g_mode;


__global__ void __launch_bounds__(64, 1) stream(const uint8_t* src, size_t set_bytes, int tile, int stages, int iters, int split,
                                                unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t full[16];
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) ptx::mbar_init(&full[s], 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int ntiles = (int)(set_bytes / tile);
    unsigned long long t0 = clock64();
    int issued = 0, done = 0;
    const int total = iters;
    // prime
    while (issued < total && issued < stages) {
        const int s = issued % stages;
        ptx::mbar_arrive_expect_tx(&full[s], tile);
        for (int c = 0; c < split; ++c)
            ptx::bulk_g2s(smem + (size_t)s * tile + c * (tile / split),
                          src + (size_t)((issued + blockIdx.x) % ntiles) * tile + c * (tile / split), tile / split, &full[s]);
        ++issued;
    }
    while (done < total) {
        const int s = done % stages;
        if (g_mode == 0)
            ptx::mbar_wait(&full[s], (done / stages) & 1);
        else if (g_mode == 1)
            while (!mbar_test(&full[s], (done / stages) & 1)) {
            }
        else
            while (!mbar_try_hint(&full[s], (done / stages) & 1)) {
            }
        ++done;
        if (issued < total) {
            const int s2 = issued % stages;
            ptx::mbar_arrive_expect_tx(&full[s2], tile);
            for (int c = 0; c < split; ++c)
                ptx::bulk_g2s(smem + (size_t)s2 * tile + c * (tile / split),
                              src + (size_t)((issued + blockIdx.x) % ntiles) * tile + c * (tile / split), tile / split,
                              &full[s2]);
            ++issued;
        }
    }
    out[blockIdx.x] = clock64() - t0;
}

int main() {
    const size_t set = 5 << 20;
    uint8_t* src;
    cudaMalloc(&src, set);
    cudaMemset(src, 1, set);
    unsigned long long* out;
    cudaMallocManaged(&out, 1024 * 8);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Case { int grid, tile, stages, split; };
    const Case cases[] = {{148, 32768, 4, 1}, {1, 16384, 4, 1}, {1, 32768, 4, 1}, {148, 16384, 4, 1}, {148, 32768, 4, 1},
                          {148, 16384, 8, 1}};
    for (int mode = 0; mode < 3; ++mode)
    for (const Case& c : cases) {
        cudaMemcpyToSymbol(g_mode, &mode, 4);
        const int iters = 4000;
        stream<<<c.grid, 64, c.tile * c.stages>>>(src, set, c.tile, c.stages, iters, c.split, out);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        stream<<<c.grid, 64, c.tile * c.stages>>>(src, set, c.tile, c.stages, iters, c.split, out);
        cudaEventRecord(b);
        cudaError_t e = cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double mx = 0;
        for (int i = 0; i < c.grid; ++i) mx = mx > out[i] ? mx : out[i];
        const double bytes = (double)c.tile * iters;
        printf("mode %d grid %3d tile %6d x%2d copies stages %2d: per-SM %6.1f GB/s (%.0f cyc/stage) total %7.1f GB/s err=%d\n",
               mode, c.grid, c.tile, c.split, c.stages, bytes / (ms * 1e-3) / 1e9, mx / iters,
               bytes * c.grid / (ms * 1e-3) / 1e9, (int)e);
    }
    return 0;
}
