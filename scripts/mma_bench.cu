// mma_bench.cu — dev microbenchmark: back-to-back tcgen05.mma throughput vs shape
// (single CTA M=128 x N, and CTA-pair M=256 x N), operands static in SMEM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I.. mma_bench.cu -o mma_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2007_13988_b200/csrc/tc_ptx.cuh"

using namespace icg;

template <int N, bool PAIR, int NMMA>
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out, int reps) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) {
        if (PAIR)
            ptx::tmem_alloc2<512>(&tbase);
        else
            ptx::tmem_alloc<512>(&tbase);
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    if (PAIR)
        ptx::cluster_sync();
    else
        __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tbase;
    const bool issuer = threadIdx.x == 0 && (!PAIR || ptx::cluster_rank() == 0);
    if (issuer) {
        const uint32_t a = ptx::smem_u32(smem), b = a + 32768;
        const uint32_t idesc = ptx::idesc_bf16_f32(PAIR ? 256 : 128, N);
        const uint64_t ad = ptx::sdesc_sw128(a), bd = ptx::sdesc_sw128(b);
        uint32_t ph = 0;
        unsigned long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int i = 0; i < NMMA; ++i) {
                const uint64_t ko = (uint64_t)((i & 3) * 2);
                if (PAIR)
                    ptx::mma_bf16_pair(tmem, ad + ko, bd + ko, idesc, 1u);
                else
                    ptx::mma_bf16(tmem, ad + ko, bd + ko, idesc, 1u);
            }
            if (PAIR)
                ptx::mma_commit_pair(&bar, 1);
            else
                ptx::mma_commit(&bar);
            ptx::mbar_wait(&bar, ph);
            ph ^= 1;
        }
        unsigned long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    ptx::tc_fence_before();
    if (PAIR)
        ptx::cluster_sync();
    else
        __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        if (PAIR)
            ptx::tmem_dealloc2<512>(tmem);
        else
            ptx::tmem_dealloc<512>(tmem);
    }
}

template <int N, bool PAIR, int NMMA>
void run(const char* name) {
    auto k = bench<N, PAIR, NMMA>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    unsigned long long* out;
    cudaMallocManaged(&out, 256 * 8);
    const int reps = 200;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(PAIR ? 2 : 1);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 70000;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PAIR ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, out, reps);
    cudaDeviceSynchronize();
    cudaLaunchKernelEx(&cfg, k, out, reps);
    cudaError_t e = cudaDeviceSynchronize();
    double cyc = (double)out[0] / (reps * NMMA);
    double macs = (PAIR ? 128.0 : 128.0) * N * 16;  // per SM per MMA
    printf("%-28s err=%d  %7.1f cycles/MMA  %6.0f MAC/cycle/SM (peak ~4096)\n", name, (int)e, cyc, macs / cyc);
    cudaFree(out);
}

int main() {
    run<64, false, 4>("cta1 M128 N64  x4/commit");
    run<64, false, 16>("cta1 M128 N64  x16/commit");
    run<128, false, 16>("cta1 M128 N128 x16/commit");
    run<256, false, 16>("cta1 M128 N256 x16/commit");
    run<32, true, 16>("pair M256 N32  x16/commit");
    run<64, true, 16>("pair M256 N64  x16/commit");
    run<128, true, 4>("pair M256 N128 x4/commit");
    run<128, true, 16>("pair M256 N128 x16/commit");
    run<256, true, 16>("pair M256 N256 x16/commit");
    return 0;
}
