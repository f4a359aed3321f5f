// k_features.cu — on-device feature producer (the encoder stand-in of the frame stream, SURVEY.md
// §8(e)/(f)4): a seeded C x H x W map of N(0, 1) values generated where it is consumed, so a
// stream of frames needs no host generation and no H2D copy of its 16.8 / 67 MB feature maps.
//
// Counter-based: element e = c H W + y W + x draws Philox4x32-10 at counter (e, 0, 0, 0) under key
// (seed lo, seed hi); a = (hi:lo of words 0, 1) >> 11 and b = (words 2, 3) >> 11 as 53-bit
// uniforms (x 2^-53, a = 2^-53 if 0), then the reference's Box-Muller form sqrt(-2 ln a)
// cos(2 pi b) (random.hpp:32-37) in fp64, rounded to fp32.  (A different stream from the host
// Rng's mt19937_64; the oracle restates it for parity.)  One thread per element, coalesced.
#include "icg_internal.h"

namespace icg {

__device__ __forceinline__ void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        c[1] = (uint32_t)p1;
        c[3] = (uint32_t)p0;
        c[0] = n0;
        c[2] = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

__global__ void __launch_bounds__(256) k_feature_normals(uint64_t seed, size_t n, float* __restrict__ out) {
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        uint32_t c[4] = {(uint32_t)e, (uint32_t)(e >> 32), 0u, 0u};
        philox10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
        double a = (double)((((uint64_t)c[0] << 32) | c[1]) >> 11) * 0x1.0p-53;
        const double b = (double)((((uint64_t)c[2] << 32) | c[3]) >> 11) * 0x1.0p-53;
        if (a <= 0.0) a = 0x1.0p-53;
        out[e] = (float)(sqrt(-2.0 * log(a)) * cos(2.0 * 3.14159265358979323846 * b));
    }
}

int launch_feature_normals(uint64_t seed, size_t n, float* out, cudaStream_t s) {
    const unsigned blocks = (unsigned)((n + 255) / 256 < 148u * 64u ? (n + 255) / 256 : 148u * 64u);
    k_feature_normals<<<blocks ? blocks : 1, 256, 0, s>>>(seed, n, out);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

}  // namespace icg
