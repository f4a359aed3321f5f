// mlp_pack.cu — host-side packing of the fp32 epilogue operands every
// tensor-core field kernel shares: per-layer biases with the weight column of
// the skip input's z (rank-1 term applied in the epilogue, not by an MMA), and
// the 1- / 3-wide output layer kept in fp32 for the CUDA-core final dot.
// (The weight tiles themselves are packed per kernel: pair_pack /
// pair_pack_factored in k_mlp_pair.cu.)
#include <cstring>

#include "icg_internal.h"

namespace icg {

size_t tc_bias_floats(int which) {
    return which == ICG_MLP_GEOMETRY ? (1024 + 512 + 256 + 128 + 1) * 2 + 2 : (1024 + 512 + 256 + 128 + 3) * 2 + 2;
}
size_t tc_wlast_floats(int which) { return which == ICG_MLP_GEOMETRY ? 1 * (128 + 257) : 3 * (128 + 513); }

// bias block layout per layer l (l < 4): [b_l (out), wz_l (out)] where wz is
// the weight column of the skip's z input (the last input of every layer);
// then the final-layer biases.  wlast: final layer row-major [out][128 + skip].
int tc_pack_epilogue(int which, const float* const* w, const float* const* b, float* bias, float* wlast) {
    const bool geo = which == ICG_MLP_GEOMETRY;
    const int* outs = geo ? kGeoOut : kTexOut;
    const int skip = geo ? kGeoSkip : kTexSkip;
    int ins[5];
    for (int l = 0; l < 5; ++l) ins[l] = (l ? outs[l - 1] : 0) + skip;
    size_t off = 0;
    for (int l = 0; l < 4; ++l) {
        for (int o = 0; o < outs[l]; ++o) bias[off + o] = b[l][o];
        for (int o = 0; o < outs[l]; ++o) bias[off + outs[l] + o] = w[l][(size_t)o * ins[l] + ins[l] - 1];
        off += 2 * (size_t)outs[l];
    }
    for (int o = 0; o < outs[4]; ++o) bias[off + o] = b[4][o];
    std::memcpy(wlast, w[4], sizeof(float) * (size_t)outs[4] * ins[4]);
    return ICG_OK;
}

}  // namespace icg
