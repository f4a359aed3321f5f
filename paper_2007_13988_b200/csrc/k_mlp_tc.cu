// k_mlp_tc.cu — tcgen05/TMEM fused PIFu MLP (placeholder until the tensor-core
// engine lands; FP32/BF16 precisions report EINVAL until then).
#include "eval_common.cuh"

namespace icg {

size_t tc_stream_bytes(int) { return 0; }
size_t tc_bias_floats(int) { return 0; }
size_t tc_wlast_floats(int) { return 0; }
int tc_pack_mlp(int, const float* const*, const float* const*, uint8_t*, float*, float*) { return ICG_OK; }

int launch_pifu_tc_eval(const FieldDev&, const TcMlp&, const EvalJob&, unsigned int, bool, cudaStream_t) {
    set_error("tensor-core MLP not available in this build");
    return ICG_EINVAL;
}
int launch_pifu_tc_texture(const FieldDev&, const TcMlp&, const TcMlp&, const EvalJob&, unsigned int, bool,
                           cudaStream_t) {
    set_error("tensor-core MLP not available in this build");
    return ICG_EINVAL;
}

}  // namespace icg
