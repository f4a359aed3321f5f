// k_analytic.cu — analytic occupancy field on sm_100a (BASELINE config 0).
//
// Replaces build_oracle's evaluator (field.hpp:83-91): O(P) = 1/(1+exp(d/tau)),
// d = union SDF of the scene (scene.hpp:103,130-146).  fp64 in the reference's
// operation order (this file is compiled with -fmad=false), then cast to fp32
// on store like evaluate_nodes (localize.hpp:86).  One thread per point; the
// kernel is compute-light (15 capsules x ~30 flops) and grid-strided over a
// device-resident count so it can sit inside a captured frame graph.
#include "eval_common.cuh"

namespace icg {

__global__ void __launch_bounds__(256) k_analytic_eval(const DevScene* __restrict__ scene, FieldDev f, EvalJob job) {
    __shared__ DevScene s;
    if (blockIdx.x * blockDim.x >= job_count(job)) {
        job_account(job);
        return;
    }
    for (int i = threadIdx.x; i < (int)(sizeof(DevScene) / 8); i += blockDim.x)
        reinterpret_cast<double*>(&s)[i] = reinterpret_cast<const double*>(scene)[i];
    __syncthreads();
    job_account(job);
    unsigned n = job_count(job);
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        double p[3];
        field_point_d(f, job, t, p);
        double d = scene_sdf(s, p);
        double occ = __ddiv_rn(1.0, __dadd_rn(1.0, exp(__ddiv_rn(d, s.tau))));
        float v = (float)occ;
        if (job_is_grid(job))
            grid_epilogue(job, job_node(job, t), v);
        else
            job.out[t] = v;
    }
}

// SceneSpec::texture_color at explicit world points (texture_batch, field.hpp:56-63); render jobs
// (out_pixel set) clamp to [0, 1] like render_view (render.hpp:276) and scatter to their pixel
__global__ void __launch_bounds__(256) k_analytic_texture(const DevScene* __restrict__ scene, EvalJob job) {
    __shared__ DevScene s;
    for (int i = threadIdx.x; i < (int)(sizeof(DevScene) / 8); i += blockDim.x)
        reinterpret_cast<double*>(&s)[i] = reinterpret_cast<const double*>(scene)[i];
    __syncthreads();
    const unsigned n = job_count(job);
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        double p[3], c[3];
        job_point_d(job, t, p);
        scene_texture(s, p, c);
        if (job.out_pixel) {
            const size_t px = (size_t)job.out_pixel[t] * 3;
            for (int d = 0; d < 3; ++d) job.out[px + d] = (float)(c[d] < 0.0 ? 0.0 : (c[d] > 1.0 ? 1.0 : c[d]));
        } else {
            for (int d = 0; d < 3; ++d) job.out[(size_t)t * 3 + d] = (float)c[d];
        }
    }
}

int launch_analytic_texture(const FieldDev& f, const EvalJob& job, unsigned int max_points, cudaStream_t s) {
    unsigned blocks = (max_points + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks == 0) blocks = 1;
    k_analytic_texture<<<blocks, 256, 0, s>>>(f.scene, job);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

int launch_analytic_eval(const FieldDev& f, const EvalJob& job, unsigned int max_points, cudaStream_t s) {
    unsigned blocks = (max_points + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks == 0) blocks = 1;
    k_analytic_eval<<<blocks, 256, 0, s>>>(f.scene, f, job);
    ICG_CUDA_TRY(cudaGetLastError());
    return ICG_OK;
}

}  // namespace icg
